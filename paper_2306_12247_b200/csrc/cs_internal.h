// Internal layout shared by the host staging code (staging.cpp), the kernels (kernels.cu) and
// the C-ABI glue (capi.cpp). Not part of the public ABI (include/capsim_b200.h).
#pragma once

#include <cstdint>
#include <string>
#include <deque>
#include <vector>

#include "../../include/capsim_b200.h"

#if defined(__CUDACC__)
#define CS_HD __host__ __device__ __forceinline__
#else
#define CS_HD inline
#endif

namespace cs {

// ---------------------------------------------------------------------------------------
// Bucketed threshold LUT.
//
// A cap c maps to its union bin  b(c) = #{distinct thresholds T_j : T_j <= c}  (bisect_right
// over the merged, de-duplicated power thresholds of all grids; policy.py:139). Non-negative
// IEEE floats order like their bit patterns, so the search runs on integer bits.
//
// fp32 (the streaming path):
//   x  = clamp((int32)bits, LO, HI)                   LO = KBASE << S1, HI = ((KBASE + NB) << S1) - 1:
//                                                    bucket 0 and NB-1 are empty guard buckets, so
//                                                    -0.0 / negatives / tiny caps land in bin 0 and
//                                                    caps above every threshold (and NaN) in the top bin
//   e  = lut[(x >> S1) - KBASE]
//   while e & 2 (redirect): s = (e >> 2) & 31; e = lut[(e >> 9) + ((x >> s) & 15)]
//   b  = (e + (x << 2)) >> 16                         one LEA + one PRMT per cap
// Leaf encoding (S <= 14 for every fp32 bucket): with the bucket [start, start + 2^S), a leaf
// holds E - (start << 2) mod 2^32 where E's hi16 = base bin (thresholds below the bucket) and
// lo16 = K: K = 0 when no threshold lies in the bucket (or it sits on the bucket start: base is
// then +1), else K = (0x4000 - (T - start)) << 2 — so e + (x << 2) = E + ((x - start) << 2)
// carries into bit 16 exactly when T <= cap, and no mask of the cap's low bits is needed (the
// clamp keeps x inside its bucket). Bit 0 (K is a multiple of 4) marks a leaf that is NOT proven
// violation-free (selected power <= every cap it serves): the kernel's per-step power check is
// an OR of that bit, with an exact recount when it is ever set. Bit 1 marks a redirect:
// (byte offset of the sub-table in the LUT << 7) | (S' << 2) | 2, the sub-table splitting its
// bucket 16 ways at S' = S - 4 (byte offsets: the kernel forms the entry's address with adds).
//
// fp64 (drop-in PowerTrace values): u = clamp(bits, LO, HI); level-1 = (u >> S1) - KBASE;
// leaf hi16 = base, bit 0 = n in {0, 1}, bit 14 = not proven violation-free; b = base +
// (n && T64[base] <= u); redirect = 0x8000|s with hi16 = sub-table index.
// ---------------------------------------------------------------------------------------
constexpr uint32_t kRedirect32 = 2u;  // fp32 redirect flag bit (leaves keep bit 1 clear)
constexpr uint32_t kMaxShift32 = 14;  // fp32 bucket shifts (the leaf's K has 14 bits)
constexpr uint32_t kRedirect = 0x8000u;        // fp64 redirect flag
constexpr int kSubFan = 16;
constexpr uint32_t kMaxSub32 = 32768;  // 15-bit sub-table id in an fp32 redirect entry

struct LutView {
  int64_t lo, hi;      // fp64: clamp bounds on the signed bit pattern
  uint64_t kbase;      // level-1 bucket offset
  uint32_t shift1;     // S1
  uint32_t sub0;       // first sub-table entry index (= level-1 size)
  const uint32_t* lut;
  const uint64_t* thr64;  // fp64 thresholds (bits), fp64 tables only
};

CS_HD uint32_t bin_f32(uint32_t bits, uint32_t s1, int32_t kbase, int32_t nb, uint32_t sub0, const uint32_t* lut) {
  const int32_t lo = kbase << s1, hi = ((kbase + nb) << s1) - 1;
  int32_t xi = (int32_t)bits;
  xi = xi < lo ? lo : xi;
  xi = xi > hi ? hi : xi;
  const uint32_t x = (uint32_t)xi;
  uint32_t e = lut[(xi >> s1) - kbase];
  while (e & kRedirect32) e = lut[(e >> 9) + ((x >> ((e >> 2) & 31u)) & 15u)];  // (e >> 7: byte offset)
  return (e + (x << 2)) >> 16;
}

CS_HD uint32_t bin_f64(uint64_t bits, int64_t lo, int64_t hi, uint32_t s1, uint64_t kbase, uint32_t sub0,
                       const uint32_t* lut, const uint64_t* thr64) {
  int64_t si = (int64_t)bits;
  si = si < lo ? lo : si;
  si = si > hi ? hi : si;
  uint64_t u = (uint64_t)si;
  uint32_t e = lut[(uint32_t)((u >> s1) - kbase)];
  while (e & kRedirect) {
    uint32_t s = e & 0x3Fu;
    e = lut[sub0 + (e >> 16) * kSubFan + (uint32_t)((u >> s) & 15u)];
  }
  uint32_t base = e >> 16;
  return base + (((e & 1u) != 0u && thr64[base] <= u) ? 1u : 0u);
}

// Clamped bit pattern used by the fp64 violation self-check (same clamp as the lookup).
CS_HD uint64_t clamp_bits_f64(uint64_t bits, int64_t lo, int64_t hi) {
  int64_t si = (int64_t)bits;
  si = si < lo ? lo : si;
  si = si > hi ? hi : si;
  return (uint64_t)si;
}

// Device-side view of the staged tables: pointers into one device blob.
struct DevTables {
  int32_t cap_dtype, M, U, maxB;
  int32_t n_lut;
  int32_t n_level1;
  int32_t batching_mtl, mt_bs;
  LutView lv;
  LutView lv_big;          // finer fp32 LUT for eval_kernel (n_lut_big == 0: none)
  int32_t n_lut_big, n_level1_big;
  LutView lv_huge;         // finer still (many grids: thousands of thresholds; n_lut_huge == 0: none)
  int32_t n_lut_huge, n_level1_huge;
  const uint64_t* vio;     // [U] lowest admissible cap bits per union bin (0 for bin 0)
  const uint64_t* sig;     // [M][U] segment ids of the 3 policies, 16 bits each
  const int32_t* seg_off;  // [M*3+1] offsets into seg
  const int4* seg;         // selection segments per (grid, policy): {u_lo, u_hi, grid bin, 0}
  const uint16_t* umap;    // [M][U] union bin -> grid bin
  const int32_t* sel;      // [M][3][maxB] selected entry (caller order) or -1
  const double* sthr;      // [M][3][maxB] selected throughput (0 when idle)
  const double* spw;       // [M][3][maxB] selected power (0 when idle)
  const double* idle_pw;   // [M] idle power charged to idle steps (0 when None)
  const int32_t* e_off;    // [M+1] raw entries, caller order
  const int32_t* e_mtl;
  const int32_t* e_bs;
  const double* e_thr;
  const double* e_pw;
  // sampling selector (policy.py:191-273)
  const int32_t* csort;    // [e_off[M]] per grid: caller index of the j-th entry in (power, mtl, bs) order
  const int32_t* ccnt;     // [M][maxB] combination feasible count per grid bin
  const int32_t* nbr;      // [e_off[M]][4] present neighbours (caller index, -1 pad)   policy.py:200-215
};

// Host-side staged tables (cs_tables in the C ABI).
struct Tables {
  int32_t cap_dtype = CS_CAP_F32;
  int32_t M = 0, U = 0, maxB = 0;
  int32_t batching_mtl = 1, mt_bs = 1;
  std::vector<uint64_t> thresholds;   // [U-1] union thresholds (bits)
  std::vector<int32_t> grid_bins;     // [M]
  std::vector<uint16_t> umap;         // [M][U]
  std::vector<int32_t> sel;           // [M][3][maxB]
  std::vector<int64_t> cnt;           // [M][3][maxB]
  std::vector<double> sthr, spw;      // [M][3][maxB]
  std::vector<double> idle_pw;        // [M]
  std::vector<uint64_t> sig;          // [M][U]
  std::vector<int32_t> seg_off;       // [M*3+1]
  std::vector<int32_t> seg;           // [n_seg][4] {u_lo, u_hi, grid bin, 0}: maximal union-bin
                                      // runs with one selected config (policy.py:131-134 prefix best)
  std::vector<uint64_t> vio;          // [U]
  std::vector<int32_t> e_off, e_mtl, e_bs;
  std::vector<double> e_thr, e_pw;
  std::vector<int32_t> csort, ccnt, nbr;
  // LUT
  int64_t lo = 0, hi = 0;
  uint64_t kbase = 0;
  uint32_t shift1 = 0;
  uint32_t n_level1 = 0, n_sub = 0;
  uint32_t n_unsafe = 0;  // fp32 leaves not proven violation-free (0 for well-formed tables)
  std::vector<uint32_t> lut;
  // the LUT sizes built (lut_main mirrors the fields above; lut_big is empty when no finer
  // level 1 exists, else eval_kernel's choice when shared memory allows)
  struct Lut {
    uint64_t kbase = 0;
    uint32_t shift1 = 0, n_level1 = 0, n_sub = 0, n_unsafe = 0;
    std::vector<uint32_t> lut;
  };
  Lut lut_main, lut_big, lut_huge;
  // device copies (per device ordinal)
  struct Dev {
    int device = -1;
    void* blob = nullptr;
    size_t bytes = 0;
    DevTables view{};
  };
  std::deque<Dev> devs;
};

std::string build_tables(const cs_grid_desc* grids, int32_t n_grids, int32_t cap_dtype, int32_t batching_mtl,
                         int32_t mt_bs, Tables& out);

void set_error(const std::string& msg);

}  // namespace cs
