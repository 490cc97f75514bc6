// N2 + N3 — the per-timestep policy kernel fused with its accumulation (sm_100a).
//
// Reference path: simulate() (sim.py:130-188) = PolicyIndex.select per cap (policy.py:136-148)
// then _aggregate (sim.py:104-127), for every (trace, grid, policy).
//
// eval_kernel (persistent, one CTA per SM slot):
//   * stages the threshold LUT (+ violation floors, switch signatures) into shared memory once;
//   * worker groups of `wpg` warps each own a per-trace bin histogram in shared memory and
//     stream their trace's caps from HBM with 128-bit non-allocating loads, 4 vectors in flight
//     per thread;
//   * per cap: clamp -> LUT bucket (1 LDS) -> leaf carry (rare sub-table redirect) -> union bin;
//     one shared-memory atomic adds the step to the histogram; the leaves carry a proof bit that
//     every selection they yield fits the caps they serve (StepRecord, sim.py:50-54), with an
//     exact recount if an unproven leaf is ever met;
//   * at the end of a trace the group turns the histogram into avg throughput / energy / idle /
//     switch counts for every grid x policy: per union bin (one grid, no penalty), per selection
//     segment (warp-owned (grid, policy) pairs), or per touched bin (PK, one grid with a penalty),
//     from {hi, lo}-split values whose hi sums are exact, so the result equals the reference's
//     exactly rounded math.fsum; the histogram also folds into the global bin histogram.
// finalize_kernel: the same epilogue for traces split across groups (few, long traces).
// prep_kernel: per-bin fp64 values for this launch (energy needs step_seconds, penalty needs pf).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "cs_internal.h"

#ifndef CS_PF_DIST
#define CS_PF_DIST 0  // bulk L2 prefetch distance in batches (0: off)
#endif

namespace cs {
namespace {

#define CS_CUDA_TRY(x)                                                                                  \
  do {                                                                                                  \
    cudaError_t e_ = (x);                                                                               \
    if (e_ != cudaSuccess) return std::string("CUDA error: ") + cudaGetErrorString(e_) + " (" #x ")"; \
  } while (0)

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ double4 ldg4(const double4* p) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

// ---- double-double accumulation (error-free transforms; the build uses -fmad=false) ----
struct dd {
  double hi, lo;
};
__device__ __forceinline__ void dd_add2(dd& x, double p, double pe) {
  const double s = __dadd_rn(x.hi, p);
  const double bb = __dsub_rn(s, x.hi);
  double e = __dadd_rn(__dsub_rn(x.hi, __dsub_rn(s, bb)), __dsub_rn(p, bb));
  e = __dadd_rn(e, __dadd_rn(x.lo, pe));
  const double h = __dadd_rn(s, e);
  x.lo = __dsub_rn(e, __dsub_rn(h, s));
  x.hi = h;
}
__device__ __forceinline__ void dd_add_prod(dd& x, double c, double v) {
  const double p = __dmul_rn(c, v);
  dd_add2(x, p, __fma_rn(c, v, -p));
}

}  // namespace

struct EvalParams {
  DevTables tb;
  LutView lv;  // the LUT this launch stages (tb.lv or, when it fits, the finer tb.lv_big)
  int32_t n_lut, n_level1;
  const void* caps;
  int64_t T, S, ld;
  int64_t seg_len;
  int32_t nseg;
  int32_t step_seconds;
  uint16_t* step_bins;
  int64_t ld_bins;
  cs_agg* agg;
  unsigned long long* hist;
  uint32_t* part_hist;  // split mode: [T][U]
  uint32_t* part_sw;    // [T][NSEG] switched steps per selection segment (PEN)
  uint32_t* part_vio;   // [T][M*3]
  // per selection segment of this launch (prep_kernel), structure of arrays:
  //   seg_hdr[k]  = u_lo | u_hi << 16 (union-bin range of segment k)
  //   seg_idle[mp] = 1 when (grid, policy) mp's first segment is the idle selection
  //   seg_val as double2 {hi, lo} pairs [j * NSEG + k], j = thr, energy, penalised thr: each value
  //   split so that count x hi accumulates EXACTLY (see prep_kernel)
  // staged into shared memory at off_seg when it fits (seg_smem_bytes > 0)
  const uint32_t* seg_hdr;
  const int32_t* seg_idle;
  const double* seg_val;
  // compact form for the epilogue that reads them from global memory: per segment the unsplit
  // {thr (0 when idle), energy} pair; per (grid, policy) {Q_thr, 1/Q_thr, Q_energy, 1/Q_energy}
  // (the split is recomputed with the same formula: split_q)
  const double2* seg_raw;
  const double* seg_q;
  int32_t off_seg, seg_smem_bytes;
  // bin epilogue (one grid, no penalty): per union bin u and policy p the {hi, lo} pairs of the
  // step's throughput and energy, bin_val[(2p + j) * U4 + u] (j = 0 thr, 1 energy), staged at
  // off_seg; bins u < fidle[p] are idle for policy p
  const double2* bin_val;
  int32_t bin_epi;
  int32_t fin_split;  // finalize_kernel: per-grid CTAs on shared-memory histogram copies
  int32_t fidle[3];
  int32_t U4;    // histogram row stride (U rounded up to a multiple of 4)
  int32_t NSEG;  // selection segments over all grids x policies
  double omp;
  int32_t wpg, gpc;
  // fp32 LUT constants of the redirect step derived on the host (kernel-parameter operands,
  // never rematerialised in the loop): the shift one level down (s1 - 4)
  uint32_t lut_s2;
  // fp32 bits of the lowest union threshold: caps below it are union bin 0 (idle everywhere)
  int32_t t0_bits;
  // shared-memory layout (bytes)
  int32_t off_vio, off_sig, off_ghist, off_groups, group_bytes, off_g_sw, off_g_vio, off_g_scr;
  int32_t off_pkq, off_g_edge;  // PK: the 3 policies' quanta (CTA), block edges (per group)
  int32_t gh_direct;  // long traces: fold each trace's histogram straight into hist (no CTA copy)
  int32_t hist_store;  // one-CTA launches: the CTA histogram is stored into hist (no memset before the launch)
  unsigned long long* work;  // {items handed out after the first n_groups, groups done} (dynamic scheduling)
  int32_t off_g_ring;  // CS_TMA variant: per-warp bulk-copy rings (per group)
};

namespace {

__device__ __forceinline__ void group_sync(int gid_local, int gsize) {
  if (gsize == 32)
    __syncwarp();
  else
    asm volatile("bar.sync %0, %1;" ::"r"(1 + gid_local), "r"(gsize) : "memory");
}

#ifdef CS_TMA
// ---- TMA-unit bulk copies (A/B variant CS_TMA=<stages>): cp.async.bulk global -> shared with an
// mbarrier per stage, one 512-B pass (32 vectors) per copy ----
constexpr int kTmaStages = CS_TMA;
constexpr int kTmaStageBytes = 512;
constexpr int kTmaWarpBytes = kTmaStages * (kTmaStageBytes + 8);
__device__ __forceinline__ void mbar_init(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "n"(kTmaStageBytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "n"(kTmaStageBytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
#endif

// Stage n 32-bit words from global into shared memory (both 16-B aligned) with 128-bit loads, four
// in flight per thread: a word per thread per round left small launches waiting on a dozen
// serial L2 round trips for the LUT alone.
__device__ __forceinline__ void stage_words(uint32_t* dst, const uint32_t* src, int n) {
  const int n4 = n >> 2, T = (int)blockDim.x;
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  int i = threadIdx.x;
  for (; i + 3 * T < n4; i += 4 * T) {
    const uint4 a = __ldg(s4 + i), b = __ldg(s4 + i + T), c = __ldg(s4 + i + 2 * T), d = __ldg(s4 + i + 3 * T);
    d4[i] = a, d4[i + T] = b, d4[i + 2 * T] = c, d4[i + 3 * T] = d;
  }
  for (; i < n4; i += T) d4[i] = __ldg(s4 + i);
  for (int j = 4 * n4 + threadIdx.x; j < n; j += T) dst[j] = __ldg(src + j);
}

// shared-memory counter += 1 (shared-window address)
__device__ __forceinline__ void red_inc(uint32_t saddr) {
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(saddr) : "memory");
}

// Switched-step counting for one step of one grid, branch-free: sc / sprev are the step's and the
// previous step's signatures (three 16-bit selection-segment ids); each policy whose segment
// changed counts one step for its new segment (counters at sw_s + 4 * (o_p + id)), the others
// count into the lane's own dummy slot, which is never read. (Branches around each atomic cost
// more than the extra conflict-free atomics: C5 5.02 -> 4.17 ms.)
__device__ __forceinline__ void count_switches(uint64_t sc, uint64_t sprev, int o0, int o1, int o2, uint32_t sw_s,
                                               uint32_t dummy) {
  const uint32_t lo = (uint32_t)sc, hi = (uint32_t)(sc >> 32);
  const uint32_t xl = lo ^ (uint32_t)sprev, xh = hi ^ (uint32_t)(sprev >> 32);
  red_inc((xl & 0xFFFFu) ? sw_s + 4u * (o0 + (lo & 0xFFFFu)) : dummy);
  red_inc((xl >> 16) ? sw_s + 4u * (o1 + (lo >> 16)) : dummy);
  red_inc((xh & 0xFFFFu) ? sw_s + 4u * (o2 + (hi & 0xFFFFu)) : dummy);
}

// prep: per selection segment, the fp64 values of this launch computed exactly like the
// reference per step (sim.py:111, 119-122): thr, thr * (1 - pf), (power or idle) * step / 3600.
// Each value v is split as v = hi + lo with hi = floor(v / Q) * Q, Q = 2^(E+1-L) (E: exponent of
// the (grid, policy) table's largest value, L = 53 - bits(S)): for any count c <= S, c * hi and
// the running sum of such products over a trace are EXACT (integers times Q below 2^53 Q); the
// small lo parts are summed in plain fp64 (error ~2^-(53+L) of the total), so the final
// hi + lo rounds to the exactly rounded sum the reference's math.fsum returns.
// Segment tables (structure of arrays, one block per (grid, policy)): seg_hdr[k] = u_lo | u_hi << 16,
// {hi, lo} pairs seg_val2[j * NSEG + k] for j = thr, energy, penalised thr, and seg_idle[mp].
__device__ __forceinline__ double2 split_q(double v, double q, double qi) {
  const double hi = __dmul_rn(floor(__dmul_rn(v, qi)), q);  // floor(v / Q) * Q, exact (powers of two)
  return make_double2(hi, __dsub_rn(v, hi));
}
__device__ __forceinline__ double quantum(int eq) { return ldexp(1.0, max(-1000, min(1000, eq))); }

__global__ void prep_kernel(const DevTables tb, double step, double omp, int L, int nseg, uint32_t* hdr,
                            int32_t* idlef, double* val, double2* binval, int U4, double2* raw,
                            double* qtab, unsigned long long* work) {  // L: see split_q
  __shared__ double red[2][256];
  if (blockIdx.x == 0 && threadIdx.x == 0) work[0] = work[1] = 0ull;  // eval_kernel's item counters
  const int mp = blockIdx.x, m = mp / 3, B = tb.maxB;
  const size_t ob = (size_t)mp * B;
  const double idle_e = __ddiv_rn(__dmul_rn(tb.idle_pw[m], step), 3600.0);
  double mt = 0.0, me = 0.0;
  for (int r = threadIdx.x; r < B; r += blockDim.x) {
    const bool idle = tb.sel[ob + r] < 0;
    mt = fmax(mt, idle ? 0.0 : tb.sthr[ob + r]);
    me = fmax(me, idle ? idle_e : __ddiv_rn(__dmul_rn(tb.spw[ob + r], step), 3600.0));
  }
  red[0][threadIdx.x] = mt;
  red[1][threadIdx.x] = me;
  __syncthreads();
  for (int k = blockDim.x / 2; k > 0; k >>= 1) {
    if (threadIdx.x < k) {
      red[0][threadIdx.x] = fmax(red[0][threadIdx.x], red[0][threadIdx.x + k]);
      red[1][threadIdx.x] = fmax(red[1][threadIdx.x], red[1][threadIdx.x + k]);
    }
    __syncthreads();
  }
  int et = 0, ee = 0;
  frexp(red[0][0] > 0.0 ? red[0][0] : 1.0, &et);  // max < 2^et
  frexp(red[1][0] > 0.0 ? red[1][0] : 1.0, &ee);
  et -= L;
  ee -= L;
  const double qt = quantum(et), qit = quantum(-et), qe = quantum(ee), qie = quantum(-ee);
  if (threadIdx.x == 0) qtab[4 * mp] = qt, qtab[4 * mp + 1] = qit, qtab[4 * mp + 2] = qe, qtab[4 * mp + 3] = qie;
  if (binval) {  // bin epilogue tables (M == 1: union bins are the grid's bins)
    const int p = mp % 3;
    for (int r = threadIdx.x; r < B; r += blockDim.x) {
      const bool idle = tb.sel[ob + r] < 0;
      binval[(size_t)(2 * p) * U4 + r] = split_q(idle ? 0.0 : tb.sthr[ob + r], qt, qit);
      binval[(size_t)(2 * p + 1) * U4 + r] =
          split_q(idle ? idle_e : __ddiv_rn(__dmul_rn(tb.spw[ob + r], step), 3600.0), qe, qie);
    }
  }
  const int k0 = tb.seg_off[mp], k1 = tb.seg_off[mp + 1];
  if (threadIdx.x == 0) idlef[mp] = (k1 > k0 && tb.sel[ob + tb.seg[k0].z] < 0) ? 1 : 0;
  for (int k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
    const int4 sg = tb.seg[k];
    const size_t i = ob + sg.z;
    const bool idle = tb.sel[i] < 0;  // only ever the first segment (feasibility is monotone in the cap)
    hdr[k] = (uint32_t)sg.x | ((uint32_t)sg.y << 16);
    const double thr = idle ? 0.0 : tb.sthr[i];
    const double en = idle ? idle_e : __ddiv_rn(__dmul_rn(tb.spw[i], step), 3600.0);
    raw[k] = make_double2(thr, en);
    const double2 t = split_q(thr, qt, qit);
    const double2 e = split_q(en, qe, qie);
    const double2 q = split_q(__dmul_rn(thr, omp), qt, qit);  // idle: 0 * omp = 0
    double2* v2 = reinterpret_cast<double2*>(val);
    v2[0 * (size_t)nseg + k] = t;
    v2[1 * (size_t)nseg + k] = e;
    v2[2 * (size_t)nseg + k] = q;
  }
}

// In-place inclusive prefix sum of a[0..U4) by one worker group, 4 bins per lane (LDS.128):
// each warp scans a contiguous range, then adds the totals of the ranges before it. Raw counts
// are folded into ghist on the way (the global config histogram).
template <typename GH>
__device__ __forceinline__ void group_scan(uint32_t* a, int U4, GH* ghist, uint32_t* wtot, int gtid, int gsize,
                                           int gid_local) {
  const int lane = gtid & 31, w = gtid >> 5, nw = gsize >> 5;
  const int per = ((U4 + nw - 1) / nw + 127) & ~127;
  const int lo = min(U4, w * per), hi = min(U4, lo + per);
  uint32_t carry = 0;
  for (int base = lo; base < hi; base += 128) {
    const int u = base + 4 * lane;
    uint4 x = make_uint4(0u, 0u, 0u, 0u);
    if (u < hi) x = *reinterpret_cast<const uint4*>(a + u);
    if (ghist) {
      if (x.x) atomicAdd(&ghist[u], (GH)x.x);
      if (x.y) atomicAdd(&ghist[u + 1], (GH)x.y);
      if (x.z) atomicAdd(&ghist[u + 2], (GH)x.z);
      if (x.w) atomicAdd(&ghist[u + 3], (GH)x.w);
    }
    x.y += x.x;
    x.z += x.y;
    x.w += x.z;
    uint32_t sum = x.w;
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, sum, k);
      if (lane >= k) sum += y;
    }
    const uint32_t excl = sum - x.w + carry;
    x.x += excl, x.y += excl, x.z += excl, x.w += excl;
    if (u < hi) *reinterpret_cast<uint4*>(a + u) = x;
    carry += __shfl_sync(0xffffffffu, sum, 31);
  }
  if (nw > 1) {
    if (lane == 0) wtot[w] = carry;
    group_sync(gid_local, gsize);
    uint32_t off = 0;
    for (int i = 0; i < w; ++i) off += wtot[i];
    if (off)
      for (int u = lo + lane; u < hi; u += 32) a[u] += off;
    group_sync(gid_local, gsize);
  }
}

// Transposed butterfly reduction of 4 per-lane doubles across a warp (reduce-scatter):
// 2+1+1+1+1 = 6 exchanges instead of 4 x 5. Afterwards lane kLaneOf4[j] holds the warp total
// of value j.
__constant__ int kLaneOf4[4] = {0, 8, 16, 24};

__device__ __forceinline__ double xreduce4(const double (&v)[4], int lane) {
  const unsigned FULL = 0xffffffffu;
  const bool b4 = lane & 16, b3 = lane & 8;
  double a[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double keep = b4 ? v[2 + i] : v[i], send = b4 ? v[i] : v[2 + i];
    a[i] = __dadd_rn(keep, __shfl_xor_sync(FULL, send, 16));
  }
  const double keep = b3 ? a[1] : a[0], send = b3 ? a[0] : a[1];
  double c = __dadd_rn(keep, __shfl_xor_sync(FULL, send, 8));
  c = __dadd_rn(c, __shfl_xor_sync(FULL, c, 4));
  c = __dadd_rn(c, __shfl_xor_sync(FULL, c, 2));
  return __dadd_rn(c, __shfl_xor_sync(FULL, c, 1));
}

// Combine a group's per-warp sums (wpg > 1) and write grid m's three cs_agg records of trace t:
// lane kLaneOf4[c] of warp 0 holds component c (thr hi, lo, energy hi, lo) of mine[p];
// ired = idle steps (3) and switched steps (3).
__device__ __forceinline__ void store_aggs(const EvalParams& P, int64_t t, int m, double (&mine)[3],
                                           uint32_t (&ired)[6], const uint32_t* vcnt, double* scratch, int lane,
                                           int wig, int nw, int gid_local, int gsize) {
  const int M = P.tb.M;
  if (nw > 1) {  // combine the warps of the group through shared scratch (18 + 6 words / warp)
    double* d = scratch + wig * 24;
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (lane == kLaneOf4[c]) d[4 * p + c] = mine[p];
    if (lane == 0)
      for (int j = 0; j < 6; ++j) d[12 + j] = __longlong_as_double((long long)ired[j]);
    group_sync(gid_local, gsize);
    if (wig == 0) {
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (lane == kLaneOf4[c])
            for (int w = 1; w < nw; ++w) mine[p] = __dadd_rn(mine[p], scratch[w * 24 + 4 * p + c]);
      for (int w = 1; w < nw; ++w)
        for (int j = 0; j < 6; ++j) ired[j] += (uint32_t)__double_as_longlong(scratch[w * 24 + 12 + j]);
    }
    group_sync(gid_local, gsize);
  }
  if (wig == 0) {
    // lane q (< 3) gathers policy q's six sums and writes its aggregate
    double part[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double x0 = __shfl_sync(0xffffffffu, mine[0], kLaneOf4[c]);
      const double x1 = __shfl_sync(0xffffffffu, mine[1], kLaneOf4[c]);
      const double x2 = __shfl_sync(0xffffffffu, mine[2], kLaneOf4[c]);
      part[c] = lane == 0 ? x0 : (lane == 1 ? x1 : x2);
    }
    if (lane < 3 && P.agg) {
      dd tsum{part[0], 0.0}, esum{part[2], 0.0};
      dd_add2(tsum, part[1], 0.0);
      dd_add2(esum, part[3], 0.0);
      const uint32_t id = lane == 0 ? ired[0] : (lane == 1 ? ired[1] : ired[2]);
      const uint32_t sc = lane == 0 ? ired[3] : (lane == 1 ? ired[4] : ired[5]);
      cs_agg a;
      a.avg_throughput_ips = __ddiv_rn(__dadd_rn(tsum.hi, tsum.lo), (double)P.S);  // fsum(ips)/n
      a.energy_proxy_wh = __dadd_rn(esum.hi, esum.lo);
      a.idle_steps = id;
      a.switches = sc;
      a.violations = vcnt ? vcnt[3 * m + lane] : 0;
      a.num_steps = P.S;
      P.agg[t * M * 3 + 3 * m + lane] = a;
    }
  }
}

// Per-trace epilogue: every (grid, policy) aggregate of _aggregate (sim.py:104-127) from the
// group's prefix-summed histogram. Union bins with the same selected config form a segment
// (staged in tb.seg); a segment's step count is C[hi] - C[lo-1]. Threads stride over a
// policy's segments accumulating count x {hi, mid, lo} per value (hi and mid sums are exact),
// then one transposed warp reduction per policy; lanes 0..2 finalize one policy each.
//   C[u]                prefix-summed step counts (scanned in place)
//   SW[(m*3+p)*U4 + u]  prefix-summed switched-step counts (PEN)
template <bool PEN, bool COMPACT>
__device__ __forceinline__ void epilogue(const EvalParams& P, int64_t t, const uint32_t* C, const uint32_t* SW,
                                         const uint32_t* vcnt, const uint32_t* shdr, const int32_t* sidle,
                                         const double2* sval, double* scratch, int gtid, int gsize, int gid_local,
                                         int m_begin = 0, int m_end = -1) {
  const DevTables& tb = P.tb;
  const int M = tb.M, NS = P.NSEG;
  const int lane = gtid & 31, wig = gtid >> 5, nw = gsize >> 5;
  if (m_end < 0) m_end = M;
  for (int m = m_begin; m < m_end; ++m) {
    double mine[3];
    uint32_t ired[6];
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      const int mp = 3 * m + p;
      const int k0 = __ldg(tb.seg_off + mp), k1 = __ldg(tb.seg_off + mp + 1);
      const uint32_t* sw = PEN ? SW + k0 : nullptr;  // switched steps per segment of (m, p)
      const int kidle = sidle[mp] ? k0 : -1;         // the idle selection is always the first segment
      double a[4] = {0.0, 0.0, 0.0, 0.0};  // thr hi, lo, energy hi, lo
      uint32_t idle = 0, swc = 0;
      double qt = 0.0, qit = 0.0, qe = 0.0, qie = 0.0;
      if (COMPACT) qt = __ldg(P.seg_q + 4 * mp), qit = __ldg(P.seg_q + 4 * mp + 1), qe = __ldg(P.seg_q + 4 * mp + 2),
                   qie = __ldg(P.seg_q + 4 * mp + 3);
      auto seg = [&](int k) {
        const uint32_t hd = shdr[k];
        const uint32_t ulo = hd & 0xFFFFu, uhi = hd >> 16;
        const uint32_t cnt = C[uhi] - (ulo ? C[ulo - 1] : 0u);
        if (cnt == 0) return;
        const double dc = (double)cnt;
        double2 r = make_double2(0.0, 0.0);
        if (COMPACT) r = __ldg(P.seg_raw + k);  // 16 B instead of 48 B of pre-split values
        const double2 ve = COMPACT ? split_q(r.y, qe, qie) : sval[NS + k];
        a[2] = __fma_rn(dc, ve.x, a[2]);
        a[3] = __fma_rn(dc, ve.y, a[3]);
        uint32_t scnt = 0;
        if (PEN) {
          scnt = sw[k - k0];
          swc += scnt;
        }
        if (k == kidle) {
          idle += cnt;  // idle segments carry zero throughput
        } else {
          const double dn = (double)(cnt - scnt);
          const double2 vt = COMPACT ? split_q(r.x, qt, qit) : sval[k];
          a[0] = __fma_rn(dn, vt.x, a[0]);
          a[1] = __fma_rn(dn, vt.y, a[1]);
          if (PEN && scnt) {
            const double ds = (double)scnt;
            const double2 vp = COMPACT ? split_q(__dmul_rn(r.x, P.omp), qt, qit) : sval[2 * NS + k];
            a[0] = __fma_rn(ds, vp.x, a[0]);
            a[1] = __fma_rn(ds, vp.y, a[1]);
          }
        }
      };
      // two segments per iteration so their dependent load chains (header -> prefix counts ->
      // values) overlap; same accumulation order as one at a time
      int k = k0 + gtid;
      for (; k + gsize < k1; k += 2 * gsize) {
        seg(k);
        seg(k + gsize);
      }
      if (k < k1) seg(k);
      mine[p] = xreduce4(a, lane);
      ired[p] = __reduce_add_sync(0xffffffffu, idle);
      ired[3 + p] = PEN ? __reduce_add_sync(0xffffffffu, swc) : 0u;
    }
    store_aggs(P, t, m, mine, ired, vcnt, scratch, lane, wig, nw, gid_local, gsize);
  }
}

// Warp-owned variant of epilogue() for the main kernel: each (grid, policy) pair belongs to one
// warp of the group, whose lanes stride over the pair's selection segments and whose lane 0
// writes the record — no cross-warp combine, so no barriers between the pairs (the per-pair
// combine through shared scratch cost two group barriers per grid: ~13 % of C3's warp time was
// spent waiting at them). Same per-segment arithmetic as epilogue().
template <bool PEN, bool COMPACT>
__device__ __forceinline__ void epilogue_warps(const EvalParams& P, int64_t t, const uint32_t* C, const uint32_t* SW,
                                               const uint32_t* vcnt, const uint32_t* shdr, const int32_t* sidle,
                                               const double2* sval, int gtid, int gsize) {
  const DevTables& tb = P.tb;
  const int M = tb.M, NS = P.NSEG;
  const int lane = gtid & 31, wig = gtid >> 5, nw = gsize >> 5;
  const unsigned FULL = 0xffffffffu;
  for (int mp = wig; mp < 3 * M; mp += nw) {
    const int m = mp / 3;
    const int k0 = __ldg(tb.seg_off + mp), k1 = __ldg(tb.seg_off + mp + 1);
    const uint32_t* sw = PEN ? SW + k0 : nullptr;
    const int kidle = sidle[mp] ? k0 : -1;
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    uint32_t idle = 0, swc = 0;
    double qt = 0.0, qit = 0.0, qe = 0.0, qie = 0.0;
    if (COMPACT) qt = __ldg(P.seg_q + 4 * mp), qit = __ldg(P.seg_q + 4 * mp + 1), qe = __ldg(P.seg_q + 4 * mp + 2),
                 qie = __ldg(P.seg_q + 4 * mp + 3);
    auto seg = [&](int k) {
      const uint32_t hd = shdr[k];
      const uint32_t ulo = hd & 0xFFFFu, uhi = hd >> 16;
      const uint32_t cnt = C[uhi] - (ulo ? C[ulo - 1] : 0u);
      if (cnt == 0) return;
      const double dc = (double)cnt;
      double2 r = make_double2(0.0, 0.0);
      if (COMPACT) r = __ldg(P.seg_raw + k);
      const double2 ve = COMPACT ? split_q(r.y, qe, qie) : sval[NS + k];
      a[2] = __fma_rn(dc, ve.x, a[2]);
      a[3] = __fma_rn(dc, ve.y, a[3]);
      uint32_t scnt = 0;
      if (PEN) {
        scnt = sw[k - k0];
        swc += scnt;
      }
      if (k == kidle) {
        idle += cnt;
      } else {
        const double dn = (double)(cnt - scnt);
        const double2 vt = COMPACT ? split_q(r.x, qt, qit) : sval[k];
        a[0] = __fma_rn(dn, vt.x, a[0]);
        a[1] = __fma_rn(dn, vt.y, a[1]);
        if (PEN && scnt) {
          const double ds = (double)scnt;
          const double2 vp = COMPACT ? split_q(__dmul_rn(r.x, P.omp), qt, qit) : sval[2 * NS + k];
          a[0] = __fma_rn(ds, vp.x, a[0]);
          a[1] = __fma_rn(ds, vp.y, a[1]);
        }
      }
    };
    int k = k0 + lane;
    for (; k + 32 < k1; k += 64) {  // two segments per iteration: their load chains overlap
      seg(k);
      seg(k + 32);
    }
    if (k < k1) seg(k);
    const double mine = xreduce4(a, lane);  // lane kLaneOf4[c] holds component c
    const uint32_t id = __reduce_add_sync(FULL, idle), sc = __reduce_add_sync(FULL, swc);
    const double c0 = __shfl_sync(FULL, mine, kLaneOf4[0]), c1 = __shfl_sync(FULL, mine, kLaneOf4[1]),
                 c2 = __shfl_sync(FULL, mine, kLaneOf4[2]), c3 = __shfl_sync(FULL, mine, kLaneOf4[3]);
    if (lane == 0 && P.agg) {
      dd tsum{c0, 0.0}, esum{c2, 0.0};
      dd_add2(tsum, c1, 0.0);
      dd_add2(esum, c3, 0.0);
      cs_agg r;
      r.avg_throughput_ips = __ddiv_rn(__dadd_rn(tsum.hi, tsum.lo), (double)P.S);  // fsum(ips)/n
      r.energy_proxy_wh = __dadd_rn(esum.hi, esum.lo);
      r.idle_steps = id;
      r.switches = PEN ? sc : 0u;
      r.violations = vcnt ? vcnt[mp] : 0u;
      r.num_steps = P.S;
      P.agg[t * M * 3 + mp] = r;
    }
  }
}

// Bin epilogue (one grid, no switch penalty): every bin carries its three policies' values, so
// the trace's sums are sum_u h[u] x v_p(u) straight from the histogram — no prefix scan, no
// segment ranges — and the same pass folds h into the CTA histogram and re-zeroes it.
template <typename GH>
__device__ __forceinline__ void finish_trace_bins(const EvalParams& P, int64_t t, uint32_t* h, const uint32_t* vcnt,
                                                  GH* ghist, const double2* bv, double* scratch, int gtid, int gsize,
                                                  int gid_local) {
  const int U = P.tb.U, U4 = P.U4;
  const int lane = gtid & 31, wig = gtid >> 5, nw = gsize >> 5;
  double a[3][4];
  uint32_t idl[3] = {0u, 0u, 0u};
#pragma unroll
  for (int p = 0; p < 3; ++p) a[p][0] = a[p][1] = a[p][2] = a[p][3] = 0.0;
  for (int u = gtid; u < U; u += gsize) {
    const uint32_t c = h[u];
    if (c == 0) continue;
    h[u] = 0u;
    if (ghist) atomicAdd(&ghist[u], (GH)c);
    const double dc = (double)c;
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      const double2 vt = bv[(size_t)(2 * p) * U4 + u];
      const double2 ve = bv[(size_t)(2 * p + 1) * U4 + u];
      a[p][0] = __fma_rn(dc, vt.x, a[p][0]);
      a[p][1] = __fma_rn(dc, vt.y, a[p][1]);
      a[p][2] = __fma_rn(dc, ve.x, a[p][2]);
      a[p][3] = __fma_rn(dc, ve.y, a[p][3]);
      idl[p] += u < P.fidle[p] ? c : 0u;
    }
  }
  double mine[3];
  uint32_t ired[6];
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    mine[p] = xreduce4(a[p], lane);
    ired[p] = __reduce_add_sync(0xffffffffu, idl[p]);
    ired[3 + p] = 0u;
  }
  store_aggs(P, t, 0, mine, ired, vcnt, scratch, lane, wig, nw, gid_local, gsize);
}

// Scan + epilogue over a group histogram (smem in the main kernel, global in finalize); the
// histogram (and switch histograms) are left zeroed for the next trace.
template <bool PEN, bool COMPACT, typename GH>
__device__ __forceinline__ void finish_trace(const EvalParams& P, int64_t t, uint32_t* h, uint32_t* sw,
                                             const uint32_t* vcnt, GH* ghist, const uint32_t* shdr,
                                             const int32_t* sidle, const double2* sval, double* scratch, int gtid,
                                             int gsize, int gid_local) {
  const int U4 = P.U4, M = P.tb.M;
  uint32_t* wtot = reinterpret_cast<uint32_t*>(scratch);  // reused: scan totals, then partial sums
  group_scan(h, U4, ghist, wtot, gtid, gsize, gid_local);
  group_sync(gid_local, gsize);
  // warp-owned pairs when there are at least as many (grid, policy) pairs as warps (C3: 30 over
  // 8); otherwise (a whole-CTA group on one grid: C1) every pair is summed by all the group's
  // threads — one segment each instead of a warp walking hundreds in turn (C1 18.0 -> 16.9 us)
  if (3 * M >= (gsize >> 5))
    epilogue_warps<PEN, COMPACT>(P, t, h, sw, vcnt, shdr, sidle, sval, gtid, gsize);
  else
    epilogue<PEN, COMPACT>(P, t, h, sw, vcnt, shdr, sidle, sval, scratch, gtid, gsize, gid_local);
  group_sync(gid_local, gsize);
  for (int u = 4 * gtid; u < U4; u += 4 * gsize) *reinterpret_cast<uint4*>(h + u) = make_uint4(0u, 0u, 0u, 0u);
  if (PEN)
    for (int i = gtid; i < P.NSEG; i += gsize) sw[i] = 0u;
}

// Exact violation recount of a segment (slow path; only runs if the fast check fired).
template <typename CapT>
__device__ void recount_violations(const EvalParams& P, const uint32_t* s_lut, const CapT* row, int64_t s0,
                                   int64_t s1e, uint32_t* vcnt, int gtid, int gsize) {
  const DevTables& tb = P.tb;
  for (int64_t i = s0 + gtid; i < s1e; i += gsize) {
    uint32_t b;
    double cap;
    if constexpr (sizeof(CapT) == 4) {
      const uint32_t x = __ldg(reinterpret_cast<const uint32_t*>(row) + i);
      b = bin_f32(x, P.lv.shift1, (int32_t)P.lv.kbase, P.n_level1, P.lv.sub0, s_lut);
      cap = (double)__uint_as_float(x);
    } else {
      const unsigned long long x = __ldg(reinterpret_cast<const unsigned long long*>(row) + i);
      b = bin_f64(x, P.lv.lo, P.lv.hi, P.lv.shift1, P.lv.kbase, P.lv.sub0, s_lut, P.lv.thr64);
      cap = __longlong_as_double((long long)x);
    }
    for (int m = 0; m < tb.M; ++m) {
      const int r = (tb.M > 1) ? (int)tb.umap[(size_t)m * tb.U + b] : (int)b;
      for (int p = 0; p < 3; ++p) {
        const size_t o = ((size_t)m * 3 + p) * tb.maxB + r;
        if (tb.sel[o] >= 0 && tb.spw[o] > cap) atomicAdd(&vcnt[m * 3 + p], 1u);
      }
    }
  }
}

// fp32 LUT search with its constants held in registers (encoding: cs_internal.h).
struct Lut32 {
  const uint32_t* lut;   // shared
  uint32_t lutk;         // shared-window address of lut[-KBASE]: the bucket load is one SHF + LEA
                         // (through inline PTX, or the compiler re-derives lut + (k - KBASE))
  int32_t lo, hi, kb;    // clamp range of the cap bits (guard buckets included), level-1 offset
  uint32_t s1, s2, sub0;  // level-1 shift, the shift one level down (s1 - 4), first sub-table entry
  uint32_t lutb, s2m2;    // shared-window address of lut[0]; s2 - 2 (staging keeps s1 >= 6)

  // the clamp keeps every cap inside its bucket (buckets 0 and NB-1 are empty guards: -0.0 /
  // negatives land in bin 0, caps above every threshold and NaN in the top bin), so a leaf needs
  // no mask of the cap's low bits
  __device__ __forceinline__ uint32_t clampx(uint32_t x) const { return (uint32_t)min(max((int32_t)x, lo), hi); }
  __device__ __forceinline__ uint32_t entry(uint32_t xc) const {
    uint32_t e;
    asm("ld.shared.u32 %0, [%1];" : "=r"(e) : "r"(lutk + ((uint32_t)((int32_t)xc >> s1) << 2)));
    return e;
  }
  __device__ __forceinline__ static uint32_t leaf(uint32_t e, uint32_t xc) {
    // e + (cap << 2) carries into bit 16 iff the bucket's threshold <= cap (one LEA); the high
    // half is taken with PRMT so the histogram address becomes one more LEA (bin * 4 + base)
    return __byte_perm(e + (xc << 2), 0u, 0x4432);
  }
  // redirect entries hold their sub-table's byte offset (<< 7): any level, shift s
  __device__ __forceinline__ uint32_t sub(uint32_t e, uint32_t xc, uint32_t s) const {
    return lut[(e >> 9) + ((xc >> s) & 15u)];
  }
  // the first redirect level (constant shift s2): the entry's byte address from adds only
  __device__ __forceinline__ uint32_t sub_addr(uint32_t e, uint32_t xc) const {
    return lutb + (e >> 7) + ((xc >> s2m2) & 0x3Cu);
  }
  __device__ __forceinline__ static uint32_t lds(uint32_t addr) {
    uint32_t r;
    asm("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(addr));
    return r;
  }
  // resolve through redirect sub-tables; ORs the final leaf's "unproven" bit into flags
  __device__ __forceinline__ uint32_t deep(uint32_t e, uint32_t xc, uint32_t& flags) const {
    while (e & kRedirect32) e = sub(e, xc, (e >> 2) & 31u);
    flags |= e;
    return leaf(e, xc);
  }
  __device__ __forceinline__ uint32_t bin(uint32_t x, uint32_t& flags) const {
    const uint32_t xc = clampx(x);
    const uint32_t e = entry(xc);
    if (e & kRedirect32) return deep(e, xc, flags);
    flags |= e;
    return leaf(e, xc);
  }
};

constexpr uint32_t kStepZero = 0xFFFFFFFFu;  // "no previous step" (never a bin)

// The hot loop over one segment [s0, s1e) of trace t. Returns true if a cap met a LUT leaf
// that is not proven violation-free (the caller then recounts violations exactly).
template <bool PEN, bool STEP, bool VIO, bool UNI>
__device__ __forceinline__ bool run_segment_f32(const EvalParams& P, const Lut32& L, uint32_t* h, uint32_t* sw,
                                                const uint64_t* s_sig, int64_t t, int64_t s0, int64_t s1e, int gtid,
                                                int gsize, uint32_t& tma_seq) {
  const int U = P.tb.U, M = P.tb.M;
  const uint32_t* row = reinterpret_cast<const uint32_t*>(P.caps) + t * P.ld;
  const unsigned char* vrow = reinterpret_cast<const unsigned char*>(row + s0);
  const int n = (int)(s1e - s0);
  const int nvf = n >> 2;
  uint32_t flags = 0;  // OR of the leaf entries used: bit 0 = leaf not proven violation-free
  const uint32_t sw_s = PEN ? (uint32_t)__cvta_generic_to_shared(sw) : 0u;
  const uint32_t sw_dummy = sw_s + 4u * (uint32_t)(P.NSEG + (gtid & 31));  // 32 slots after the counters
  auto switches = [&](uint32_t cb, uint32_t pb) {
    if (cb != pb)
      for (int m = 0; m < M; ++m)
        count_switches(s_sig[(size_t)m * U + cb], s_sig[(size_t)m * U + pb], 0, 0, 0, sw_s, sw_dummy);
  };
  // union bins of one 16-B vector (4 caps) into b[] (LUT search only)
  auto lut4 = [&](const uint4 raw, uint32_t (&b)[4]) {
    const uint32_t u[4] = {L.clampx(raw.x), L.clampx(raw.y), L.clampx(raw.z), L.clampx(raw.w)};
    uint32_t e[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
#ifdef CS_DIAG_NO_LUT  // diagnostic build only: replaces the LUT load by arithmetic (wrong bins)
      e[k] = (((u[k] >> L.s1) & 511u) << 16);
#else
      e[k] = L.entry(u[k]);
#endif
    }
    const uint32_t any = e[0] | e[1] | e[2] | e[3];
    // UNI (A/B build CS_UNI): a warp with any redirecting lane runs only the redirect path
    // (correct for plain leaves too) instead of the per-lane branch; it won on C3 while the
    // per-lane sub-table step compiled to divergent branches, and lost once that step became a
    // predicated load (__activemask: the main loops' last iteration can be divergent)
    const bool plain = UNI ? !__any_sync(__activemask(), (any & kRedirect32) != 0u) : (any & kRedirect32) == 0u;
    if (plain) {
      if (VIO) flags |= any;
#pragma unroll
      for (int k = 0; k < 4; ++k) b[k] = Lut32::leaf(e[k], u[k]);
    } else {
      // one sub-table step per element — a level-1 redirect always splits its bucket at shift
      // s1 - 4 (staging.cpp: LutBuilder::make), so the shift is a constant — then the general
      // loop only for chains (rare)
      if (UNI) {  // branch-free: every element loads (non-redirects read entry 0, a broadcast;
                  // the predicated loads compiled to four divergent branches: C3 +2.4 %, iid +5.7 %)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const bool r = (e[k] & kRedirect32) != 0u;
          const uint32_t e2 = Lut32::lds(r ? L.sub_addr(e[k], u[k]) : L.lutb);
          e[k] = r ? e2 : e[k];
        }
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (e[k] & kRedirect32) e[k] = Lut32::lds(L.sub_addr(e[k], u[k]));
      }
      if ((e[0] | e[1] | e[2] | e[3]) & kRedirect32) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          while (e[k] & kRedirect32) e[k] = L.sub(e[k], u[k], (e[k] >> 2) & 31u);
      }
      if (VIO) flags |= e[0] | e[1] | e[2] | e[3];
#pragma unroll
      for (int k = 0; k < 4; ++k) b[k] = Lut32::leaf(e[k], u[k]);
    }
  };
  // bins of one 16-B vector (4 caps) into b[], histogram atomics, per-step output
  auto bins4 = [&](const uint4 raw, int v, uint32_t (&b)[4]) {
    lut4(raw, b);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
#ifdef CS_DIAG_NO_ATOMS  // diagnostic build only: no histogram update (wrong aggregates)
      flags ^= b[k] << 1;
#else
      atomicAdd(&h[b[k]], 1u);
#endif
    }
    if (STEP) {
      uint2 o;
      o.x = (b[0] & 0xFFFFu) | (b[1] << 16);
      o.y = (b[2] & 0xFFFFu) | (b[3] << 16);
      *reinterpret_cast<uint2*>(P.step_bins + t * P.ld_bins + s0 + 4 * (int64_t)v) = o;
    }
  };
  // switched steps of one vector given pb, the bin of the cap before it (PEN)
  auto sw4 = [&](const uint32_t (&b)[4], uint32_t pb) {
    if (M == 1) {  // one signature load per step, chained through the vector
      uint64_t sg[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) sg[k] = s_sig[b[k]];
      const uint64_t sp = pb == b[0] ? sg[0] : s_sig[pb];
      auto sw1 = [&](uint64_t sc, uint64_t sprev) { count_switches(sc, sprev, 0, 0, 0, sw_s, sw_dummy); };
      sw1(sg[0], sp);
      sw1(sg[1], sg[0]);
      sw1(sg[2], sg[1]);
      sw1(sg[3], sg[2]);
    } else {
      switches(b[0], pb);
      switches(b[1], b[0]);
      switches(b[2], b[1]);
      switches(b[3], b[2]);
    }
  };

  if constexpr (PEN) {
    // Warp-contiguous chunks: each warp owns a run of vectors, lanes interleaved inside it, so the
    // cap before lane l's vector is lane l-1's last cap (a shuffle) and lane 0's is lane 31's of
    // the previous pass (carried in a register); only a warp's first vector reloads a cap.
    const int lane = gtid & 31, nwg = gsize >> 5;
    const int per = (((nvf + nwg - 1) / nwg) + 7) & ~7;  // 128-B aligned warp chunks
    const int vb = min(nvf, (gtid >> 5) * per), ve = min(nvf, vb + per);
    uint32_t carry = 0;
    if (vb < ve) {
      const int64_t i0 = s0 + 4 * (int64_t)vb;
      uint32_t dummy = 0;
      carry = i0 > 0 ? L.bin(__ldg(row + i0 - 1), dummy) : kStepZero;  // step 0 is never penalised (sim.py:119)
    }
    auto pass = [&](const uint4 raw, int v) {
      uint32_t b[4] = {0u, 0u, 0u, 0u};
      const bool act = v < ve;
      if (act) bins4(raw, v, b);
      const uint32_t left = __shfl_sync(0xffffffffu, b[3], (lane + 31) & 31);
      uint32_t pb = lane == 0 ? carry : left;
      carry = __shfl_sync(0xffffffffu, b[3], 31);
      if (pb == kStepZero) pb = b[0];
      if (act) sw4(b, pb);
    };
    // 4 loads in flight per lane, then ONE copy of the pass body: the penalty kernel's code
    // otherwise overflows the instruction cache (unrolled passes: C5 4.48 ms, rolled: 3.53 ms;
    // the eval loops without a penalty are smaller and lose 15-18 % rolled)
    int base = vb;
    for (; base + 96 < ve; base += 128) {
      const int v = base + lane;
      uint4 r0 = ldg_stream(vrow + (size_t)v * 16);
      uint4 r1 = ldg_stream(vrow + (size_t)(v + 32) * 16);
      uint4 r2 = ldg_stream(vrow + (size_t)(v + 64) * 16);
      uint4 r3 = make_uint4(0u, 0u, 0u, 0u);
      if (v + 96 < ve) r3 = ldg_stream(vrow + (size_t)(v + 96) * 16);
#pragma unroll 1
      for (int j = 0; j < 4; ++j) {
        pass(r0, v + 32 * j);
        r0 = r1, r1 = r2, r2 = r3;
      }
    }
    for (; base < ve; base += 32) {
      const int v = base + lane;
      uint4 r = make_uint4(0u, 0u, 0u, 0u);
      if (v < ve) r = ldg_stream(vrow + (size_t)v * 16);
      pass(r, v);
    }
  } else {
    auto vec4 = [&](const uint4 raw, int v) {
      uint32_t b[4];
      bins4(raw, v, b);
    };
    int v = gtid;
    // (warp-contiguous chunks per group warp, so the warps do not update the same bins at the same
    // time, measured: C3 -0.5 %, within noise; 16/32-warp groups stay 25-90 % slower either way)
#ifdef CS_TMA
    if (!STEP) {
      // each warp streams its passes (32 consecutive vectors, 512 B, every gsize vectors) through a
      // kTmaStages-deep shared-memory ring filled by the TMA unit (lane 0 issues, all lanes wait on
      // the stage's mbarrier, then read their 16 B with LDS.128)
      const int lane = gtid & 31, wig = gtid >> 5;
      unsigned char* ring = reinterpret_cast<unsigned char*>(h) + P.off_g_ring + wig * kTmaWarpBytes;
      const uint32_t rs = (uint32_t)__cvta_generic_to_shared(ring);
      const uint32_t bs = rs + kTmaStages * kTmaStageBytes;
      const int first = wig * 32;
      const int npass = nvf >= first + 32 ? (nvf - first - 32) / gsize + 1 : 0;
      // (the barriers are initialised once per kernel; tma_seq counts this warp's stage uses
      // across traces, so stage = seq % stages and the phase parity = (seq / stages) & 1)
      if (npass > 0) {
        const uint32_t q0 = tma_seq;
        if (lane == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          for (int k = 0; k < kTmaStages && k < npass; ++k) {
            const uint32_t st = (q0 + k) % kTmaStages;
            bulk_load(rs + st * kTmaStageBytes, vrow + (size_t)(first + k * gsize) * 16, bs + 8 * st);
          }
        }
        __syncwarp();
        for (int p = 0; p < npass; ++p) {
          const uint32_t q = q0 + p, st = q % kTmaStages;
          mbar_wait(bs + 8 * st, (q / kTmaStages) & 1u);
          const uint4 raw = *reinterpret_cast<const uint4*>(ring + st * kTmaStageBytes + lane * 16);
          vec4(raw, first + p * gsize + lane);
          __syncwarp();
          if (lane == 0 && p + kTmaStages < npass) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bulk_load(rs + st * kTmaStageBytes, vrow + (size_t)(first + (p + kTmaStages) * gsize) * 16, bs + 8 * st);
          }
        }
        tma_seq = q0 + npass;
      }
      v = first + npass * gsize + lane;  // the remaining (partial) pass goes through the loops below
    }
#endif
    // (tried and measured, not kept: time-clustered lanes — 32 consecutive caps per warp
    // instruction via 32-bit loads, C4 -5 % / C3 -4 %; a rolling reload pipeline, C3 +-0)
    // each lane keeps 4 independent 128-bit loads in flight per pass
    for (; v + 3 * gsize < nvf; v += 4 * gsize) {
#if CS_PF_DIST > 0
      // bulk L2 prefetch (TMA unit, no registers) of this warp's 2-KB slice of the group's batch
      // CS_PF_DIST batches ahead, so the loads below hit L2 instead of waiting on DRAM
      if ((gtid & 31) == 0) {
        const int64_t pv = (int64_t)(v - gtid) + (int64_t)CS_PF_DIST * 4 * gsize + (int64_t)(gtid >> 5) * 128;
        if (pv + 128 <= nvf)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], 2048;" ::"l"(vrow + pv * 16) : "memory");
      }
#endif
      const uint4 r0 = ldg_stream(vrow + (size_t)v * 16);
      const uint4 r1 = ldg_stream(vrow + (size_t)(v + gsize) * 16);
      const uint4 r2 = ldg_stream(vrow + (size_t)(v + 2 * gsize) * 16);
      const uint4 r3 = ldg_stream(vrow + (size_t)(v + 3 * gsize) * 16);
      vec4(r0, v);
      vec4(r1, v + gsize);
      vec4(r2, v + 2 * gsize);
      vec4(r3, v + 3 * gsize);
    }
    for (; v < nvf; v += gsize) vec4(ldg_stream(vrow + (size_t)v * 16), v);
  }
  // tail (< 4 caps at the very end of a trace)
  for (int i = 4 * nvf + gtid; i < n; i += gsize) {
    const int64_t gi = s0 + i;
    const uint32_t u = __ldg(row + gi);
    const uint32_t b = L.bin(u, flags);
    atomicAdd(&h[b], 1u);
    if (PEN) {
      uint32_t dummy = 0;
      switches(b, gi > 0 ? L.bin(__ldg(row + gi - 1), dummy) : b);
    }
    if (STEP) P.step_bins[t * P.ld_bins + gi] = (uint16_t)b;
  }
  return VIO && (flags & 1u);
}

// ---------------------------------------------------------------------------------------------
// PK: one grid, switching penalty, whole traces of < 2^16 steps (C5's shape). Per worker group:
//   h[u]  = A word: steps in union bin u | switched steps of policy 1 << 16
//   hw[u] = W word: switched steps of policy 2 | of policy 0 << 16, + 32 per-lane dummy slots
//   edges[i] = first bin | last bin << 16 of block i (kPkBlkVec vectors, dealt round-robin)
// 16-bit fields cannot carry: a trace has < 2^16 steps (the plan also counts the fill below).
// ---------------------------------------------------------------------------------------------
constexpr int kPkBlkVec = 32;  // vectors (4 caps each) per block: one 32-lane pass, grabbed dynamically

// bins of 4 caps (no redirect-uniform variant), ORing the leaves into flags
__device__ __forceinline__ void lut4_f32(const Lut32& L, const uint4 raw, uint32_t (&b)[4], uint32_t& flags) {
  const uint32_t u[4] = {L.clampx(raw.x), L.clampx(raw.y), L.clampx(raw.z), L.clampx(raw.w)};
  uint32_t e[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) e[k] = L.entry(u[k]);
  const uint32_t any = e[0] | e[1] | e[2] | e[3];
  if ((any & kRedirect32) == 0u) {
    flags |= any;
#pragma unroll
    for (int k = 0; k < 4; ++k) b[k] = Lut32::leaf(e[k], u[k]);
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (e[k] & kRedirect32) e[k] = Lut32::lds(L.sub_addr(e[k], u[k]));
    if ((e[0] | e[1] | e[2] | e[3]) & kRedirect32) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        while (e[k] & kRedirect32) e[k] = L.sub(e[k], u[k], (e[k] >> 2) & 31u);
    }
    flags |= e[0] | e[1] | e[2] | e[3];
#pragma unroll
    for (int k = 0; k < 4; ++k) b[k] = Lut32::leaf(e[k], u[k]);
  }
}

// One step of bin b whose segments are sc after sp (sim.py:119: a policy whose config changed pays
// the penalty). Three shared atomics, none predicated (ptxas turns predicated atomics into
// branches): the step count is ATOMS.POPC.INC — hardware-aggregated for equal addresses, where a
// register-operand add serialises (tools/microbench/mb_atoms.cu) — and the two switch increments
// go to the lane's own dummy slot when zero. sig = {seg2 | seg0 << 16, seg1} (absolute segment
// ids), so sc ^ sp names the policies whose config changed.
__device__ __forceinline__ void pk_count(uint32_t hA, uint32_t hW, uint32_t dummy, uint32_t b, uint2 sc, uint2 sp) {
  const uint32_t a = hA + 4u * b;
  red_inc(a);
  uint32_t inc;  // 1 in each 16-bit half whose segment id changed (VIMNMX.U16x2)
  asm("min.u16x2 %0, %1, %2;" : "=r"(inc) : "r"(sc.x ^ sp.x), "r"(0x00010001u));
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(inc ? hW + 4u * b : dummy), "r"(inc) : "memory");
  asm volatile("red.shared.add.u32 [%0], 65536;" ::"r"(sc.y != sp.y ? a : dummy) : "memory");
}

// Main loop of one whole trace (s0 = 0), in blocks of one 32-lane pass grabbed from a per-group
// counter (ctr), so the warps of a group finish the trace together whatever its day/night
// pattern (round-robin blocks left them waiting at the per-trace barrier: C5 -6 %). Inside a
// block the cap before lane l's vector is lane l-1's last (a shuffle); the block's first step
// (lane 0's first cap) is counted unswitched and its (first, last) bins go to edges[] —
// pk_finish adds the switches across block boundaries, so no block needs the bin of the cap
// before it. Each warp keeps its next block's load in flight under the current one (two unrolled
// passes, no register rotation). Vectors past the end of the trace replicate its last full
// vector's last cap (no predication in the passes; applied at use — a select right after the
// load stalls the prefetch); their steps, all in that cap's bin, are subtracted once. Returns
// true if a cap met an unproven leaf.
__device__ __forceinline__ bool pk_main(const EvalParams& P, const Lut32& L, uint32_t* h, uint32_t* hw,
                                            uint32_t* edges, const uint2* s_sig2, uint32_t* ctr, int64_t t,
                                            int gtid, int gsize) {
  const int n = (int)P.S;
  const uint32_t* row = reinterpret_cast<const uint32_t*>(P.caps) + t * P.ld;
  const uint4* vrow = reinterpret_cast<const uint4*>(row);
  const int nvf = n >> 2;
  const int lane = gtid & 31, wig = gtid >> 5, nwg = gsize >> 5;
  const int nblk = (nvf + kPkBlkVec - 1) / kPkBlkVec;
  const unsigned FULL = 0xffffffffu;
  const uint32_t hA = (uint32_t)__cvta_generic_to_shared(h), hW = (uint32_t)__cvta_generic_to_shared(hw);
  const uint32_t dummy = hW + 4u * (uint32_t)(P.U4 + lane);
  const int32_t t0 = P.t0_bits;
  uint32_t flags = 0;
  auto grab = [&]() -> int {
    uint32_t b = 0;
    if (lane == 0) b = atomicAdd(ctr, 1u);
    return (int)__shfl_sync(FULL, b, 0) + nwg;  // the first nwg blocks are taken statically
  };
  auto ldv = [&](int blk) -> uint4 { return ldg_stream(vrow + min(blk * kPkBlkVec + lane, nvf - 1)); };
  auto pass = [&](uint4 raw, int blk) {
    if (blk == nblk - 1 && blk * kPkBlkVec + lane >= nvf) raw = make_uint4(raw.w, raw.w, raw.w, raw.w);
    const bool low = (int32_t)raw.x < t0 && (int32_t)raw.y < t0 && (int32_t)raw.z < t0 && (int32_t)raw.w < t0;
    uint32_t last = 0u;
    if (__all_sync(FULL, low)) {
      if (lane == 0) {
        asm volatile("red.shared.add.u32 [%0], 128;" ::"r"(hA) : "memory");
        edges[blk] = 0u;
      }
    } else {
      uint32_t b[4];
      lut4_f32(L, raw, b, flags);
      last = __shfl_sync(FULL, b[3], 31);
      if (lane == 0) edges[blk] = b[0] | (last << 16);
      uint2 sg[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) sg[k] = s_sig2[b[k]];
      // the signature of the step before lane l's vector is lane l-1's sg[3] (that step's): two
      // shuffles instead of another LDS.64 on the L1TEX-bound loop; lane 0 (block start) counts
      // its first step unswitched
      const uint32_t px = __shfl_sync(FULL, sg[3].x, (lane + 31) & 31), py = __shfl_sync(FULL, sg[3].y, (lane + 31) & 31);
      const uint2 sp = lane == 0 ? sg[0] : make_uint2(px, py);
      pk_count(hA, hW, dummy, b[0], sg[0], sp);
      pk_count(hA, hW, dummy, b[1], sg[1], sg[0]);
      pk_count(hA, hW, dummy, b[2], sg[2], sg[1]);
      pk_count(hA, hW, dummy, b[3], sg[3], sg[2]);
    }
    const int nfill = nblk * kPkBlkVec - nvf;  // the last block's fill steps, all in bin `last`
    if (blk == nblk - 1 && lane == 0 && nfill > 0) atomicSub(&h[last], 4u * (uint32_t)nfill);
  };
  int b0 = wig;
  // (three blocks in flight — three unrolled passes or a rotated register queue — measured
  // slower: C5 2.74 / 2.55 vs 2.32 ms)
  if (b0 < nblk) {
    uint4 r0 = ldv(b0);
    int b1 = grab();
    uint4 r1 = ldv(b1);
    for (;;) {
      pass(r0, b0);
      if (b1 >= nblk) break;
      b0 = grab();
      r0 = ldv(b0);
      pass(r1, b1);
      if (b0 >= nblk) break;
      b1 = grab();
      r1 = ldv(b1);
    }
  }
  for (int i = 4 * nvf + gtid; i < n; i += gsize) {  // tail (< 4 caps at the end)
    const uint32_t b = L.bin(__ldg(row + i), flags);
    uint32_t dummyf = 0;
    const uint32_t pb = i > 0 ? L.bin(__ldg(row + i - 1), dummyf) : b;  // step 0 is never penalised
    pk_count(hA, hW, dummy, b, s_sig2[b], s_sig2[pb]);
  }
  return (flags & 1u) != 0u;
}

// PK epilogue: every aggregate of the trace from the touched bins only (a few hundred of C5's
// 2,038), each reading its three selection segments from the staged signature — no prefix scan,
// no pass over every segment. Per policy p and bin u with c steps of which s switched into u:
// thr += (c - s) x thr_k + s x thr_k (1 - pf), energy += c x energy_k, k = seg_p(u), every value
// split {hi, lo} with split_q exactly as prep_kernel does (sim.py:111, 119-122): the count x hi
// products and their sums are exact. The block-boundary steps pk_main counted unswitched enter
// as (c = 0, s = 1) corrections. Each warp compacts the nonzero bins of its 128-bin chunks into a
// LIFO queue in its scratch and processes them 32 at a time with every lane busy; the bins are
// re-zeroed on the way. Warp 0 writes the records and resets the counters: the only barrier is
// the one before warp 0 combines the warps' partial sums (the next trace's first barrier orders
// the scratch and counter reuse).
//   sraw[k] = {thr (0 when idle), energy} per selection segment; sq[4p..4p+3] = {Q_thr, 1/Q_thr,
//   Q_energy, 1/Q_energy} of policy p (shared)
constexpr int kPkScrWarp = 40;  // doubles of scratch per warp: a 160-entry u16 queue / 24 partials

template <bool STAGED, typename GH>
__device__ __forceinline__ void pk_finish(const EvalParams& P, int64_t t, uint32_t* h, uint32_t* hw,
                                          const uint32_t* edges, const uint2* s_sig2, uint32_t* vcnt, int vflag,
                                          GH* ghist, const double2* sraw, const double* sq, double* scratch, int gtid,
                                          int gsize, int gid_local) {
  const int U = P.tb.U;
  const int lane = gtid & 31, wig = gtid >> 5, nw = gsize >> 5;
  const unsigned FULL = 0xffffffffu;
  double a[3][4];
  uint32_t idl[3] = {0u, 0u, 0u}, swc[3] = {0u, 0u, 0u};
#pragma unroll
  for (int p = 0; p < 3; ++p) a[p][0] = a[p][1] = a[p][2] = a[p][3] = 0.0;
  auto acc = [&](int u, uint32_t c, const uint32_t (&ss)[3]) {
    const uint2 sg = s_sig2[u];
    const uint32_t kk[3] = {sg.x >> 16, sg.y, sg.x & 0xFFFFu};
    const double dc = (double)c;
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      const double2 r = STAGED ? sraw[kk[p]] : __ldg(sraw + kk[p]);
      const double q0 = sq[4 * p], q1 = sq[4 * p + 1];
      if (c) {
        const double2 ve = split_q(r.y, sq[4 * p + 2], sq[4 * p + 3]);
        a[p][2] = __fma_rn(dc, ve.x, a[p][2]);
        a[p][3] = __fma_rn(dc, ve.y, a[p][3]);
      }
      swc[p] += ss[p];
      if (u < P.fidle[p]) {
        idl[p] += c;  // idle selection: zero throughput, switched or not
      } else {
        const double2 vt = split_q(r.x, q0, q1);
        const double dn = (double)((int32_t)c - (int32_t)ss[p]);
        a[p][0] = __fma_rn(dn, vt.x, a[p][0]);
        a[p][1] = __fma_rn(dn, vt.y, a[p][1]);
        if (ss[p]) {
          const double ds = (double)ss[p];
          const double2 vp = split_q(__dmul_rn(r.x, P.omp), q0, q1);
          a[p][0] = __fma_rn(ds, vp.x, a[p][0]);
          a[p][1] = __fma_rn(ds, vp.y, a[p][1]);
        }
      }
    }
  };
  // (1) switches across block boundaries (a block's first step was counted unswitched)
  const int nblk = ((int)(P.S >> 2) + kPkBlkVec - 1) / kPkBlkVec;
  for (int i = gtid + 1; i < nblk; i += gsize) {
    const uint32_t b = edges[i] & 0xFFFFu, pb = edges[i - 1] >> 16;
    if (b != pb) {
      const uint2 sc = s_sig2[b], sp = s_sig2[pb];
      const uint32_t x = sc.x ^ sp.x;
      const uint32_t ss[3] = {(x >> 16) ? 1u : 0u, sc.y != sp.y ? 1u : 0u, (x & 0xFFFFu) ? 1u : 0u};
      if (ss[0] | ss[1] | ss[2]) acc((int)b, 0u, ss);
    }
  }
  // (2) the touched bins, 4 per lane per chunk, compacted through the warp's LIFO queue
  uint16_t* q = reinterpret_cast<uint16_t*>(scratch + wig * kPkScrWarp);
  auto bin = [&](int u) {
    const uint32_t wa = h[u], wb = hw[u];
    h[u] = 0u;
    hw[u] = 0u;
    const uint32_t c = wa & 0xFFFFu;
    if (ghist) atomicAdd(&ghist[u], (GH)c);
    const uint32_t ss[3] = {wb >> 16, wa >> 16, wb & 0xFFFFu};
    acc(u, c, ss);
  };
  const uint32_t lt = (1u << lane) - 1u;
  int n = 0;
  uint32_t* ctr2 = vcnt + 6;  // 128-bin chunks are grabbed dynamically too (the first nw statically)
  const uint32_t qs = (uint32_t)__cvta_generic_to_shared(q);  // queue base (shared window, kept in a register)
  for (int base = wig * 128; base < U;) {
    const int u = base + 4 * lane;
    uint4 w = make_uint4(0u, 0u, 0u, 0u);
    if (u < U) w = *reinterpret_cast<const uint4*>(h + u);  // h[U..U4) stay zero
    if (__any_sync(FULL, (w.x | w.y | w.z | w.w) != 0u)) {  // (a quarter of C5's chunks are empty)
      const uint32_t m = (w.x ? 1u : 0u) | (w.y ? 2u : 0u) | (w.z ? 4u : 0u) | (w.w ? 8u : 0u);
      const uint32_t c = __popc(m);
      const uint32_t b0 = __ballot_sync(FULL, c & 1u), b1 = __ballot_sync(FULL, c & 2u),
                     b2 = __ballot_sync(FULL, c & 4u);
      uint32_t pa = qs + 2u * (uint32_t)(n + __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt));
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (m & (1u << k)) {
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(pa), "h"((unsigned short)(u + k)) : "memory");
          pa += 2u;
        }
      n += __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
      __syncwarp();
      while (n >= 32) {
        n -= 32;
        bin(q[n + lane]);
      }
      __syncwarp();
    }
    uint32_t g = 0;
    if (lane == 0) g = atomicAdd(ctr2, 1u);
    base = 128 * ((int)__shfl_sync(FULL, g, 0) + nw);
  }
  if (lane < n) bin(q[lane]);
  __syncwarp();
  // (3) reduce and write: warp 0 combines the group's partial sums (one barrier)
  double mine[3];
  uint32_t ired[6];
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    mine[p] = xreduce4(a[p], lane);
    ired[p] = __reduce_add_sync(FULL, idl[p]);
    ired[3 + p] = __reduce_add_sync(FULL, swc[p]);
  }
  if (nw > 1) {
    double* d = scratch + wig * kPkScrWarp;
    if (wig > 0) {
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (lane == kLaneOf4[c]) d[4 * p + c] = mine[p];
      if (lane == 0)
        for (int j = 0; j < 6; ++j) d[12 + j] = __longlong_as_double((long long)ired[j]);
    }
    group_sync(gid_local, gsize);
    if (wig > 0) return;
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (lane == kLaneOf4[c])
          for (int w = 1; w < nw; ++w) mine[p] = __dadd_rn(mine[p], scratch[w * kPkScrWarp + 4 * p + c]);
    for (int w = 1; w < nw; ++w)
      for (int j = 0; j < 6; ++j) ired[j] += (uint32_t)__double_as_longlong(scratch[w * kPkScrWarp + 12 + j]);
  }
  double part[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double x0 = __shfl_sync(FULL, mine[0], kLaneOf4[c]);
    const double x1 = __shfl_sync(FULL, mine[1], kLaneOf4[c]);
    const double x2 = __shfl_sync(FULL, mine[2], kLaneOf4[c]);
    part[c] = lane == 0 ? x0 : (lane == 1 ? x1 : x2);
  }
  if (lane < 3) {
    dd tsum{part[0], 0.0}, esum{part[2], 0.0};
    dd_add2(tsum, part[1], 0.0);
    dd_add2(esum, part[3], 0.0);
    cs_agg r;
    r.avg_throughput_ips = __ddiv_rn(__dadd_rn(tsum.hi, tsum.lo), (double)P.S);  // fsum(ips)/n
    r.energy_proxy_wh = __dadd_rn(esum.hi, esum.lo);
    r.idle_steps = lane == 0 ? ired[0] : (lane == 1 ? ired[1] : ired[2]);
    r.switches = lane == 0 ? ired[3] : (lane == 1 ? ired[4] : ired[5]);
    r.violations = vcnt[lane];
    r.num_steps = P.S;
    if (P.agg) P.agg[t * 3 + lane] = r;
  }
  __syncwarp();
  if (lane < 3) vcnt[lane] = 0u;  // recounts of the next trace come after its first barrier
  if (lane == 0) vcnt[3 + vflag] = 0u;
  if (lane == 0) vcnt[6] = 0u;  // scan-chunk counter (all grabs of this trace were before the barrier)
}

// fp64 LUT search (cs_internal.h encoding) with thresholds and LUT in shared memory; leaves' bit 14
// (not proven violation-free) is ORed into flags like the fp32 path's bit 0.
struct Lut64 {
  const uint32_t* lut;
  const uint64_t* thr;
  int64_t lo, hi;
  uint64_t kbase;
  uint32_t s1, sub0;

  __device__ __forceinline__ uint64_t clampu(uint64_t x) const {
    int64_t si = (int64_t)x;
    si = si < lo ? lo : si;
    si = si > hi ? hi : si;
    return (uint64_t)si;
  }
  __device__ __forceinline__ uint32_t entry(uint64_t u) const { return lut[(uint32_t)((u >> s1) - kbase)]; }
  __device__ __forceinline__ uint32_t resolve(uint32_t e, uint64_t u, uint32_t& flags) const {
    while (e & kRedirect) e = lut[sub0 + (e >> 16) * kSubFan + (uint32_t)((u >> (e & 0x3Fu)) & 15u)];
    flags |= e;
    const uint32_t base = e >> 16;
    return base + (((e & 1u) != 0u && thr[base] <= u) ? 1u : 0u);
  }
  __device__ __forceinline__ uint32_t bin(uint64_t x, uint32_t& flags) const {
    const uint64_t u = clampu(x);
    return resolve(entry(u), u, flags);
  }
};

template <bool PEN, bool STEP, bool VIO>
__device__ __forceinline__ bool run_segment_f64(const EvalParams& P, const Lut64& L, uint32_t* h, uint32_t* sw,
                                                const uint64_t* s_sig, int64_t t, int64_t s0, int64_t s1e, int gtid,
                                                int gsize) {
  const DevTables& tb = P.tb;
  const int U = tb.U, M = tb.M;
  const unsigned long long* row = reinterpret_cast<const unsigned long long*>(P.caps) + t * P.ld;
  const unsigned char* vrow = reinterpret_cast<const unsigned char*>(row + s0);
  const int n = (int)(s1e - s0);
  uint32_t flags = 0;
  const uint32_t sw_s = PEN ? (uint32_t)__cvta_generic_to_shared(sw) : 0u;
  const uint32_t sw_dummy = sw_s + 4u * (uint32_t)(P.NSEG + (gtid & 31));  // 32 slots after the counters
  auto switches = [&](uint32_t cb, uint32_t pb) {
    if (cb != pb)
      for (int m = 0; m < M; ++m)
        count_switches(s_sig[(size_t)m * U + cb], s_sig[(size_t)m * U + pb], 0, 0, 0, sw_s, sw_dummy);
  };
  // 4 caps (two 128-bit loads) per lane and pass: entries first, then the leaves, for ILP
  const int nq = n >> 2;
  auto bins4 = [&](int q, uint32_t (&b)[4]) {
    const uint4 ra = ldg_stream(vrow + (size_t)q * 32), rb = ldg_stream(vrow + (size_t)q * 32 + 16);
    uint64_t u[4] = {((uint64_t)ra.y << 32) | ra.x, ((uint64_t)ra.w << 32) | ra.z, ((uint64_t)rb.y << 32) | rb.x,
                     ((uint64_t)rb.w << 32) | rb.z};
    uint32_t e[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) u[k] = L.clampu(u[k]);
#pragma unroll
    for (int k = 0; k < 4; ++k) e[k] = L.entry(u[k]);
#pragma unroll
    for (int k = 0; k < 4; ++k) b[k] = L.resolve(e[k], u[k], flags);
#pragma unroll
    for (int k = 0; k < 4; ++k) atomicAdd(&h[b[k]], 1u);
    if (STEP) {
      uint2 o;
      o.x = (b[0] & 0xFFFFu) | (b[1] << 16);
      o.y = (b[2] & 0xFFFFu) | (b[3] << 16);
      *reinterpret_cast<uint2*>(P.step_bins + t * P.ld_bins + s0 + 4 * (int64_t)q) = o;
    }
  };
  if constexpr (PEN) {
    // warp-contiguous runs of 4-cap groups, the previous step's bin through shuffles (as in the
    // fp32 loop): only a warp's first group reloads a cap
    const int lane = gtid & 31, nwg = gsize >> 5;
    const int per = (((nq + nwg - 1) / nwg) + 3) & ~3;  // 128-B aligned warp runs
    const int qb = min(nq, (gtid >> 5) * per), qe = min(nq, qb + per);
    uint32_t carry = kStepZero;
    if (qb < qe && s0 + 4 * (int64_t)qb > 0) {
      uint32_t dummy = 0;
      carry = L.bin(__ldg(row + s0 + 4 * (int64_t)qb - 1), dummy);
    }
    for (int base = qb; base < qe; base += 32) {
      const int q = base + lane;
      const bool act = q < qe;
      uint32_t b[4] = {0u, 0u, 0u, 0u};
      if (act) bins4(q, b);
      const uint32_t left = __shfl_sync(0xffffffffu, b[3], (lane + 31) & 31);
      uint32_t pb = lane == 0 ? carry : left;
      carry = __shfl_sync(0xffffffffu, b[3], 31);
      if (pb == kStepZero) pb = b[0];  // step 0 is never penalised (sim.py:119)
      if (act) {
        switches(b[0], pb);
        switches(b[1], b[0]);
        switches(b[2], b[1]);
        switches(b[3], b[2]);
      }
    }
  } else {
    for (int q = gtid; q < nq; q += gsize) {
      uint32_t b[4];
      bins4(q, b);
    }
  }
  for (int i = 4 * nq + gtid; i < n; i += gsize) {  // tail (< 4 caps at the end of the segment)
    const int64_t gi = s0 + i;
    const uint32_t b = L.bin(__ldg(row + gi), flags);
    atomicAdd(&h[b], 1u);
    if (PEN) {
      uint32_t dummy = 0;
      switches(b, gi > 0 ? L.bin(__ldg(row + gi - 1), dummy) : b);
    }
    if (STEP) P.step_bins[t * P.ld_bins + gi] = (uint16_t)b;
  }
  return VIO && (flags & 0x4000u);
}

template <typename CapT, bool PEN, bool STEP, bool VIO, bool UNI = false, bool PK = false>
__global__ void __launch_bounds__(1024, 1) eval_kernel(const __grid_constant__ EvalParams P) {
  constexpr bool F32 = sizeof(CapT) == 4;
  extern __shared__ __align__(16) unsigned char smem[];
  const DevTables& tb = P.tb;
  const int U = tb.U, M = tb.M;

  // ---- N1: stage the tables into shared memory once per CTA ----
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(smem);
  stage_words(s_lut, P.lv.lut, P.n_lut);
  // fp64 tables: the thresholds the leaves compare against (fp32 leaves need none)
  uint64_t* s_thr = reinterpret_cast<uint64_t*>(smem + P.off_vio);
  if (!F32)
    for (int i = threadIdx.x; i < U - 1; i += blockDim.x) s_thr[i] = __ldg(P.lv.thr64 + i);
  uint64_t* s_sig = reinterpret_cast<uint64_t*>(smem + P.off_sig);
  if (PK) {
    // {seg2 | seg0 << 16, seg1}: absolute segment ids (see pk_step)
    uint2* s2 = reinterpret_cast<uint2*>(s_sig);
    const uint32_t f0 = (uint32_t)__ldg(tb.seg_off), f1 = (uint32_t)__ldg(tb.seg_off + 1),
                   f2 = (uint32_t)__ldg(tb.seg_off + 2);
    for (int i = threadIdx.x; i < U; i += blockDim.x) {
      const uint64_t g = __ldg(tb.sig + i);
      s2[i] = make_uint2((f2 + (uint32_t)((g >> 32) & 0xFFFFu)) | ((f0 + (uint32_t)(g & 0xFFFFu)) << 16),
                         f1 + (uint32_t)((g >> 16) & 0xFFFFu));
    }
  } else if (PEN) {
    // signatures with each (grid, policy)'s first segment index folded in, so the 16-bit fields
    // are absolute switch-counter indices (the plan keeps NSEG <= 0xFFFF, so no field carries)
    for (int i = threadIdx.x; i < M * U; i += blockDim.x) {
      const int m = i / U;
      const uint64_t fold = (uint64_t)(uint32_t)__ldg(tb.seg_off + 3 * m) |
                            ((uint64_t)(uint32_t)__ldg(tb.seg_off + 3 * m + 1) << 16) |
                            ((uint64_t)(uint32_t)__ldg(tb.seg_off + 3 * m + 2) << 32);
      s_sig[i] = __ldg(tb.sig + i) + fold;
    }
  }
  // CTA-level global histogram in 32-bit counters (native shared atomics); a group that would
  // push the CTA's running step count past 2^31 first drains the counters into the global u64
  // histogram (atomicExch, so concurrent groups lose nothing).
  uint32_t* s_ghist = reinterpret_cast<uint32_t*>(smem + P.off_ghist);
  uint32_t* s_gsteps = s_ghist + U;
  const bool want_hist = P.hist != nullptr && P.nseg == 1;
  const bool gh_direct = want_hist && P.gh_direct != 0;
  if (want_hist && !gh_direct) {
    for (int i = threadIdx.x; i < U; i += blockDim.x) s_ghist[i] = 0u;
    if (threadIdx.x == 0) *s_gsteps = 0u;
  }

  // per-launch segment tables (prep_kernel): staged when they fit, else read through L1
  const bool seg_staged = P.seg_smem_bytes > 0;
  uint32_t* s_seghdr = reinterpret_cast<uint32_t*>(smem + P.off_seg);
  int32_t* s_segidle = reinterpret_cast<int32_t*>(s_seghdr + ((P.NSEG + 3) & ~3));
  double2* s_segval = reinterpret_cast<double2*>(s_segidle + ((M * 3 + 3) & ~3));
  double2* s_binval = reinterpret_cast<double2*>(smem + P.off_seg);
  double2* s_pkraw = reinterpret_cast<double2*>(smem + P.off_seg);  // PK: {thr, energy} per segment
  double* s_pkq = reinterpret_cast<double*>(smem + P.off_pkq);         //     the 3 policies' quanta
  if (PK) {
    if (seg_staged)
      for (int i = threadIdx.x; i < P.NSEG; i += blockDim.x) s_pkraw[i] = __ldg(P.seg_raw + i);
    if (threadIdx.x < 12) s_pkq[threadIdx.x] = __ldg(P.seg_q + threadIdx.x);
  } else if (!PEN && P.bin_epi) {
    stage_words(reinterpret_cast<uint32_t*>(s_binval), reinterpret_cast<const uint32_t*>(P.bin_val), 24 * P.U4);
  } else if (seg_staged) {
    const int NS = P.NSEG, NV = PEN ? 3 : 2;
    const double2* gv = reinterpret_cast<const double2*>(P.seg_val);
    for (int i = threadIdx.x; i < NS; i += blockDim.x) s_seghdr[i] = __ldg(P.seg_hdr + i);
    for (int i = threadIdx.x; i < M * 3; i += blockDim.x) s_segidle[i] = __ldg(P.seg_idle + i);
    for (int i = threadIdx.x; i < NV * NS; i += blockDim.x) s_segval[i] = __ldg(gv + i);
  }

  const int gsize = P.wpg * 32;
  const int gid_local = threadIdx.x / gsize;
  const int gtid = threadIdx.x - gid_local * gsize;
  unsigned char* gbase = smem + P.off_groups + (size_t)gid_local * P.group_bytes;
  uint32_t* h = reinterpret_cast<uint32_t*>(gbase);
  uint32_t* sw = reinterpret_cast<uint32_t*>(gbase + P.off_g_sw);
  uint32_t* vcnt = reinterpret_cast<uint32_t*>(gbase + P.off_g_vio);
  double* scratch = reinterpret_cast<double*>(gbase + P.off_g_scr);
  const int U4 = P.U4;
  for (int u = gtid; u < U4; u += gsize) h[u] = 0u;
  if (PK)
    for (int u = gtid; u < U4; u += gsize) sw[u] = 0u;
  else if (PEN)
    for (int i = gtid; i < P.NSEG; i += gsize) sw[i] = 0u;
  if (gtid < M * 3) vcnt[gtid] = 0u;
  if (gtid == 0) vcnt[M * 3] = 0u;  // group "violation seen" flag (the plan keeps 3M < group size)
  if (PK && gtid == 0) vcnt[M * 3 + 1] = vcnt[M * 3 + 2] = vcnt[M * 3 + 3] = 0u;  // PK: 2nd flag, counters
  uint32_t* edges = reinterpret_cast<uint32_t*>(gbase + P.off_g_edge);
  __syncthreads();

  Lut64 L64;
  L64.lut = s_lut;
  L64.thr = s_thr;
  L64.lo = P.lv.lo;
  L64.hi = P.lv.hi;
  L64.kbase = P.lv.kbase;
  L64.s1 = P.lv.shift1;
  L64.sub0 = P.lv.sub0;
  Lut32 L;
  L.lut = s_lut;
  L.kb = (int32_t)P.lv.kbase;
  L.s1 = P.lv.shift1;
  L.lo = L.kb << L.s1;
  L.lutk = (uint32_t)__cvta_generic_to_shared(s_lut) - 4u * (uint32_t)L.kb;
  L.hi = ((L.kb + P.n_level1) << L.s1) - 1;
  L.sub0 = P.lv.sub0;
  L.s2 = P.lut_s2;
  L.lutb = (uint32_t)__cvta_generic_to_shared(s_lut);
  L.s2m2 = L.s2 >= 2u ? L.s2 - 2u : 0u;

  const int64_t n_items = P.T * (int64_t)P.nseg;
  const int64_t n_groups = (int64_t)gridDim.x * P.gpc;
  uint32_t tma_seq = 0;  // CS_TMA variant: this warp's bulk-copy stage uses so far
#ifdef CS_TMA
  if ((gtid & 31) == 0) {
    const uint32_t bs = (uint32_t)__cvta_generic_to_shared(gbase + P.off_g_ring + (gtid >> 5) * kTmaWarpBytes) +
                        kTmaStages * kTmaStageBytes;
    for (int k = 0; k < kTmaStages; ++k) mbar_init(bs + 8 * k);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
#endif
  // Items (traces, or trace segments) are handed out dynamically: the first n_groups statically, then
  // each group's leader takes the next from a global counter while its group still works on the
  // current one, so groups finish together whatever the traces' costs (static round-robin left a
  // tail of up to one trace per group: a few % at C3, more with few traces per group at N GPUs).
  // The next item travels through the group's shared slot across a barrier the item has anyway.
  uint32_t* s_next = vcnt + 3 * M + 4;  // [lo, hi]
  auto grab_next = [&]() {
    if (gtid == 0) {
      const unsigned long long nx = (unsigned long long)n_groups + atomicAdd(P.work, 1ull);
      s_next[0] = (uint32_t)nx;
      s_next[1] = (uint32_t)(nx >> 32);
    }
  };
  auto read_next = [&]() -> int64_t { return (int64_t)((uint64_t)s_next[0] | ((uint64_t)s_next[1] << 32)); };
  int iter = 0;
  for (int64_t item = (int64_t)blockIdx.x * P.gpc + gid_local; item < n_items; ++iter) {
    if constexpr (PK) {  // whole traces (nseg == 1), two barriers per trace (pk_finish)
      const int64_t t = item;
      const int vflag = iter & 1;
      const bool bad = pk_main(P, L, h, sw, edges, reinterpret_cast<const uint2*>(s_sig), vcnt + 5, t, gtid, gsize);
      if (VIO && bad) atomicOr(&vcnt[3 + vflag], 1u);
      grab_next();
      group_sync(gid_local, gsize);
      item = read_next();
      if (gtid == 0) vcnt[5] = 0u;  // block counter: every grab of this trace came before the barrier
      if (VIO && vcnt[3 + vflag]) {  // never taken when the tables are right: exact recount
        const CapT* row = reinterpret_cast<const CapT*>(P.caps) + t * P.ld;
        recount_violations<CapT>(P, s_lut, row, 0, P.S, vcnt, gtid, gsize);
        group_sync(gid_local, gsize);
      }
      if (want_hist) {
        uint32_t before = 0;
        if (gtid == 0) before = atomicAdd(s_gsteps, (uint32_t)P.S);
        before = __shfl_sync(0xffffffffu, before, 0);
        if (before > (1u << 31) && gtid < 32) {  // rare: drain the 32-bit counters (this warp)
          if (gtid == 0) atomicExch(s_gsteps, 0u);
          for (int u = gtid; u < U; u += 32) {
            const uint32_t c = atomicExch(&s_ghist[u], 0u);
            if (c) atomicAdd(P.hist + u, (unsigned long long)c);
          }
        }
      }
      uint32_t* gh = want_hist ? s_ghist : (uint32_t*)nullptr;
      if (seg_staged)
        pk_finish<true>(P, t, h, sw, edges, reinterpret_cast<const uint2*>(s_sig), vcnt, vflag, gh, s_pkraw, s_pkq,
                        scratch, gtid, gsize, gid_local);
      else
        pk_finish<false>(P, t, h, sw, edges, reinterpret_cast<const uint2*>(s_sig), vcnt, vflag, gh, P.seg_raw,
                         s_pkq, scratch, gtid, gsize, gid_local);
      continue;  // (item was set after the first barrier)
    }
    const int64_t t = item / P.nseg;
    const int64_t s0 = (item - t * P.nseg) * P.seg_len;
    const int64_t s1e = min(P.S, s0 + P.seg_len);
    bool bad;
    if constexpr (F32)
      bad = run_segment_f32<PEN, STEP, VIO, UNI>(P, L, h, sw, s_sig, t, s0, s1e, gtid, gsize, tma_seq);
    else
      bad = run_segment_f64<PEN, STEP, VIO>(P, L64, h, sw, s_sig, t, s0, s1e, gtid, gsize);
    if (VIO && bad) atomicOr(&vcnt[M * 3], 1u);
    group_sync(gid_local, gsize);
    if (VIO && vcnt[M * 3]) {  // never taken when the tables are right: exact recount
      const CapT* row = reinterpret_cast<const CapT*>(P.caps) + t * P.ld;
      recount_violations<CapT>(P, s_lut, row, s0, s1e, vcnt, gtid, gsize);
      group_sync(gid_local, gsize);
    }
    if (P.nseg == 1) {
      if (want_hist && !gh_direct) {
        uint32_t before = 0;
        if (gtid == 0) before = atomicAdd(s_gsteps, (uint32_t)(s1e - s0));
        before = __shfl_sync(0xffffffffu, before, 0);
        if (before > (1u << 31)) {  // rare: drain the 32-bit counters (this warp does it)
          if (gtid < 32) {
            if (gtid == 0) atomicExch(s_gsteps, 0u);
            for (int u = gtid; u < U; u += 32) {
              const uint32_t c = atomicExch(&s_ghist[u], 0u);
              if (c) atomicAdd(P.hist + u, (unsigned long long)c);
            }
          }
        }
      }
      uint32_t* gh = want_hist ? s_ghist : (uint32_t*)nullptr;
      if (gh_direct) {  // (the plan takes it only with the segment epilogues)
        if (seg_staged)
          finish_trace<PEN, false>(P, t, h, sw, vcnt, P.hist, s_seghdr, s_segidle, s_segval, scratch, gtid, gsize,
                                   gid_local);
        else
          finish_trace<PEN, true>(P, t, h, sw, vcnt, P.hist, P.seg_hdr, P.seg_idle,
                                  reinterpret_cast<const double2*>(P.seg_val), scratch, gtid, gsize, gid_local);
      } else if (!PEN && P.bin_epi)
        finish_trace_bins(P, t, h, vcnt, gh, s_binval, scratch, gtid, gsize, gid_local);
      else if (seg_staged)  // two instantiations so each reads its tables with a known address space
        finish_trace<PEN, false>(P, t, h, sw, vcnt, gh, s_seghdr, s_segidle, s_segval, scratch, gtid, gsize, gid_local);
      else
        finish_trace<PEN, true>(P, t, h, sw, vcnt, gh, P.seg_hdr, P.seg_idle, reinterpret_cast<const double2*>(P.seg_val),
                          scratch, gtid, gsize, gid_local);
    } else {
      // split trace: fold this segment's partial histogram into the trace's global partials
      for (int u = gtid; u < U; u += gsize) {
        const uint32_t c = h[u];
        if (c) {
          atomicAdd(&P.part_hist[t * U4 + u], c);
          h[u] = 0u;
        }
      }
      if (PEN)
        for (int i = gtid; i < P.NSEG; i += gsize) {
          const uint32_t sv = sw[i];
          if (sv) {
            atomicAdd(&P.part_sw[t * P.NSEG + i], sv);
            sw[i] = 0u;
          }
        }
      if (gtid < M * 3 && vcnt[gtid]) atomicAdd(&P.part_vio[t * M * 3 + gtid], vcnt[gtid]);
    }
    grab_next();
    group_sync(gid_local, gsize);
    if (gtid <= M * 3) vcnt[gtid] = 0u;
    group_sync(gid_local, gsize);
    item = read_next();
  }
  if (gtid == 0 && atomicAdd(P.work + 1, 1ull) == (unsigned long long)n_groups - 1ull) {
    P.work[0] = 0ull;  // every group has taken its last item: re-arm for the next launch
    P.work[1] = 0ull;
  }

  if (want_hist && !gh_direct) {
    __syncthreads();
    for (int u = threadIdx.x; u < U; u += blockDim.x) {
      const uint32_t c = s_ghist[u];
      if (P.hist_store)
        P.hist[u] = c;
      else if (c)
        atomicAdd(P.hist + u, (unsigned long long)c);
    }
  }
}

// Epilogue of traces split across worker groups: one CTA per (trace, grid). Each CTA scans its
// own shared-memory copy of the trace's partial histogram (the (t, 0) CTA also folds it into the
// global histogram) and writes that grid's three aggregates — M-way parallel for the few long
// traces of C1/C2-like sweeps instead of one CTA walking every grid's segments.
template <bool PEN>
__global__ void __launch_bounds__(1024) finalize_kernel(const __grid_constant__ EvalParams P) {
  extern __shared__ __align__(16) unsigned char fsmem[];
  const int64_t t = blockIdx.x;
  const int U4 = P.U4, M = P.tb.M;
  // gridDim.y == M: per-grid CTAs on a shared-memory copy; gridDim.y == 1: one CTA per trace
  // scanning the global partial histogram in place (unions too large for shared memory)
  const bool split = P.fin_split != 0;
  const int m = blockIdx.y;
  uint32_t* hg = P.part_hist + t * U4;
  uint32_t* h = split ? reinterpret_cast<uint32_t*>(fsmem) : hg;
  double* scratch = reinterpret_cast<double*>(fsmem + (split ? (size_t)U4 * 4 : 0));
  if (split)
    for (int u = 4 * threadIdx.x; u < U4; u += 4 * blockDim.x)
      *reinterpret_cast<uint4*>(h + u) = *reinterpret_cast<const uint4*>(hg + u);
  __syncthreads();
  if (split && P.hist) {
    // the trace's histogram folds into the global one in M slices, one per grid CTA (a single
    // CTA issuing all U global atomics was the longest part of C2's finalize)
    const int U = P.tb.U, lo = (int)((int64_t)U * m / M), hi = (int)((int64_t)U * (m + 1) / M);
    for (int u = lo + threadIdx.x; u < hi; u += blockDim.x)
      if (h[u]) atomicAdd(P.hist + u, (unsigned long long)h[u]);
    __syncthreads();  // the scan below rewrites h in place
  }
  group_scan(h, U4, (!split && m == 0) ? P.hist : (unsigned long long*)nullptr, reinterpret_cast<uint32_t*>(scratch),
             threadIdx.x, blockDim.x, 0);
  group_sync(0, blockDim.x);
  const uint32_t* sw = PEN ? P.part_sw + t * (int64_t)P.NSEG : nullptr;
  const uint32_t* vc = P.part_vio + t * (int64_t)M * 3;
  // (warp-owned pairs here too measured equal at C2: 31.3 us/step either way)
  epilogue<PEN, true>(P, t, h, sw, vc, P.seg_hdr, P.seg_idle, reinterpret_cast<const double2*>(P.seg_val), scratch,
                threadIdx.x, blockDim.x, 0, split ? m : 0, split ? m + 1 : M);
}

// ----------------------------------------------------------------------------------------
// host side: launch planning
// ----------------------------------------------------------------------------------------
thread_local cudaEvent_t g_ev0 = nullptr, g_ev1 = nullptr;
thread_local int g_last_launches = 0;
thread_local cs_eval_plan g_last_plan{};
thread_local bool g_timed = false;

struct Plan {
  int threads, wpg, gpc, ctas;
  bool uni = false;
  bool pk = false;  // packed-penalty variant (PK)  // warp-uniform redirect variant (sub-tables > 5 % of the staged LUT's level-1 buckets)
  int32_t nseg;
  int64_t seg_len;
  size_t smem;
  size_t ws_prep, ws_split;
  EvalParams P;
};

int sm_count(int dev) {
  static int cache[64] = {0};
  if (dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev);
  return cache[dev];
}

template <typename CapT, bool PEN, bool STEP, bool VIO, bool UNI = false, bool PK = false>
void* kptr() {
  return (void*)eval_kernel<CapT, PEN, STEP, VIO, UNI, PK>;
}

// uni: the warp-uniform redirect variant (fp32, no penalty, no per-step output only; CS_UNI builds)
// pk: the packed-penalty variant (fp32, one grid, penalty, no per-step output, < 2^16 steps)
void* pick_kernel(bool f32, bool pen, bool step, bool vio, bool uni = false, bool pk = false) {
  if (pk && f32 && pen && !step)
    return vio ? kptr<float, true, false, true, false, true>() : kptr<float, true, false, false, false, true>();
#ifdef CS_UNI
  if (uni && f32 && !pen && !step) return vio ? kptr<float, false, false, true, true>() : kptr<float, false, false, false, true>();
#endif
#define CS_K(A, B, C) \
  if (pen == A && step == B && vio == C) return f32 ? kptr<float, A, B, C>() : kptr<double, A, B, C>();
  CS_K(false, false, false)
  CS_K(false, false, true)
  CS_K(false, true, false)
  CS_K(false, true, true)
  CS_K(true, false, false)
  CS_K(true, false, true)
  CS_K(true, true, false)
  CS_K(true, true, true)
#undef CS_K
  return nullptr;
}

size_t a16(size_t x) { return (x + 15) & ~(size_t)15; }
size_t bin_bytes_of(const EvalParams& P) { return (size_t)6 * P.U4 * 16; }

// Resident CTAs per SM for (kernel, block size, dynamic smem), memoised: the plan search asks
// for dozens of candidates per launch and the occupancy API dominates small launches otherwise.
int blocks_per_sm(void* fn, int dev, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<void*, int, int, size_t>, int> cache;
  const auto key = std::make_tuple(fn, dev, threads, smem);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  int per_sm = 0;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    per_sm = 0;
  }
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = per_sm;
  return per_sm;
}

std::string make_plan(const Tables& t, const DevTables& view, const cs_eval_args* a, int dev, Plan& pl,
                      bool allow_pk = true) {
  const bool f32 = t.cap_dtype == CS_CAP_F32;
  const bool pen = a->switch_penalty_s > 0.0;
  const bool vio = (a->flags & CS_FLAG_CHECK_VIOLATIONS) != 0;
  const int U = t.U, M = t.M;
  // PK: 16-bit packed step / switched-step counters need < 2^16 steps per trace (whole traces per
  // group; re-planned without it when the plan splits traces); CS_PLAN_NO_PK: tuning only
  static const bool no_pk_env = std::getenv("CS_PLAN_NO_PK") != nullptr;
  // (the last block's fill steps count too: < 4 kPkBlkVec of them)
  const bool pk = allow_pk && !no_pk_env && f32 && pen && M == 1 && a->step_bins == nullptr &&
                  a->n_steps <= 0xFFFF - 4 * kPkBlkVec && !(a->flags & CS_FLAG_SEGMENT_EPILOGUE);
  const int pk_nblk = pk ? (int)((a->n_steps / 4 + kPkBlkVec - 1) / kPkBlkVec) : 0;
  const size_t pkq_bytes = pk ? 128 : 0;  // the 3 policies' quanta (12 doubles)
  void* fn = pick_kernel(f32, pen, a->step_bins != nullptr, vio, false, pk);
  int smem_optin = 232448;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int nsm = sm_count(dev);
  const size_t lut_bytes = a16((size_t)t.lut.size() * 4);
  const size_t vio_bytes = !f32 ? a16((size_t)U * 8) : 0;  // fp64: the thresholds (s_thr)
  const int U4 = (U + 3) & ~3;
  const int nsegs = (int)(t.seg.size() / 4);
  if (pen && nsegs > 0xFFFF)  // the engine then evaluates the grids in chunks
    return "tables too large for shared memory (" + std::to_string(nsegs) +
           " selection segments: switch counters use 16-bit indices)";
  const size_t sig_bytes = pen ? a16((size_t)M * U * 8 + (size_t)(M * 3 + 1) * 4) : 0;
  // long traces with the segment epilogue fold each trace's histogram straight into hist (U global
  // atomics per trace are < 2 % of its steps) instead of keeping a CTA copy in shared memory
  static const char* ghd_env = std::getenv("CS_PLAN_GH_DIRECT");  // tuning only
  const bool gh_direct = a->hist != nullptr && !pk && !(M == 1 && !pen) &&
                         (ghd_env ? std::atoi(ghd_env) != 0 : (int64_t)U * 64 <= a->n_steps);
  const size_t gh_bytes = a->hist && !gh_direct ? a16((size_t)U * 4 + 4) : 0;
  // segment tables (prep_kernel): hdr [NS] u32, idle flags [M*3] i32, values [6][NS] f64 in the
  // workspace; the kernel stages hdr, flags and the 4 (6 with a penalty) value arrays it reads
  const size_t seg_hdr_b = (size_t)((nsegs + 3) & ~3) * 4, seg_idle_b = (size_t)((M * 3 + 3) & ~3) * 4;
  const size_t seg_ws = a16(seg_hdr_b + seg_idle_b + (size_t)(6 + 2) * nsegs * 8 + (size_t)M * 3 * 4 * 8);
  // one grid without a penalty: the bin epilogue's per-bin tables replace the segment tables
  const bool bin_epi = !pen && M == 1 && (double)a->n_traces * (double)a->n_steps >= (double)(1 << 22) &&
                       !(a->flags & CS_FLAG_SEGMENT_EPILOGUE);
  const size_t bin_bytes = (size_t)6 * U4 * 16;
  const size_t seg_smem = pk        ? a16((size_t)nsegs * 16)  // PK: {thr, energy} per segment
                          : bin_epi ? bin_bytes
                                    : a16(seg_hdr_b + seg_idle_b + (size_t)(pen ? 6 : 4) * nsegs * 8);
  auto group_bytes = [&](int wpg, size_t* off_sw, size_t* off_v, size_t* off_scr) {
    size_t gb = a16((size_t)U4 * 4);
    *off_sw = gb;
    // PK: the second packed word per bin; else + 32 dummy slots (branch-free switch counting)
    gb += pk ? a16((size_t)(U4 + 32) * 4) : pen ? a16((size_t)(nsegs + 32) * 4) : 0;
    *off_v = gb;
    gb += a16((size_t)(M * 3 + 6) * 4);  // PK: + alternating flag, block / scan-chunk counters; next item
    if (pk) gb += a16((size_t)pk_nblk * 4);  // block edges (pk_main)
#ifdef CS_TMA
    gb = a16(gb);
    *off_scr = gb;  // (the ring is placed by the kernel at off_g_ring = this + scratch)
    gb += (size_t)wpg * (pk ? kPkScrWarp : 24) * 8;
    gb = (gb + 127) & ~(size_t)127;
    gb += (size_t)wpg * kTmaWarpBytes;
    return a16(gb);
#endif
    *off_scr = gb;
    gb += (size_t)wpg * (pk ? kPkScrWarp : 24) * 8;
    return a16(gb);
  };
  // candidates: most resident warps per SM first, then the smallest worker group; the segment
  // tables go to shared memory unless that costs resident warps, and so does the big LUT
  struct Cand {
    int warps = -1, threads = 0, wpg = 0, per_sm = 0;
    size_t smem = 0;
    bool staged = false;
  };
  // small launches (latency-bound: a few traces x a few thousand steps) skip the optional
  // stagings — loading ~100 KB of tables per CTA costs more than the lookups it speeds up
  const bool small = (double)a->n_traces * (double)a->n_steps < (double)(1 << 22);
  // tiny launches (fewer traces than SMs, <= 1M timesteps): a trace per CTA, all its warps on it
  const bool tiny = a->n_traces < nsm && (double)a->n_traces * (double)a->n_steps <= (double)(1 << 20);
  static const int force_wpg = std::getenv("CS_PLAN_WPG") ? std::atoi(std::getenv("CS_PLAN_WPG")) : 0;  // tuning only
  auto search = [&](size_t lut_b) {
    Cand b;
    const size_t fixed0 = lut_b + vio_bytes + sig_bytes + gh_bytes + pkq_bytes;
    for (int staged = small ? 0 : 1; staged >= 0; --staged)
      for (int threads : {1024, 512, 256, 128}) {
        for (int wpg : {1, 2, 4, 8, 16, 32}) {
          const int wpc = threads / 32;
          if (wpg > wpc) continue;
          if (tiny ? wpg != wpc : (wpg == 32 && force_wpg != 32)) continue;  // tiny: one whole-CTA group per trace
          // ... of at most 512 threads when the trace is too short to split (C1, 1440 steps:
          // 14.7 us per step at 512 threads, 16.8 at 1024 — staging and barriers dominate)
          // (unless the 3M + 1 per-group counters need the bigger CTA: > 170 grids)
          if (tiny && a->n_steps < 4096 && threads > 512 && M * 3 + 1 <= 512) continue;
          if (force_wpg && wpg != force_wpg) continue;
          if (wpg * 32 < M * 3 + 1) continue;  // one thread per violation counter (+ the flag)
          const int gpc = wpc / wpg;
          if (wpg > 1 && gpc > 15) continue;  // named barriers 1..15
          size_t o1, o2, o3;
          const size_t smem = fixed0 + (staged ? seg_smem : 0) + (size_t)gpc * group_bytes(wpg, &o1, &o2, &o3);
          if (smem > (size_t)smem_optin) continue;
          const int per_sm = blocks_per_sm(fn, dev, threads, smem);
          if (per_sm < 1) continue;
          const int warps = tiny ? wpc : per_sm * wpc;  // tiny: the biggest CTA, it runs alone
          // PK: the smaller worker group wins even unstaged — its per-trace barriers and epilogue
          // cost more than reading the compact segment pairs through L1 (C5: 4-warp groups with
          // the tables in global memory 2.64 ms, 8-warp groups staged 3.23 ms)
          if (warps > b.warps ||
              (warps == b.warps && wpg < b.wpg && (pk || staged == (int)b.staged))) {
            b.warps = warps, b.threads = threads, b.wpg = wpg, b.per_sm = per_sm, b.smem = smem;
            b.staged = staged != 0;
          }
        }
      }
    return b;
  };
  Cand c = search(lut_bytes);
  int big = 0;  // 1: the big LUT, 2: the huge one
  if (f32 && !small && !std::getenv("CS_PLAN_NO_BIG")) {  // env: tuning only
    // a finer LUT when it costs no resident warps and no bigger worker groups: a group's barriers,
    // shared histogram and per-trace epilogue cost more than the finer LUT saves (C5: 8-warp
    // groups with the big LUT 5.41 ms, 4-warp groups with the main 4.99; C3: 16-warp groups with
    // the shift-11 LUT 6.63 ms, 8-warp groups with the shift-12 5.86)
    const Cand c0 = c;
    for (int which : {2, 1}) {
      const int32_t n = which == 2 ? view.n_lut_huge : view.n_lut_big;
      if (n <= 0) continue;
      const Cand cb = search(a16((size_t)n * 4));
      if (cb.warps >= c0.warps && cb.warps > 0 && cb.wpg <= c0.wpg && (cb.staged || !c0.staged)) {
        c = cb, big = which;
        break;
      }
    }
  }
  const int32_t n_lut_sel = big == 2 ? view.n_lut_huge : big == 1 ? view.n_lut_big : view.n_lut;
  const size_t lut_b = a16((size_t)n_lut_sel * 4);  // the LUT staged
  const size_t fixed0 = lut_b + vio_bytes + sig_bytes + gh_bytes + pkq_bytes;
  int best_warps = c.warps, b_threads = c.threads, b_wpg = c.wpg, b_per_sm = c.per_sm;
  size_t b_smem = c.smem;
  bool b_staged = c.staged;
  if (best_warps < 0)
    return "tables too large for shared memory (" + std::to_string(U) + " union bins, " +
           std::to_string(t.lut.size()) + " LUT entries)";
  pl.threads = b_threads;
  pl.wpg = b_wpg;
  pl.gpc = b_threads / 32 / b_wpg;
  pl.smem = b_smem;
  const int64_t groups_total = (int64_t)nsm * b_per_sm * pl.gpc;
  int64_t nseg = 1;
  if (a->n_traces < 2 * groups_total) {  // too few traces to fill the machine: split them
    const int64_t want = (2 * groups_total + a->n_traces - 1) / std::max<int64_t>(a->n_traces, 1);
    nseg = std::max<int64_t>(1, std::min(want, std::max<int64_t>(1, a->n_steps / 2048)));
  }
  int64_t seg_len = (a->n_steps + nseg - 1) / nseg;
  seg_len = (seg_len + 127) / 128 * 128;
  nseg = (a->n_steps + seg_len - 1) / seg_len;
  if (pk && nseg > 1) return make_plan(t, view, a, dev, pl, false);
  pl.pk = pk;
  pl.nseg = (int32_t)nseg;
  pl.seg_len = seg_len;
  pl.ctas = (int)std::max<int64_t>(
      1, std::min<int64_t>((int64_t)nsm * b_per_sm, (a->n_traces * nseg + pl.gpc - 1) / pl.gpc));
  pl.ws_prep = seg_ws + (bin_epi && b_staged ? bin_bytes : 0);
  pl.ws_split = nseg > 1 ? (size_t)a->n_traces *
                               ((size_t)U4 + (pen ? (size_t)nsegs : 0) + (size_t)M * 3) * sizeof(uint32_t)
                         : 0;

  EvalParams& P = pl.P;
  P = EvalParams{};
  P.tb = view;
  P.lv = big == 2 ? view.lv_huge : big == 1 ? view.lv_big : view.lv;
  P.n_lut = n_lut_sel;
  P.n_level1 = big == 2 ? view.n_level1_huge : big == 1 ? view.n_level1_big : view.n_level1;
  {
    const uint32_t s1 = P.lv.shift1 < 32 ? P.lv.shift1 : 31, s2 = s1 >= 4 ? s1 - 4 : 0;
    P.lut_s2 = s2;
    // the warp-uniform redirect variant (UNI) served redirect-heavy tables (C3) while the per-lane
    // redirect step compiled to divergent branches; with predicated sub-table loads the per-lane
    // path is faster there too (C3 5.36 -> 5.31 ms, iid equal): UNI is an A/B build only now
#ifdef CS_UNI
    pl.uni = f32 && (double)(P.n_lut - P.n_level1) / kSubFan > 0.05 * (double)P.n_level1;
#else
    pl.uni = false;
#endif
  }
  P.t0_bits = (f32 && !t.thresholds.empty()) ? (int32_t)(uint32_t)t.thresholds[0] : INT32_MIN;
  P.caps = a->caps;
  P.T = a->n_traces;
  P.S = a->n_steps;
  P.ld = a->ld;
  P.seg_len = seg_len;
  P.nseg = (int32_t)nseg;
  P.step_seconds = a->step_seconds;
  {
    const double step = (double)a->step_seconds;
    const double pen_s = a->switch_penalty_s < step ? a->switch_penalty_s : step;  // sim.py:111
    P.omp = 1.0 - pen_s / step;
  }
  P.step_bins = a->step_bins;
  P.ld_bins = a->ld_bins;
  P.agg = a->agg;
  P.hist = reinterpret_cast<unsigned long long*>(a->hist);
  P.wpg = pl.wpg;
  P.gpc = pl.gpc;
  P.U4 = U4;
  P.NSEG = nsegs;
  P.off_vio = (int32_t)lut_b;
  P.off_sig = (int32_t)(lut_b + vio_bytes);
  P.off_ghist = (int32_t)(lut_b + vio_bytes + sig_bytes);
  P.off_pkq = (int32_t)(lut_b + vio_bytes + sig_bytes + gh_bytes);
  P.gh_direct = gh_direct ? 1 : 0;
  P.off_seg = (int32_t)fixed0;
  P.seg_smem_bytes = b_staged ? (int32_t)seg_smem : 0;
  P.bin_epi = (bin_epi && b_staged) ? 1 : 0;  // only with its tables in shared memory
  for (int pp = 0; pp < 3; ++pp) {
    int f = 0;
    while (f < t.grid_bins[0] && t.sel[(size_t)pp * t.maxB + f] < 0) ++f;
    P.fidle[pp] = f;
  }
  P.off_groups = (int32_t)(fixed0 + (b_staged ? seg_smem : 0));
  size_t o1, o2, o3;
  P.group_bytes = (int32_t)group_bytes(pl.wpg, &o1, &o2, &o3);
  P.off_g_sw = (int32_t)o1;
  P.off_g_vio = (int32_t)o2;
  P.off_g_scr = (int32_t)o3;
  P.off_g_edge = (int32_t)(o2 + a16((size_t)(M * 3 + 6) * 4));
#ifdef CS_TMA
  P.off_g_ring = (int32_t)((o3 + (size_t)pl.wpg * (pk ? kPkScrWarp : 24) * 8 + 127) & ~(size_t)127);
#endif
  return std::string();
}

}  // namespace

void set_last_launches(int n) { g_last_launches = n; }

std::string eval_workspace(const Tables& t, const DevTables& view, const cs_eval_args* a, int dev, size_t* bytes) {
  Plan pl;
  std::string err = make_plan(t, view, a, dev, pl);
  if (!err.empty()) return err;
  *bytes = a16(pl.ws_prep + pl.ws_split) + 16;  // + the dynamic-scheduling counter
  return std::string();
}

std::string launch_eval(const Tables& t, const DevTables& view, const cs_eval_args* a, int dev, cudaStream_t st) {
  Plan pl;
  std::string err = make_plan(t, view, a, dev, pl);
  if (!err.empty()) return err;
  const bool f32 = t.cap_dtype == CS_CAP_F32;
  const bool pen = a->switch_penalty_s > 0.0;
  const bool vio = (a->flags & CS_FLAG_CHECK_VIOLATIONS) != 0;
  EvalParams& P = pl.P;
  const size_t need = a16(pl.ws_prep + pl.ws_split) + 16;  // + the dynamic-scheduling counter
  if (a->workspace == nullptr || a->workspace_bytes < need)
    return "workspace too small: need " + std::to_string(need) + " bytes (cs_eval_workspace_size)";
  unsigned char* ws = reinterpret_cast<unsigned char*>(a->workspace);
  {
    const int NS = P.NSEG, M = t.M;
    P.seg_hdr = reinterpret_cast<const uint32_t*>(ws);
    P.seg_idle = reinterpret_cast<const int32_t*>(ws + (size_t)((NS + 3) & ~3) * 4);
    P.seg_val = reinterpret_cast<const double*>(ws + (size_t)((NS + 3) & ~3) * 4 + (size_t)((M * 3 + 3) & ~3) * 4);
    P.seg_raw = reinterpret_cast<const double2*>(P.seg_val + (size_t)6 * NS);
    P.seg_q = reinterpret_cast<const double*>(P.seg_raw + NS);
  }
  // bits of the exact hi part: counts up to S must keep sum(count x hi) below 2^53 quanta
  int L = 52;
  while (L > 1 && (double)a->n_steps >= std::ldexp(1.0, 53 - L)) --L;
  int launches = 0;
  P.bin_val = P.bin_epi ? reinterpret_cast<const double2*>(ws + pl.ws_prep - bin_bytes_of(P)) : nullptr;
  // dynamic scheduling counters {next item, groups done}: zeroed by prep_kernel, re-armed by the
  // last group out of each eval launch, so graph replays (no prep kernel) need no memset node
  P.work = reinterpret_cast<unsigned long long*>(ws + a16(pl.ws_prep + pl.ws_split));
  if (!(a->flags & CS_FLAG_PREPARED)) {  // the launch's value tables (constant across graph replays)
    prep_kernel<<<(unsigned)(t.M * 3), 256, 0, st>>>(view, (double)a->step_seconds, P.omp, L, P.NSEG,
                                                      const_cast<uint32_t*>(P.seg_hdr), const_cast<int32_t*>(P.seg_idle),
                                                      const_cast<double*>(P.seg_val), const_cast<double2*>(P.bin_val),
                                                      P.U4, const_cast<double2*>(P.seg_raw), const_cast<double*>(P.seg_q),
                                                      P.work);
    CS_CUDA_TRY(cudaGetLastError());
    ++launches;
  }
  // a single CTA owns the whole histogram: it stores it (the 32-bit CTA counters cannot wrap
  // below 2^31 timesteps) — one memset node less per graph replay for one-trace sweeps (C1)
  P.hist_store = (a->hist && !(a->flags & CS_FLAG_ACCUMULATE_HIST) && pl.ctas == 1 && pl.nseg == 1 && !P.gh_direct &&
                  (double)a->n_traces * (double)a->n_steps < 2147483648.0)
                     ? 1
                     : 0;
  if (a->hist && !(a->flags & CS_FLAG_ACCUMULATE_HIST) && !P.hist_store)
    CS_CUDA_TRY(cudaMemsetAsync(a->hist, 0, (size_t)t.U * 8, st));
  if (pl.nseg > 1) {
    uint32_t* w = reinterpret_cast<uint32_t*>(ws + pl.ws_prep);
    P.part_hist = w;
    P.part_sw = w + (size_t)a->n_traces * P.U4;
    P.part_vio = P.part_sw + (pen ? (size_t)a->n_traces * P.NSEG : 0);
    CS_CUDA_TRY(cudaMemsetAsync(w, 0, pl.ws_split, st));
  }
  void* fn = pick_kernel(f32, pen, a->step_bins != nullptr, vio, pl.uni, pl.pk);
  CS_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
  if (!g_ev0) {
    CS_CUDA_TRY(cudaEventCreate(&g_ev0));
    CS_CUDA_TRY(cudaEventCreate(&g_ev1));
  }
  CS_CUDA_TRY(cudaEventRecord(g_ev0, st));
  void* args[] = {(void*)&P};
  CS_CUDA_TRY(cudaLaunchKernel(fn, dim3(pl.ctas), dim3(pl.threads), args, pl.smem, st));
  CS_CUDA_TRY(cudaEventRecord(g_ev1, st));
  g_timed = true;
  ++launches;
  if (pl.nseg > 1) {
    void* ff = pen ? (void*)finalize_kernel<true> : (void*)finalize_kernel<false>;
    int optin = 232448;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const size_t scr = 32 * 24 * 8;
    const bool split = (size_t)P.U4 * 4 + scr <= (size_t)optin;
    const size_t fsm = (split ? (size_t)P.U4 * 4 : 0) + scr;
    P.fin_split = split ? 1 : 0;
    CS_CUDA_TRY(cudaFuncSetAttribute(ff, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm));
    CS_CUDA_TRY(cudaLaunchKernel(ff, dim3((unsigned)a->n_traces, split ? (unsigned)t.M : 1u), dim3(1024), args, fsm,
                                 st));
    ++launches;
  }
  g_last_launches = launches;
  g_last_plan.ctas = pl.ctas;
  g_last_plan.threads = pl.threads;
  g_last_plan.warps_per_group = pl.wpg;
  g_last_plan.smem_bytes = (int32_t)pl.smem;
  g_last_plan.trace_segments = pl.nseg;
  g_last_plan.lut_entries = P.n_lut;
  g_last_plan.lut_shift = (int32_t)P.lv.shift1;
  g_last_plan.epilogue = pl.pk ? (P.seg_smem_bytes > 0 ? 4 : 3) : P.bin_epi ? 2 : (P.seg_smem_bytes > 0 ? 1 : 0);
  g_last_plan.redirect_uniform = (pl.uni && f32 && !pen && a->step_bins == nullptr) ? 1 : 0;
  return std::string();
}

std::string last_kernel_ms(float* ms) {
  if (!g_timed) return "no cs_eval launch on this thread yet";
  CS_CUDA_TRY(cudaEventElapsedTime(ms, g_ev0, g_ev1));
  return std::string();
}

int last_launches() { return g_last_launches; }
cs_eval_plan last_plan() { return g_last_plan; }

}  // namespace cs
