// B200 (sm_100a) kernels of the trace-driven policy-evaluation path.
//
//   eval_kernel      N2+N3: streams caps from HBM with 128-bit loads, maps every cap to its
//                    union threshold bin through the shared-memory LUT (one search serves all
//                    grids x 3 policies), and accumulates a per-trace bin histogram in shared
//                    memory. At the end of each trace a fused epilogue turns the histogram into
//                    the SimReport aggregates (sim.py:104-127) with double-double sums (so the
//                    average matches the reference's math.fsum to the last bit in practice), and
//                    folds the histogram into the global config histogram.
//   finalize_kernel  epilogue for traces that were split across several worker groups.
//   select_kernel    select_config (policy.py:172-188): warp-per-cap argmax via shuffles.
//   feasible_kernel  feasible_set (policy.py:151-169): warp-per-cap ballot bitmask.
//   gen_kernel       synthetic solar / wind / iid cap traces (counter-based RNG).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>

#include "cs_internal.h"

namespace cs {

// ----------------------------------------------------------------------------------------
// helpers
// ----------------------------------------------------------------------------------------
__device__ __forceinline__ uint4 ldg_stream_u4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

struct dd {
  double hi, lo;
};
// Error-free transformations (no contraction: explicit _rn intrinsics).
__device__ __forceinline__ void dd_add2(dd& x, double p, double pe) {
  double s = __dadd_rn(x.hi, p);
  double bb = __dsub_rn(s, x.hi);
  double e = __dadd_rn(__dsub_rn(x.hi, __dsub_rn(s, bb)), __dsub_rn(p, bb));
  e = __dadd_rn(e, __dadd_rn(x.lo, pe));
  double h = __dadd_rn(s, e);
  x.lo = __dsub_rn(e, __dsub_rn(h, s));
  x.hi = h;
}
__device__ __forceinline__ void dd_add_prod(dd& x, double c, double v) {
  double p = __dmul_rn(c, v);
  double pe = __fma_rn(c, v, -p);
  dd_add2(x, p, pe);
}
__device__ __forceinline__ double shfl_d(double v, int lane_mask) {
  return __shfl_xor_sync(0xffffffffu, v, lane_mask);
}

template <typename CapT>
struct CapTraits;
template <>
struct CapTraits<float> {
  using Bits = uint32_t;
  static constexpr int VEC = 4;
};
template <>
struct CapTraits<double> {
  using Bits = uint64_t;
  static constexpr int VEC = 2;
};

// ----------------------------------------------------------------------------------------
// evaluation kernel
// ----------------------------------------------------------------------------------------
struct EvalParams {
  DevTables tb;
  const void* caps;
  int64_t T, S, ld;
  int64_t seg_len;
  int32_t nseg;
  int32_t step_seconds;
  double omp;  // 1 - penalty_frac
  uint16_t* step_bins;
  int64_t ld_bins;
  cs_agg* agg;
  uint64_t* hist;
  // split mode partials (global)
  uint32_t* part_hist;  // [T][U]
  uint32_t* part_sw;    // [T][M*3][U]
  uint32_t* part_vio;   // [T][M*3]
  int32_t wpg;          // warps per group
  int32_t gpc;          // groups per CTA
  int32_t lut_smem;     // LUT copied to shared memory
  // shared-memory layout (bytes)
  int32_t off_vio, off_sig, off_ghist, off_groups, group_bytes;
  int32_t off_g_sw, off_g_vio, off_g_scr;  // within a group
};

template <bool CHECK>
__device__ __forceinline__ void group_sync(int gid_local, int gsize) {
  if (gsize == 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + gid_local), "r"(gsize) : "memory");
  }
}

// Per-trace epilogue over one group's histogram (sim.py:104-127 for every grid x policy).
// h: [U] step counts per union bin; sw: [M*3][U] switched-step counts (PEN only);
// vcnt: [M*3] violation counts. Writes agg[t][m][p]. One (grid, policy) pass at a time keeps
// the register footprint small (the hot loop shares the kernel).
template <bool PEN>
__device__ __noinline__ void epilogue(const EvalParams& P, int64_t t, const uint32_t* h, const uint32_t* sw,
                                      const uint32_t* vcnt, double* scratch, int gtid, int gsize, int gid_local) {
  const DevTables& tb = P.tb;
  const int U = tb.U, M = tb.M, maxB = tb.maxB;
  const int lane = gtid & 31, wig = gtid >> 5, nw = gsize >> 5;
  const double step = (double)P.step_seconds;
  for (int mp = 0; mp < M * 3; ++mp) {
    const int m = mp / 3;
    dd thr{0.0, 0.0}, en{0.0, 0.0};
    long long idle = 0, swc = 0;
    const double idle_e = __ddiv_rn(__dmul_rn(tb.idle_pw[m], step), 3600.0);
    const size_t ob = (size_t)mp * maxB;
    for (int u = gtid; u < U; u += gsize) {
      const uint32_t c = h[u];
      if (c == 0) continue;
      const int r = (M > 1) ? (int)tb.umap[(size_t)m * U + u] : u;
      const int32_t sel = __ldg(tb.sel + ob + r);
      const uint32_t s = PEN ? sw[(size_t)mp * U + u] : 0u;
      swc += s;
      if (sel < 0) {
        idle += c;
        dd_add_prod(en, (double)c, idle_e);
      } else {
        const double th = __ldg(tb.sthr + ob + r);
        const double pw = __ldg(tb.spw + ob + r);
        dd_add_prod(thr, (double)(c - s), th);
        if (PEN && s) dd_add_prod(thr, (double)s, __dmul_rn(th, P.omp));
        dd_add_prod(en, (double)c, __ddiv_rn(__dmul_rn(pw, step), 3600.0));
      }
    }
#pragma unroll
    for (int k = 16; k >= 1; k >>= 1) {
      double a = shfl_d(thr.hi, k), b = shfl_d(thr.lo, k);
      dd_add2(thr, a, b);
      a = shfl_d(en.hi, k), b = shfl_d(en.lo, k);
      dd_add2(en, a, b);
      idle += __shfl_xor_sync(0xffffffffu, idle, k);
      swc += __shfl_xor_sync(0xffffffffu, swc, k);
    }
    if (nw > 1) {
      if (lane == 0) {
        double* d = scratch + wig * 6;
        d[0] = thr.hi;
        d[1] = thr.lo;
        d[2] = en.hi;
        d[3] = en.lo;
        d[4] = __longlong_as_double(idle);
        d[5] = __longlong_as_double(swc);
      }
      group_sync<true>(gid_local, gsize);
      if (gtid == 0) {
        for (int w = 1; w < nw; ++w) {
          const double* d = scratch + w * 6;
          dd_add2(thr, d[0], d[1]);
          dd_add2(en, d[2], d[3]);
          idle += __double_as_longlong(d[4]);
          swc += __double_as_longlong(d[5]);
        }
      }
      group_sync<true>(gid_local, gsize);
    }
    if (gtid == 0 && P.agg) {
      cs_agg a;
      a.avg_throughput_ips = __ddiv_rn(__dadd_rn(thr.hi, thr.lo), (double)P.S);
      a.energy_proxy_wh = __dadd_rn(en.hi, en.lo);
      a.idle_steps = idle;
      a.switches = swc;
      a.violations = vcnt ? vcnt[mp] : 0;
      a.num_steps = P.S;
      P.agg[t * M * 3 + mp] = a;
    }
  }
}

template <typename CapT, bool PEN, bool STEP, bool VIO>
__global__ void __launch_bounds__(512) eval_kernel(const __grid_constant__ EvalParams P) {
  using Bits = typename CapTraits<CapT>::Bits;
  constexpr int VEC = CapTraits<CapT>::VEC;
  constexpr int UNR = (VEC == 4) ? 4 : 4;
  extern __shared__ __align__(16) unsigned char smem[];
  const DevTables& tb = P.tb;
  const int U = tb.U, M = tb.M;

  // ---- stage tables into shared memory (N1: once per CTA) ----
  const uint32_t* lut = tb.lv.lut;
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(smem);
  if (P.lut_smem) {
    for (int i = threadIdx.x; i < tb.n_lut; i += blockDim.x) s_lut[i] = __ldg(tb.lv.lut + i);
    lut = s_lut;
  }
  Bits* s_vio = reinterpret_cast<Bits*>(smem + P.off_vio);
  if (VIO)
    for (int i = threadIdx.x; i < U; i += blockDim.x) s_vio[i] = (Bits)__ldg(tb.vio + i);
  uint64_t* s_sig = reinterpret_cast<uint64_t*>(smem + P.off_sig);
  if (PEN)
    for (int i = threadIdx.x; i < M * U; i += blockDim.x) s_sig[i] = __ldg(tb.sig + i);
  unsigned long long* s_ghist = reinterpret_cast<unsigned long long*>(smem + P.off_ghist);
  const bool want_hist = P.hist != nullptr && P.nseg == 1;
  if (want_hist)
    for (int i = threadIdx.x; i < U; i += blockDim.x) s_ghist[i] = 0ull;

  const int gsize = P.wpg * 32;
  const int gid_local = threadIdx.x / gsize;
  const int gtid = threadIdx.x % gsize;
  unsigned char* gbase = smem + P.off_groups + (size_t)gid_local * P.group_bytes;
  uint32_t* h = reinterpret_cast<uint32_t*>(gbase);
  uint32_t* sw = reinterpret_cast<uint32_t*>(gbase + P.off_g_sw);
  uint32_t* vcnt = reinterpret_cast<uint32_t*>(gbase + P.off_g_vio);
  double* scratch = reinterpret_cast<double*>(gbase + P.off_g_scr);
  for (int i = gtid; i < U; i += gsize) h[i] = 0u;
  if (PEN)
    for (int i = gtid; i < M * 3 * U; i += gsize) sw[i] = 0u;
  if (gtid < M * 3) vcnt[gtid] = 0u;
  __syncthreads();

  const int32_t lo32 = (int32_t)tb.lv.lo, hi32 = (int32_t)tb.lv.hi;
  const uint32_t s1 = tb.lv.shift1, sub0 = tb.lv.sub0;
  const uint32_t kb32 = (uint32_t)tb.lv.kbase;

  auto bin_of = [&](Bits b) -> uint32_t {
    if constexpr (VEC == 4)
      return bin_f32((uint32_t)b, lo32, hi32, s1, kb32, sub0, lut);
    else
      return bin_f64((uint64_t)b, tb.lv.lo, tb.lv.hi, s1, tb.lv.kbase, sub0, lut, tb.lv.thr64);
  };
  auto clampb = [&](Bits b) -> Bits {
    if constexpr (VEC == 4)
      return (Bits)clamp_bits_f32((uint32_t)b, lo32, hi32);
    else
      return (Bits)clamp_bits_f64((uint64_t)b, tb.lv.lo, tb.lv.hi);
  };

  const int64_t n_items = P.T * (int64_t)P.nseg;
  const int64_t n_groups = (int64_t)gridDim.x * P.gpc;
  for (int64_t item = (int64_t)blockIdx.x * P.gpc + gid_local; item < n_items; item += n_groups) {
    const int64_t t = item / P.nseg;
    const int64_t seg = item - t * P.nseg;
    const int64_t s0 = seg * P.seg_len;
    const int64_t s1e = min(P.S, s0 + P.seg_len);
    const CapT* row = reinterpret_cast<const CapT*>(P.caps) + t * P.ld;
    const int64_t nvec = (s1e - s0 + VEC - 1) / VEC;
    const unsigned char* vrow = reinterpret_cast<const unsigned char*>(row + s0);

    auto process = [&](const uint4 raw, int64_t i0) {
      Bits x[VEC];
      if constexpr (VEC == 4) {
        x[0] = raw.x; x[1] = raw.y; x[2] = raw.z; x[3] = raw.w;
      } else {
        x[0] = ((uint64_t)raw.y << 32) | raw.x;
        x[1] = ((uint64_t)raw.w << 32) | raw.z;
      }
      const bool full = i0 + VEC <= s1e;
      uint32_t b[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        b[e] = bin_of(x[e]);
        if (!full && i0 + e >= s1e) continue;
        atomicAdd(&h[b[e]], 1u);
        if (VIO) {
          if (clampb(x[e]) < s_vio[b[e]]) {
            // slow path: re-check every (grid, policy) selection against the cap in fp64
            double cap;
            if constexpr (VEC == 4) cap = (double)__uint_as_float((uint32_t)x[e]);
            else cap = __longlong_as_double((long long)x[e]);
            for (int m = 0; m < M; ++m) {
              const int r = (M > 1) ? (int)tb.umap[(size_t)m * U + b[e]] : (int)b[e];
              for (int p = 0; p < 3; ++p) {
                const size_t o = ((size_t)m * 3 + p) * tb.maxB + r;
                if (tb.sel[o] >= 0 && tb.spw[o] > cap) atomicAdd(&vcnt[m * 3 + p], 1u);
              }
            }
          }
        }
      }
      if (PEN) {
        uint32_t pb;
        if (i0 == 0) {
          pb = b[0];  // step 0 is never penalised (sim.py:119: i > 0)
        } else {
          Bits prev;
          if constexpr (VEC == 4) prev = __ldg(reinterpret_cast<const uint32_t*>(row) + i0 - 1);
          else prev = __ldg(reinterpret_cast<const unsigned long long*>(row) + i0 - 1);
          pb = bin_of(prev);
        }
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          if (!full && i0 + e >= s1e) break;
          const uint32_t cb = b[e];
          if (cb != pb) {
            for (int m = 0; m < M; ++m) {
              const uint64_t xo = s_sig[(size_t)m * U + cb] ^ s_sig[(size_t)m * U + pb];
              for (int p = 0; p < 3; ++p)
                if ((xo >> (16 * p)) & 0xFFFFull) atomicAdd(&sw[((size_t)m * 3 + p) * U + cb], 1u);
            }
          }
          pb = cb;
        }
      }
      if (STEP) {
        uint16_t* out = P.step_bins + t * P.ld_bins + i0;
        if (full) {
          if constexpr (VEC == 4) {
            uint2 v;
            v.x = (b[0] & 0xFFFFu) | (b[1] << 16);
            v.y = (b[2] & 0xFFFFu) | (b[3] << 16);
            *reinterpret_cast<uint2*>(out) = v;
          } else {
            *reinterpret_cast<uint32_t*>(out) = (b[0] & 0xFFFFu) | (b[1] << 16);
          }
        } else {
          for (int e = 0; e < VEC; ++e)
            if (i0 + e < s1e) out[e] = (uint16_t)b[e];
        }
      }
    };

    for (int64_t v = gtid; v < nvec; v += (int64_t)gsize * UNR) {
      uint4 raw[UNR];
#pragma unroll
      for (int k = 0; k < UNR; ++k) {
        const int64_t vi = v + (int64_t)k * gsize;
        if (vi < nvec) raw[k] = ldg_stream_u4(vrow + vi * 16);
      }
#pragma unroll
      for (int k = 0; k < UNR; ++k) {
        const int64_t vi = v + (int64_t)k * gsize;
        if (vi < nvec) process(raw[k], s0 + vi * VEC);
      }
    }
    group_sync<true>(gid_local, gsize);

    if (P.nseg == 1) {
      epilogue<PEN>(P, t, h, sw, vcnt, scratch, gtid, gsize, gid_local);
      group_sync<true>(gid_local, gsize);
      for (int u = gtid; u < U; u += gsize) {
        const uint32_t c = h[u];
        if (c) {
          if (want_hist) atomicAdd(&s_ghist[u], (unsigned long long)c);
          h[u] = 0u;
          if (PEN)
            for (int mp = 0; mp < M * 3; ++mp) sw[(size_t)mp * U + u] = 0u;
        }
      }
    } else {
      // split trace: fold this segment's partial histogram into the trace's global partials
      for (int u = gtid; u < U; u += gsize) {
        const uint32_t c = h[u];
        if (c) {
          atomicAdd(&P.part_hist[t * U + u], c);
          h[u] = 0u;
          if (PEN)
            for (int mp = 0; mp < M * 3; ++mp) {
              const uint32_t s = sw[(size_t)mp * U + u];
              if (s) {
                atomicAdd(&P.part_sw[(t * M * 3 + mp) * U + u], s);
                sw[(size_t)mp * U + u] = 0u;
              }
            }
        }
      }
      if (gtid < M * 3 && vcnt[gtid]) atomicAdd(&P.part_vio[t * M * 3 + gtid], vcnt[gtid]);
    }
    group_sync<true>(gid_local, gsize);
    if (gtid < M * 3) vcnt[gtid] = 0u;
    group_sync<true>(gid_local, gsize);
  }

  if (want_hist) {
    __syncthreads();
    for (int u = threadIdx.x; u < U; u += blockDim.x) {
      const unsigned long long c = s_ghist[u];
      if (c) atomicAdd(reinterpret_cast<unsigned long long*>(P.hist) + u, c);
    }
  }
}

// Epilogue for split traces: one CTA per trace, histogram read from the global partials.
template <bool PEN>
__global__ void __launch_bounds__(256) finalize_kernel(const __grid_constant__ EvalParams P) {
  __shared__ double scratch[8 * 6];
  const int64_t t = blockIdx.x;
  const int U = P.tb.U, M = P.tb.M;
  uint32_t* h = P.part_hist + t * U;
  uint32_t* sw = PEN ? P.part_sw + t * (int64_t)M * 3 * U : nullptr;
  uint32_t* vc = P.part_vio + t * (int64_t)M * 3;
  epilogue<PEN>(P, t, h, sw, vc, scratch, threadIdx.x, blockDim.x, 0);
  if (P.hist) {
    for (int u = threadIdx.x; u < U; u += blockDim.x) {
      const uint32_t c = h[u];
      if (c) atomicAdd(reinterpret_cast<unsigned long long*>(P.hist) + u, (unsigned long long)c);
    }
  }
}

// ----------------------------------------------------------------------------------------
// per-cap kernels (select_config / feasible_set)
// ----------------------------------------------------------------------------------------
__device__ __forceinline__ bool regime_ok(int p, int mtl, int bs, int bmtl, int mbs) {
  return p == CS_BATCHING ? mtl == bmtl : (p == CS_MULTI_TENANT ? bs == mbs : true);
}

// _prefer (policy.py:90-97): a preferred over b
__device__ __forceinline__ bool prefer_dev(double ta, double pa, int ma, int ba, double tb_, double pb, int mb,
                                           int bb) {
  if (ta != tb_) return ta > tb_;
  if (pa != pb) return pa < pb;
  if (ma != mb) return ma < mb;
  return ba <= bb;
}

__global__ void select_kernel(const DevTables tb, int g, int p, const double* __restrict__ caps, int64_t n,
                              int32_t* __restrict__ sel_out, int64_t* __restrict__ cnt_out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int e0 = tb.e_off[g], ne = tb.e_off[g + 1] - e0;
  for (int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < n; q += warps) {
    double cap = caps[q];
    if (cap != cap) cap = INFINITY;  // bisect_right quirk: a NaN cap bisects to the end
    int best = -1, cnt = 0;
    double bt = 0, bp = 0;
    int bm = 0, bbs = 0;
    for (int j = lane; j < ne; j += 32) {
      const int mtl = tb.e_mtl[e0 + j], bs = tb.e_bs[e0 + j];
      const double pw = tb.e_pw[e0 + j], th = tb.e_thr[e0 + j];
      if (!regime_ok(p, mtl, bs, tb.batching_mtl, tb.mt_bs) || !(pw <= cap)) continue;
      ++cnt;
      if (best < 0 || !prefer_dev(bt, bp, bm, bbs, th, pw, mtl, bs)) {
        best = j, bt = th, bp = pw, bm = mtl, bbs = bs;
      }
    }
    // warp argmax over (throughput desc, power asc, mtl asc, bs asc) with butterfly shuffles
#pragma unroll
    for (int k = 16; k >= 1; k >>= 1) {
      const int ob = __shfl_xor_sync(0xffffffffu, best, k);
      const double ot = __shfl_xor_sync(0xffffffffu, bt, k), op = __shfl_xor_sync(0xffffffffu, bp, k);
      const int om = __shfl_xor_sync(0xffffffffu, bm, k), obs = __shfl_xor_sync(0xffffffffu, bbs, k);
      if (ob >= 0 && (best < 0 || !prefer_dev(bt, bp, bm, bbs, ot, op, om, obs))) {
        best = ob, bt = ot, bp = op, bm = om, bbs = obs;
      }
    }
    const int total = __reduce_add_sync(0xffffffffu, cnt);
    if (lane == 0) {
      sel_out[q] = best;
      cnt_out[q] = total;
    }
  }
}

__global__ void feasible_kernel(const DevTables tb, int g, int p, const double* __restrict__ caps, int64_t n,
                                uint32_t* __restrict__ mask_out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int e0 = tb.e_off[g], ne = tb.e_off[g + 1] - e0;
  const int words = (ne + 31) / 32;
  for (int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < n; q += warps) {
    const double cap = caps[q];  // literal `power_w <= cap_w` (policy.py:169): NaN admits nothing
    for (int w = 0; w < words; ++w) {
      const int j = w * 32 + lane;
      bool f = false;
      if (j < ne) f = regime_ok(p, tb.e_mtl[e0 + j], tb.e_bs[e0 + j], tb.batching_mtl, tb.mt_bs) &&
                      tb.e_pw[e0 + j] <= cap;
      const uint32_t m = __ballot_sync(0xffffffffu, f);
      if (lane == 0) mask_out[q * words + w] = m;
    }
  }
}

// ----------------------------------------------------------------------------------------
// synthetic traces
// ----------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ float u01(uint64_t h) { return (float)(h >> 40) * (1.0f / 16777216.0f); }
__device__ __forceinline__ float gauss(uint64_t h) {
  // Irwin-Hall(4), rescaled to unit variance: cheap and bounded
  float s = u01(h) + u01(h * 0x9E3779B97F4A7C15ull) + u01(splitmix(h)) + u01(splitmix(h ^ 0xABCDull));
  return (s - 2.0f) * 1.7320508f;
}

// One warp generates 32 traces (a lane each, sequential in time) and writes 32x32 tiles
// transposed through shared memory so every store is a coalesced 128-byte row segment.
__global__ void gen_kernel(float* caps, int64_t T, int64_t S, int64_t ld, int64_t first_id, int32_t step_seconds,
                           int32_t kind, float peak, uint64_t seed) {
  __shared__ float tile[8][32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t t0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + w) * 32;
  if (t0 >= T) return;
  const int64_t tid = first_id + t0 + lane;
  const uint64_t hk = splitmix(seed ^ splitmix((uint64_t)tid));
  int k = kind;
  if (k == CS_TRACE_MIXED) k = (tid & 1) ? CS_TRACE_WIND : CS_TRACE_SOLAR;
  // per-trace parameters
  const float var = 0.1f + 0.7f * u01(splitmix(hk ^ 1));           // Table-1 variation range 10%..80%
  const float phase = 86400.0f * u01(splitmix(hk ^ 2));            // start time of day offset
  const float dt = (float)step_seconds;
  const float a_cloud = __expf(-dt / 3600.0f);                      // 1 h cloud correlation time
  const float wind_mu = 5.0f + 5.0f * u01(splitmix(hk ^ 3));       // mean wind speed (m/s)
  const float theta = 1.0f / 7200.0f;                               // OU mean reversion (1/s)
  float cloud = 0.6f, wind = wind_mu;
  for (int64_t s0 = 0; s0 < S; s0 += 32) {
    for (int j = 0; j < 32; ++j) {
      const int64_t s = s0 + j;
      const uint64_t hs = splitmix(hk ^ (uint64_t)(s * 0x632BE59BD9B4E019ull));
      float v;
      if (k == CS_TRACE_IID) {
        v = peak * u01(hs);
      } else if (k == CS_TRACE_SOLAR) {
        const float tod = fmodf(phase + (float)s * dt, 86400.0f) / 3600.0f;
        const float clear = (tod > 6.0f && tod < 18.0f) ? __sinf(3.14159265f * (tod - 6.0f) / 12.0f) : 0.0f;
        cloud = a_cloud * cloud + (1.0f - a_cloud) * 0.7f +
                var * 0.5f * sqrtf(fmaxf(1.0f - a_cloud * a_cloud, 1e-6f)) * gauss(hs);
        cloud = fminf(fmaxf(cloud, 0.2f), 1.0f);
        v = peak * clear * cloud;
      } else {
        const float sdt = fminf(theta * dt, 1.0f);
        wind = wind + sdt * (wind_mu - wind) + var * 4.0f * sqrtf(2.0f * sdt) * gauss(hs);
        wind = fmaxf(wind, 0.0f);
        float f = 0.0f;
        if (wind >= 3.0f && wind < 25.0f) f = wind >= 12.0f ? 1.0f : powf((wind - 3.0f) / 9.0f, 3.0f);
        v = peak * f;
      }
      tile[w][lane][j] = fminf(fmaxf(v, 0.0f), peak);
    }
    __syncwarp();
    for (int r = 0; r < 32; ++r) {
      const int64_t tr = t0 + r;
      const int64_t s = s0 + lane;
      if (tr < T && s < S) caps[tr * ld + s] = tile[w][r][lane];
    }
    __syncwarp();
  }
}

// ----------------------------------------------------------------------------------------
// host-side launchers
// ----------------------------------------------------------------------------------------
namespace {
thread_local cudaEvent_t g_ev0 = nullptr, g_ev1 = nullptr;
thread_local int g_last_launches = 0;
thread_local bool g_timed = false;

#define CS_CUDA_TRY(x)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) return std::string("CUDA error: ") + cudaGetErrorString(e_) + " (" #x ")"; \
  } while (0)

struct Plan {
  int threads, wpg, gpc, ctas;
  int32_t nseg;
  int64_t seg_len;
  size_t smem;
  EvalParams P;
};

int sm_count(int dev) {
  static int cache[64] = {0};
  if (dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev);
  return cache[dev];
}

template <typename CapT, bool PEN, bool STEP, bool VIO>
void* kernel_ptr() {
  return (void*)eval_kernel<CapT, PEN, STEP, VIO>;
}

using KFn = void*;
KFn pick_kernel(bool f32, bool pen, bool step, bool vio) {
#define CS_K(F, A, B, C) \
  if (pen == A && step == B && vio == C) return f32 ? kernel_ptr<float, A, B, C>() : kernel_ptr<double, A, B, C>();
  CS_K(f, false, false, false)
  CS_K(f, false, false, true)
  CS_K(f, false, true, false)
  CS_K(f, false, true, true)
  CS_K(f, true, false, false)
  CS_K(f, true, false, true)
  CS_K(f, true, true, false)
  CS_K(f, true, true, true)
#undef CS_K
  return nullptr;
}

}  // namespace

size_t split_workspace_bytes(const Tables& t, int64_t T, bool pen) {
  return (size_t)T * ((size_t)t.U + (pen ? (size_t)t.M * 3 * t.U : 0) + (size_t)t.M * 3) * sizeof(uint32_t);
}

// Chooses the launch geometry: worker-group size (warps sharing one histogram) and CTAs per SM.
static std::string make_plan(const Tables& t, const DevTables& view, const cs_eval_args* a, int dev, Plan& pl,
                             bool for_size_only) {
  const bool f32 = t.cap_dtype == CS_CAP_F32;
  const bool pen = a->switch_penalty_s > 0.0;
  const bool vio = (a->flags & CS_FLAG_CHECK_VIOLATIONS) != 0;
  void* fn = pick_kernel(f32, pen, a->step_bins != nullptr, vio);
  const int U = t.U, M = t.M;
  int smem_optin = 232448;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int nsm = sm_count(dev);
  const size_t bits_sz = f32 ? 4 : 8;
  const size_t lut_bytes = ((size_t)t.lut.size() * 4 + 15) & ~(size_t)15;
  size_t fixed_nolut = 0;
  const size_t off_vio_rel = 0;
  fixed_nolut += vio ? (((size_t)U * bits_sz + 15) & ~(size_t)15) : 0;
  const size_t off_sig_rel = fixed_nolut;
  fixed_nolut += pen ? (size_t)M * U * 8 : 0;
  const size_t off_ghist_rel = fixed_nolut;
  fixed_nolut += a->hist ? (size_t)U * 8 : 0;
  fixed_nolut = (fixed_nolut + 15) & ~(size_t)15;

  // candidate geometries: prefer the most resident warps per SM, then the smallest group
  struct Cand {
    int threads, wpg, ctas_per_sm, lut_smem;
    size_t smem;
  };
  Cand best{0, 0, 0, 0, 0};
  int best_warps = -1;
  for (int lut_smem = 1; lut_smem >= 0; --lut_smem) {
    for (int threads : {512, 256, 128}) {
      for (int wpg : {1, 2, 4, 8, 16, 32}) {
        const int wpc = threads / 32;
        if (wpg > wpc) continue;
        const int gpc = wpc / wpg;
        if (wpg > 1 && gpc > 15) continue;  // named barriers 1..15
        size_t gb = (size_t)U * 4;
        const size_t off_sw = gb;
        gb += pen ? (size_t)M * 3 * U * 4 : 0;
        const size_t off_v = gb;
        gb += (size_t)M * 3 * 4;
        gb = (gb + 7) & ~(size_t)7;
        gb += (size_t)wpg * 6 * 8;
        gb = (gb + 15) & ~(size_t)15;
        (void)off_sw;
        (void)off_v;
        const size_t smem = (lut_smem ? lut_bytes : 0) + fixed_nolut + (size_t)gpc * gb;
        if (smem > (size_t)smem_optin) continue;
        int per_sm = 0;
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess) {
          cudaGetLastError();
          continue;
        }
        if (per_sm < 1) continue;
        const int warps = per_sm * wpc;
        if (warps > best_warps || (warps == best_warps && wpg < best.wpg)) {
          best_warps = warps;
          best = Cand{threads, wpg, per_sm, lut_smem, smem};
        }
      }
    }
    if (best_warps >= 16) break;  // LUT fits in shared memory with reasonable occupancy
  }
  if (best_warps < 0) return "tables too large for shared memory (union bins " + std::to_string(U) + ")";

  pl.threads = best.threads;
  pl.wpg = best.wpg;
  pl.gpc = best.threads / 32 / best.wpg;
  const int64_t groups_total = (int64_t)nsm * best.ctas_per_sm * pl.gpc;
  // split traces when there are too few of them to occupy every worker group
  int64_t nseg = 1;
  if (a->n_traces < 2 * groups_total) {
    const int64_t want = (2 * groups_total + a->n_traces - 1) / std::max<int64_t>(a->n_traces, 1);
    const int64_t max_seg = std::max<int64_t>(1, a->n_steps / 2048);
    nseg = std::max<int64_t>(1, std::min(want, max_seg));
  }
  int64_t seg_len = (a->n_steps + nseg - 1) / nseg;
  seg_len = (seg_len + 127) / 128 * 128;
  nseg = (a->n_steps + seg_len - 1) / seg_len;
  pl.nseg = (int32_t)nseg;
  pl.seg_len = seg_len;
  const int64_t items = a->n_traces * nseg;
  pl.ctas = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)nsm * best.ctas_per_sm, (items + pl.gpc - 1) / pl.gpc));
  pl.smem = best.smem;

  EvalParams& P = pl.P;
  P = EvalParams{};
  P.tb = view;
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
    const double pf = pen_s / step;
    P.omp = 1.0 - pf;
  }
  P.step_bins = a->step_bins;
  P.ld_bins = a->ld_bins;
  P.agg = a->agg;
  P.hist = a->hist;
  P.wpg = pl.wpg;
  P.gpc = pl.gpc;
  P.lut_smem = best.lut_smem;
  const size_t lut_part = best.lut_smem ? lut_bytes : 0;
  P.off_vio = (int32_t)(lut_part + off_vio_rel);
  P.off_sig = (int32_t)(lut_part + off_sig_rel);
  P.off_ghist = (int32_t)(lut_part + off_ghist_rel);
  P.off_groups = (int32_t)(lut_part + fixed_nolut);
  {
    size_t gb = (size_t)U * 4;
    P.off_g_sw = (int32_t)gb;
    gb += pen ? (size_t)M * 3 * U * 4 : 0;
    P.off_g_vio = (int32_t)gb;
    gb += (size_t)M * 3 * 4;
    gb = (gb + 7) & ~(size_t)7;
    P.off_g_scr = (int32_t)gb;
    gb += (size_t)pl.wpg * 6 * 8;
    gb = (gb + 15) & ~(size_t)15;
    P.group_bytes = (int32_t)gb;
  }
  (void)for_size_only;
  return std::string();
}

std::string eval_workspace(const Tables& t, const DevTables& view, const cs_eval_args* a, int dev, size_t* bytes) {
  Plan pl;
  std::string err = make_plan(t, view, a, dev, pl, true);
  if (!err.empty()) return err;
  *bytes = pl.nseg > 1 ? split_workspace_bytes(t, a->n_traces, a->switch_penalty_s > 0.0) : 0;
  return std::string();
}

std::string launch_eval(const Tables& t, const DevTables& view, const cs_eval_args* a, int dev, cudaStream_t st) {
  Plan pl;
  std::string err = make_plan(t, view, a, dev, pl, false);
  if (!err.empty()) return err;
  const bool f32 = t.cap_dtype == CS_CAP_F32;
  const bool pen = a->switch_penalty_s > 0.0;
  const bool step = a->step_bins != nullptr;
  const bool vio = (a->flags & CS_FLAG_CHECK_VIOLATIONS) != 0;
  EvalParams& P = pl.P;
  int launches = 0;
  if (a->hist && !(a->flags & CS_FLAG_ACCUMULATE_HIST)) {
    CS_CUDA_TRY(cudaMemsetAsync(a->hist, 0, (size_t)t.U * 8, st));
  }
  if (pl.nseg > 1) {
    const size_t need = split_workspace_bytes(t, a->n_traces, pen);
    if (a->workspace == nullptr || a->workspace_bytes < need)
      return "workspace too small: need " + std::to_string(need) + " bytes (cs_eval_workspace_size)";
    uint32_t* ws = reinterpret_cast<uint32_t*>(a->workspace);
    P.part_hist = ws;
    P.part_sw = ws + (size_t)a->n_traces * t.U;
    P.part_vio = P.part_sw + (pen ? (size_t)a->n_traces * t.M * 3 * t.U : 0);
    CS_CUDA_TRY(cudaMemsetAsync(ws, 0, need, st));
  }
  void* fn = pick_kernel(f32, pen, step, vio);
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
    CS_CUDA_TRY(cudaLaunchKernel(ff, dim3((unsigned)a->n_traces), dim3(256), args, 0, st));
    ++launches;
  }
  g_last_launches = launches;
  return std::string();
}

std::string last_kernel_ms(float* ms) {
  if (!g_timed) return "no cs_eval launch on this thread yet";
  CS_CUDA_TRY(cudaEventElapsedTime(ms, g_ev0, g_ev1));
  return std::string();
}
int last_launches() { return g_last_launches; }

std::string launch_select(const DevTables& v, int g, int p, const double* caps, int64_t n, int32_t* sel, int64_t* cnt,
                          cudaStream_t st) {
  if (n <= 0) return std::string();
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((n + 7) / 8, 148 * 32);
  select_kernel<<<(unsigned)blocks, threads, 0, st>>>(v, g, p, caps, n, sel, cnt);
  CS_CUDA_TRY(cudaGetLastError());
  g_last_launches = 1;
  return std::string();
}

std::string launch_feasible(const DevTables& v, int g, int p, const double* caps, int64_t n, uint32_t* mask,
                            cudaStream_t st) {
  if (n <= 0) return std::string();
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((n + 7) / 8, 148 * 32);
  feasible_kernel<<<(unsigned)blocks, threads, 0, st>>>(v, g, p, caps, n, mask);
  CS_CUDA_TRY(cudaGetLastError());
  g_last_launches = 1;
  return std::string();
}

std::string launch_generate(float* caps, int64_t T, int64_t S, int64_t ld, int64_t first_id, int32_t step_seconds,
                            int32_t kind, float peak, uint64_t seed, cudaStream_t st) {
  if (T <= 0 || S <= 0) return std::string();
  const int64_t warps = (T + 31) / 32;
  const int64_t blocks = (warps + 7) / 8;
  gen_kernel<<<(unsigned)blocks, 256, 0, st>>>(caps, T, S, ld, first_id, step_seconds, kind, peak, seed);
  CS_CUDA_TRY(cudaGetLastError());
  return std::string();
}

}  // namespace cs
