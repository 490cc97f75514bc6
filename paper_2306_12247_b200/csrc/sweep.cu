// Sweep totals: the per-(grid, policy) statistics of a whole Monte Carlo sweep reduced from the
// per-trace aggregates (cs_agg, one per (trace, grid, policy): _aggregate, sim.py:104-127), in a
// form whose cross-GPU reduction is a plain int64 SUM (one NCCL all-reduce, or peer atomics)
// and whose result does not depend on how the traces were sharded.
//
// Per (grid, policy) row, CS_SWEEP_WORDS u64 words (include/capsim_b200.h):
//   [0] steps  [1] idle steps  [2] switched steps  [3] violations
//   [4..7]  sum over traces of avg_throughput_ips, [8..11] sum of energy_proxy_wh, each as an
//           exact 128-bit fixed-point number (LSB 2^-50) split into four 32-bit limbs that are
//           summed independently in u64 (no carries: < 2^32 addends per limb).
// Integer sums are order-independent, so the totals are identical at 1, 2, 4 or 8 GPUs; the host
// recombines the limbs exactly (Python ints) and rounds once.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "cs_internal.h"

namespace cs {
namespace {

#define CS_CUDA_TRY(x)                                                                                  \
  do {                                                                                                  \
    cudaError_t e_ = (x);                                                                               \
    if (e_ != cudaSuccess) return std::string("CUDA error: ") + cudaGetErrorString(e_) + " (" #x ")"; \
  } while (0)

constexpr int kFixedShift = 50;  // LSB 2^-50; values up to 2^78 fit 128 bits

// x >= 0 as 128-bit fixed point m * 2^(e + 50), added limb-wise into l[0..3] (truncates below
// 2^-50: only values < 4 lose bits, deterministically)
__device__ __forceinline__ void add_fixed(unsigned long long (&l)[4], double x) {
  if (!(x > 0.0)) return;
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  int ex = (int)((b >> 52) & 0x7FF);
  unsigned long long m = b & ((1ull << 52) - 1);
  if (ex) m |= 1ull << 52;
  else ex = 1;
  const int sh = ex - 1075 + kFixedShift;
  unsigned long long lo, hi;
  if (sh >= 64) {
    lo = 0;
    hi = m << (sh - 64);
  } else if (sh > 0) {
    lo = m << sh;
    hi = m >> (64 - sh);
  } else if (sh > -64) {
    lo = m >> -sh;
    hi = 0;
  } else {
    lo = hi = 0;
  }
  l[0] += lo & 0xFFFFFFFFull;
  l[1] += lo >> 32;
  l[2] += hi & 0xFFFFFFFFull;
  l[3] += hi >> 32;
}

// One warp per (row, slice of traces): lanes stride over the slice's traces, then a butterfly
// reduction of the CS_SWEEP_WORDS words and one global atomic per nonzero word. Rows run in
// parallel (a one-trace C2 sweep has 30 rows: a block walking them in turn took 39 us).
__global__ void __launch_bounds__(256) sweep_totals_kernel(const cs_agg* __restrict__ agg, int64_t T, int rows,
                                                           int slices, int store, unsigned long long* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= (int64_t)rows * slices) return;
  const int r = (int)(wid % rows), sl = (int)(wid / rows);
  const int64_t per = (T + slices - 1) / slices;
  const int64_t t0 = (int64_t)sl * per, t1 = min(T, t0 + per);
  unsigned long long v[CS_SWEEP_WORDS];
#pragma unroll
  for (int k = 0; k < CS_SWEEP_WORDS; ++k) v[k] = 0ull;
  unsigned long long thr[4] = {0ull, 0ull, 0ull, 0ull}, en[4] = {0ull, 0ull, 0ull, 0ull};
  for (int64_t t = t0 + lane; t < t1; t += 32) {
    const cs_agg a = agg[t * rows + r];
    v[0] += (unsigned long long)a.num_steps;
    v[1] += (unsigned long long)a.idle_steps;
    v[2] += (unsigned long long)a.switches;
    v[3] += (unsigned long long)a.violations;
    add_fixed(thr, a.avg_throughput_ips);
    add_fixed(en, a.energy_proxy_wh);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) v[4 + k] = thr[k], v[8 + k] = en[k];
#pragma unroll
  for (int k = 0; k < CS_SWEEP_WORDS; ++k) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  }
  if (lane < CS_SWEEP_WORDS) {
    unsigned long long x = 0ull;
#pragma unroll
    for (int k = 0; k < CS_SWEEP_WORDS; ++k) x = lane == k ? v[k] : x;
    if (store)  // one slice per row: the warp owns the row (no memset, no atomics)
      out[(size_t)r * CS_SWEEP_WORDS + lane] = x;
    else if (x)
      atomicAdd(out + (size_t)r * CS_SWEEP_WORDS + lane, x);
  }
}

}  // namespace

std::string launch_sweep_totals(const cs_agg* agg, int64_t T, int rows, uint64_t* out, bool accumulate, int sms,
                                cudaStream_t st) {
  if (rows <= 0) return std::string();
  if (T <= 0) {
    if (!accumulate) CS_CUDA_TRY(cudaMemsetAsync(out, 0, (size_t)rows * CS_SWEEP_WORDS * 8, st));
    return std::string();
  }
  // ~8 traces per lane and slice: few enough atomics, enough warps to stream the records
  const int64_t want = (T + 255) / 256;
  const int slices = (int)std::max<int64_t>(1, std::min<int64_t>(want, std::max<int64_t>(1, (int64_t)sms * 64 / rows)));
  const int64_t warps = (int64_t)rows * slices;
  const int store = (slices == 1 && !accumulate) ? 1 : 0;  // small sweeps (C1/C2): one launch, no memset
  if (!store && !accumulate) CS_CUDA_TRY(cudaMemsetAsync(out, 0, (size_t)rows * CS_SWEEP_WORDS * 8, st));
  const int blocks = (int)((warps + 7) / 8);
  sweep_totals_kernel<<<blocks, 256, 0, st>>>(agg, T, rows, slices, store, reinterpret_cast<unsigned long long*>(out));
  CS_CUDA_TRY(cudaGetLastError());
  return std::string();
}

}  // namespace cs
