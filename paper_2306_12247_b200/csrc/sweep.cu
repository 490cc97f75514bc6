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

// One block per slice of traces; rows (grid, policy) in an outer loop; per row every thread sums
// its traces, then a warp + block reduction and CS_SWEEP_WORDS global atomics per block.
__global__ void __launch_bounds__(256) sweep_totals_kernel(const cs_agg* __restrict__ agg, int64_t T, int rows,
                                                           unsigned long long* __restrict__ out) {
  __shared__ unsigned long long red[8][CS_SWEEP_WORDS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t per = (T + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * per, t1 = min(T, t0 + per);
  for (int r = 0; r < rows; ++r) {
    unsigned long long v[CS_SWEEP_WORDS];
#pragma unroll
    for (int k = 0; k < CS_SWEEP_WORDS; ++k) v[k] = 0ull;
    unsigned long long thr[4] = {0ull, 0ull, 0ull, 0ull}, en[4] = {0ull, 0ull, 0ull, 0ull};
    for (int64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
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
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < CS_SWEEP_WORDS; ++k) red[w][k] = v[k];
    __syncthreads();
    if (threadIdx.x < CS_SWEEP_WORDS) {
      unsigned long long s = 0ull;
      for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i][threadIdx.x];
      if (s) atomicAdd(out + (size_t)r * CS_SWEEP_WORDS + threadIdx.x, s);
    }
    __syncthreads();
  }
}

}  // namespace

std::string launch_sweep_totals(const cs_agg* agg, int64_t T, int rows, uint64_t* out, bool accumulate, int sms,
                                cudaStream_t st) {
  if (!accumulate) CS_CUDA_TRY(cudaMemsetAsync(out, 0, (size_t)rows * CS_SWEEP_WORDS * 8, st));
  if (T <= 0 || rows <= 0) return std::string();
  // ~8 traces per thread per row: few enough atomics, enough blocks to stream the records
  const int64_t want = (T + 2047) / 2048;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8));
  sweep_totals_kernel<<<blocks, 256, 0, st>>>(agg, T, rows, reinterpret_cast<unsigned long long*>(out));
  CS_CUDA_TRY(cudaGetLastError());
  return std::string();
}

}  // namespace cs
