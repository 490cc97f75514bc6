// B200 (sm_100a) kernels of the trace-driven policy-evaluation path.
//
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
namespace {
#define CS_CUDA_TRY(x)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) return std::string("CUDA error: ") + cudaGetErrorString(e_) + " (" #x ")"; \
  } while (0)
}  // namespace

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

// Clear-sky curve sin(pi * x) on [0, 1] as cos(pi * w / 2), w = 2x - 1, by its Taylor polynomial
// in z = w^2 through z^5 (|error| < 5e-7): only IEEE fp32 multiplies and adds (the build uses
// -fmad=false), so the host restatement (oracle/capsim_oracle.c: ora_generate_traces) reproduces
// every sample bit for bit.
__device__ __forceinline__ float clear_sky(float x) {
  const float w = 2.0f * x - 1.0f, z = w * w;
  float p = -2.52020424e-05f;          // (-1)^k pi^2k / ((2k)! 4^k), k = 5 .. 1
  p = p * z + 9.19260275e-04f;
  p = p * z - 2.08634808e-02f;
  p = p * z + 2.53669508e-01f;
  p = p * z - 1.23370055f;
  return p * z + 1.0f;
}

// One warp generates 32 traces (a lane each, sequential in time) over one chunk of
// kGenChunk steps and writes 32x32 tiles transposed through shared memory so every store is a
// coalesced 128-byte row segment. Chunks run in parallel (blockIdx.y); each starts its AR(1) /
// OU state from a draw keyed by (seed, trace id, chunk), so the traces stay a pure function of
// the global trace id. Every operation is exactly rounded IEEE fp32 (no intrinsics, no
// contraction), so the host port produces identical traces (the reference arm of bench.py times
// the reference algorithm on exactly these caps).
constexpr int64_t kGenChunk = 4096;

__global__ void gen_kernel(float* caps, int64_t T, int64_t S, int64_t ld, int64_t first_id, int32_t step_seconds,
                           int32_t kind, float peak, uint64_t seed, float a_cloud) {
  __shared__ float tile[8][32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t t0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + w) * 32;
  if (t0 >= T) return;
  const int64_t c0 = (int64_t)blockIdx.y * kGenChunk, c1 = min(S, c0 + kGenChunk);
  const int64_t tid = first_id + t0 + lane;
  const uint64_t hk = splitmix(seed ^ splitmix((uint64_t)tid));
  int k = kind;
  if (k == CS_TRACE_MIXED) k = (tid & 1) ? CS_TRACE_WIND : CS_TRACE_SOLAR;
  // per-trace parameters
  const float var = 0.1f + 0.7f * u01(splitmix(hk ^ 1));           // Table-1 variation range 10%..80%
  const float phase = 86400.0f * u01(splitmix(hk ^ 2));            // start time of day offset
  const float dt = (float)step_seconds;
  const float wind_mu = 5.0f + 5.0f * u01(splitmix(hk ^ 3));       // mean wind speed (m/s)
  const float theta = 1.0f / 7200.0f;                               // OU mean reversion (1/s)
  const float cloud_sd = var * 0.5f * sqrtf(fmaxf(1.0f - a_cloud * a_cloud, 1e-6f));
  const float sdt = fminf(theta * dt, 1.0f);
  const float wind_sd = var * 4.0f * sqrtf(2.0f * sdt);
  const uint64_t hc = splitmix(hk ^ (0xC0FFEEull + (uint64_t)blockIdx.y));
  float cloud = fminf(fmaxf(0.7f + var * 0.5f * gauss(hc), 0.2f), 1.0f);
  float wind = fmaxf(wind_mu + var * 4.0f * 0.7f * gauss(splitmix(hc)), 0.0f);
  for (int64_t s0 = c0; s0 < c1; s0 += 32) {
    for (int j = 0; j < 32; ++j) {
      const int64_t s = s0 + j;
      const uint64_t hs = splitmix(hk ^ (uint64_t)(s * 0x632BE59BD9B4E019ull));
      float v;
      if (k == CS_TRACE_IID) {
        v = peak * u01(hs);
      } else if (k == CS_TRACE_SOLAR) {
        const float tod = fmodf(phase + (float)s * dt, 86400.0f) / 3600.0f;
        const float clear = (tod > 6.0f && tod < 18.0f) ? clear_sky((tod - 6.0f) / 12.0f) : 0.0f;
        cloud = a_cloud * cloud + (1.0f - a_cloud) * 0.7f + cloud_sd * gauss(hs);  // 1 h AR(1) cloud factor
        cloud = fminf(fmaxf(cloud, 0.2f), 1.0f);
        v = peak * clear * cloud;
      } else {
        wind = wind + sdt * (wind_mu - wind) + wind_sd * gauss(hs);  // OU wind speed
        wind = fmaxf(wind, 0.0f);
        float f = 0.0f;  // cubic power curve: cut-in 3, rated 12, cut-out 25 m/s
        if (wind >= 3.0f && wind < 25.0f) {
          const float r = (wind - 3.0f) / 9.0f;
          f = wind >= 12.0f ? 1.0f : r * r * r;
        }
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

// PolicyIndex.select (policy.py:136-148): union bin of each cap through the staged LUT (global
// memory; a handful of caps per launch). The caller decodes the bin per regime on the host.
__global__ void lookup_kernel(const DevTables tb, const double* __restrict__ caps, int64_t n,
                              int32_t* __restrict__ bins) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (tb.cap_dtype == CS_CAP_F64) {
    bins[i] = (int32_t)bin_f64((uint64_t)__double_as_longlong(caps[i]), tb.lv.lo, tb.lv.hi, tb.lv.shift1,
                               tb.lv.kbase, tb.lv.sub0, tb.lv.lut, tb.lv.thr64);
  } else {
    bins[i] = (int32_t)bin_f32(__float_as_uint((float)caps[i]), tb.lv.shift1, (int32_t)tb.lv.kbase, tb.n_level1,
                               tb.lv.sub0, tb.lv.lut);
  }
}

// ----------------------------------------------------------------------------------------
// host-side launchers
// ----------------------------------------------------------------------------------------
void set_last_launches(int n);

std::string launch_select(const DevTables& v, int g, int p, const double* caps, int64_t n, int32_t* sel, int64_t* cnt,
                          cudaStream_t st) {
  if (n <= 0) return std::string();
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((n + 7) / 8, 148 * 32);
  select_kernel<<<(unsigned)blocks, threads, 0, st>>>(v, g, p, caps, n, sel, cnt);
  CS_CUDA_TRY(cudaGetLastError());
  set_last_launches(1);
  return std::string();
}

std::string launch_lookup(const DevTables& v, const double* caps, int64_t n, int32_t* bins, cudaStream_t st) {
  if (n <= 0) return std::string();
  lookup_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(v, caps, n, bins);
  CS_CUDA_TRY(cudaGetLastError());
  set_last_launches(1);
  return std::string();
}

std::string launch_feasible(const DevTables& v, int g, int p, const double* caps, int64_t n, uint32_t* mask,
                            cudaStream_t st) {
  if (n <= 0) return std::string();
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((n + 7) / 8, 148 * 32);
  feasible_kernel<<<(unsigned)blocks, threads, 0, st>>>(v, g, p, caps, n, mask);
  CS_CUDA_TRY(cudaGetLastError());
  set_last_launches(1);
  return std::string();
}

std::string launch_generate(float* caps, int64_t T, int64_t S, int64_t ld, int64_t first_id, int32_t step_seconds,
                            int32_t kind, float peak, uint64_t seed, cudaStream_t st) {
  if (T <= 0 || S <= 0) return std::string();
  const int64_t warps = (T + 31) / 32;
  const int64_t blocks = (warps + 7) / 8;
  const int64_t chunks = (S + kGenChunk - 1) / kGenChunk;
  if (chunks > 65535) return "trace too long for the generator (> 65535 chunks)";
  // AR(1) coefficient of the 1 h cloud correlation, computed on the host in fp64 (libm exp) and
  // rounded once: the host port (ora_generate_traces) derives it with the same expression
  const float a_cloud = (float)std::exp(-(double)step_seconds / 3600.0);
  gen_kernel<<<dim3((unsigned)blocks, (unsigned)chunks), 256, 0, st>>>(caps, T, S, ld, first_id, step_seconds, kind,
                                                                       peak, seed, a_cloud);
  CS_CUDA_TRY(cudaGetLastError());
  return std::string();
}

}  // namespace cs
