// Online controller replay on the GPU (reference controller.py:96-231).
//
// The controller is a sequential state machine along time (a reconfiguration changes what is
// measured next), so one thread owns one trace; traces run in parallel (violation-fraction
// sweeps over many traces / noise seeds). Every reselection is select_config(grid, COMBINATION,
// x) (controller.py:106,136) answered with the staged fp64 rank tables (one LUT search), the
// sensor noise replays CPython's random.Random(seed) stream (MT19937 init_by_array + random() +
// uniform(), Modules/_randommodule.c, Lib/random.py) bit for bit, and the moving-average
// prediction is fsum(history) / len (statistics.fmean) computed exactly in double-double.
#include <cuda_runtime.h>

#include <string>

#include "cs_internal.h"
#include "cs_mt.cuh"

namespace cs {
namespace {

#define CS_CUDA_TRY(x)                                                                                  \
  do {                                                                                                  \
    cudaError_t e_ = (x);                                                                               \
    if (e_ != cudaSuccess) return std::string("CUDA error: ") + cudaGetErrorString(e_) + " (" #x ")"; \
  } while (0)

__device__ __forceinline__ void two_sum_acc(double& hi, double& lo, double v) {
  const double s = __dadd_rn(hi, v);
  const double bb = __dsub_rn(s, hi);
  const double e = __dadd_rn(__dsub_rn(hi, __dsub_rn(s, bb)), __dsub_rn(v, bb));
  hi = s;
  lo = __dadd_rn(lo, e);
}

struct Sel {
  int32_t entry;  // caller entry index, -1 idle
  uint16_t bin;   // grid bin (0xFFFF: the caller-supplied initial config)
  double pw, thr;
};

// select_config(grid, COMBINATION, x) through the staged fp64 tables (policy.py:172-188)
__device__ Sel select_comb(const DevTables& tb, int g, double x) {
  const uint32_t u = bin_f64((uint64_t)__double_as_longlong(x), tb.lv.lo, tb.lv.hi, tb.lv.shift1, tb.lv.kbase,
                             tb.lv.sub0, tb.lv.lut, tb.lv.thr64);
  const int r = tb.M > 1 ? (int)tb.umap[(size_t)g * tb.U + u] : (int)u;
  const size_t o = ((size_t)g * 3 + 2) * tb.maxB + r;
  Sel s;
  s.entry = tb.sel[o];
  s.bin = (uint16_t)r;
  s.pw = tb.spw[o];
  s.thr = tb.sthr[o];
  return s;
}

constexpr int kMaxKey = 8;

__global__ void replay_kernel(const DevTables tb, int g, const double* __restrict__ caps, int64_t T, int64_t S,
                              int64_t ld, int mode, int window_k, const int32_t* __restrict__ initial,
                              double noise_pct, const uint32_t* __restrict__ keys, const int32_t* __restrict__ key_len,
                              int key_stride, unsigned long long seed_base, cs_replay_step* __restrict__ steps,
                              cs_replay_agg* __restrict__ agg) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  // time-major caps ([S][ld], ld >= T): a warp's 32 traces read 256 contiguous bytes per step
  const bool tm = (mode & CS_CTRL_TIME_MAJOR) != 0;
  mode &= 0xFF;
  const double* c = tm ? caps + t : caps + t * ld;
  const int64_t cstride = tm ? ld : 1;
  Mt rng;
  if (noise_pct > 0.0) {
    uint32_t kbuf[kMaxKey];
    int kl;
    if (keys) {
      kl = key_len[t];
      for (int i = 0; i < kl; ++i) kbuf[i] = keys[t * key_stride + i];
    } else {  // seed = seed_base + t (non-negative)
      const unsigned long long sd = seed_base + (unsigned long long)t;
      kbuf[0] = (uint32_t)sd;
      kbuf[1] = (uint32_t)(sd >> 32);
      kl = kbuf[1] ? 2 : 1;
    }
    mt_seed(rng, kbuf, kl);
  }
  // initial selection: caller's config (feasible_count 0) or select_config(first cap)
  Sel cur;
  const int32_t init = initial ? initial[t] : -1;
  if (init >= 0) {
    const int e = tb.e_off[g] + init;
    cur.entry = init;
    cur.bin = 0xFFFF;
    cur.pw = tb.e_pw[e];
    cur.thr = tb.e_thr[e];
  } else {
    cur = select_comb(tb, g, c[0]);  // step 0 (same element in both layouts)
  }
  // the proactive window (ControllerState.cap_history, a deque(maxlen=k) of the caps seen so far,
  // controller.py:87,137) is the trace's own last min(k, i + 1) caps: read back from the cap row
  // itself (L1/L2-resident), so any window_k works without per-thread history storage
  long long viol = 0, rec = 0;
  double th = 0.0, tl = 0.0;
  for (int64_t i = 0; i < S; ++i) {
    const double cap = c[i * cstride];
    double meas = cur.entry < 0 ? 0.0 : cur.pw;
    if (noise_pct > 0.0 && cur.entry >= 0) {
      const double r = mt_random(rng);
      const double un = __dadd_rn(-noise_pct, __dmul_rn(__dsub_rn(noise_pct, -noise_pct), r));  // uniform(-n, n)
      meas = __dmul_rn(meas, __dadd_rn(1.0, __ddiv_rn(un, 100.0)));
    }
    uint8_t kb = 0;
    if (meas > cap) {  // _reactive_core (controller.py:96-110)
      kb |= 1;
      ++viol;
      cur = select_comb(tb, g, cap);
      ++rec;
    }
    const uint16_t bin_r = cur.bin;
    if (mode == 1) {  // step_proactive (controller.py:125-142): predicted = fmean(history)
      const int64_t hlen = i + 1 < (int64_t)window_k ? i + 1 : (int64_t)window_k;
      double sh = 0.0, sl = 0.0;
      for (int64_t q = i + 1 - hlen; q <= i; ++q) two_sum_acc(sh, sl, c[q * cstride]);
      const double predicted = __ddiv_rn(__dadd_rn(sh, sl), (double)hlen);
      if (cur.entry >= 0 && predicted < cur.pw) {
        kb |= 2;
        cur = select_comb(tb, g, predicted);
        ++rec;
      }
    }
    if (steps) {
      cs_replay_step st;
      st.measured_power_w = meas;
      st.bin_reactive = bin_r;
      st.bin_final = cur.bin;
      st.kind_bits = kb;
      st.pad[0] = st.pad[1] = st.pad[2] = 0;
      steps[t * S + i] = st;
    }
    two_sum_acc(th, tl, cur.entry < 0 ? 0.0 : cur.thr);
  }
  cs_replay_agg a;
  a.violations = viol;
  a.reconfigs = rec;
  a.violation_fraction = __ddiv_rn((double)viol, (double)S);
  a.avg_throughput_ips = __ddiv_rn(__dadd_rn(th, tl), (double)S);
  a.num_steps = S;
  agg[t] = a;
}

}  // namespace

void set_last_launches(int n);

std::string launch_replay(const DevTables& v, int g, const double* caps, int64_t T, int64_t S, int64_t ld, int mode,
                          int window_k, const int32_t* initial, double noise_pct, const uint32_t* keys,
                          const int32_t* key_len, int key_stride, unsigned long long seed_base, cs_replay_step* steps,
                          cs_replay_agg* agg, cudaStream_t st) {
  if (window_k < 1) return "window_k must be >= 1";
  if (keys && (key_stride < 1 || key_stride > kMaxKey)) return "seed keys longer than 8 words are not supported";
  if (T <= 0) return std::string();
  const int threads = 128;
  replay_kernel<<<(unsigned)((T + threads - 1) / threads), threads, 0, st>>>(
      v, g, caps, T, S, ld, mode, window_k, initial, noise_pct, keys, key_len, key_stride, seed_base, steps, agg);
  CS_CUDA_TRY(cudaGetLastError());
  set_last_launches(1);
  return std::string();
}

}  // namespace cs
