// Sampling selector on the GPU (reference policy.py:191-273, sim.py:159-163).
//
// select_sampling(grid, m, r, cap, seed) for every (trace, step) of a cap matrix, one thread per
// step (steps are independent: each draws from its own random.Random(seed * 1_000_003 + step)).
// A step is:
//   1. count = len(feasible) from the staged fp64 rank tables (one LUT search, as PolicyIndex);
//      the feasible list sorted by (power, mtl, bs) (policy.py:246) is the grid's combination
//      order csort[0 .. count), so no per-step filter or sort is needed;
//   2. count == 0 -> idle; m >= count -> every feasible entry is a sample, so the best one is the
//      combination selection (and no neighbour can improve on a global maximum);
//   3. otherwise random.sample(range(count), m) replayed bit for bit (Lib/random.py: the pool
//      branch when count <= setsize, else the rejection-set branch; both hold at most m
//      positions, so the per-thread state is O(m), not O(count)), best = highest throughput,
//      ties to the lower sorted position (_prefer, policy.py:88-97);
//   4. up to r hill-climb rounds over the staged neighbour lists (policy.py:255-266).
#include <cuda_runtime.h>

#include <string>

#include "cs_internal.h"
#include "cs_mt.cuh"

namespace cs {
namespace {

constexpr int kMaxBudget = CS_SAMPLING_MAX_BUDGET;

struct SampleParams {
  DevTables tb;
  int g;
  const double* caps;
  int64_t T, S, ld;
  int64_t budget, rounds, setsize;
  unsigned long long seed_lo;
  long long seed_hi;
  int32_t* out_entry;
  int32_t* out_count;
  uint16_t* scratch;       // BIG only: [threads][scratch_stride] pool / bitmap words
  int64_t scratch_stride;  // uint16 words per thread
};

// _prefer(a, b) == a for caller entries a != b (policy.py:88-97)
__device__ __forceinline__ bool prefer_a(const DevTables& tb, int base, int a, int b) {
  const double ta = tb.e_thr[base + a], tb_ = tb.e_thr[base + b];
  if (ta != tb_) return ta > tb_;
  const double pa = tb.e_pw[base + a], pb = tb.e_pw[base + b];
  if (pa != pb) return pa < pb;
  if (tb.e_mtl[base + a] != tb.e_mtl[base + b]) return tb.e_mtl[base + a] < tb.e_mtl[base + b];
  return tb.e_bs[base + a] <= tb.e_bs[base + b];
}

// BIG (budgets above kMaxBudget): the pool is materialised in a per-thread global scratch row
// (n uint16 positions, or an n-bit bitmap for the set branch) instead of the O(m) slot list.
template <bool BIG>
__global__ void __launch_bounds__(128) sampling_kernel(const __grid_constant__ SampleParams P) {
  const DevTables& tb = P.tb;
  const int g = P.g;
  const int base = tb.e_off[g];
  const int64_t total = P.T * P.S;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = q / P.S, i = q - t * P.S;
    const double cap = P.caps[t * P.ld + i];
    const uint32_t u = bin_f64((uint64_t)__double_as_longlong(cap), tb.lv.lo, tb.lv.hi, tb.lv.shift1, tb.lv.kbase,
                               tb.lv.sub0, tb.lv.lut, tb.lv.thr64);
    const int r = tb.M > 1 ? (int)tb.umap[(size_t)g * tb.U + u] : (int)u;
    const int n = tb.ccnt[(size_t)g * tb.maxB + r];
    int cur = -1;
    if (n > 0 && P.budget >= n) {
      cur = tb.sel[((size_t)g * 3 + 2) * tb.maxB + r];
    } else if (n > 0) {
      // random.Random(seed_base + i): init_by_array key = 32-bit words of abs(seed)
      __int128 v = (__int128)(((unsigned __int128)(unsigned long long)P.seed_hi << 64) | P.seed_lo) + (__int128)i;
      unsigned __int128 a = v < 0 ? (unsigned __int128)(-v) : (unsigned __int128)v;
      uint32_t key[4];
      int kl = 0;
      do {
        key[kl++] = (uint32_t)a;
        a >>= 32;
      } while (a && kl < 4);
      MtLazy rng;
      mt_lazy_seed(rng, key, kl);
      const int k = (int)P.budget;
      const int* cs = tb.csort + base;
      int best = -1;
      double best_thr = 0.0;
      auto consider = [&](int pos) {
        const double th = tb.e_thr[base + cs[pos]];
        if (best < 0 || th > best_thr || (th == best_thr && pos < best)) best = pos, best_thr = th;
      };
      if (BIG) {
        uint16_t* row = P.scratch + ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * P.scratch_stride;
        if ((int64_t)n <= P.setsize) {
          for (int z = 0; z < n; ++z) row[z] = (uint16_t)z;
          for (int s = 0; s < k; ++s) {
            const int j = (int)mt_randbelow(rng, (uint32_t)(n - s));
            consider(row[j]);
            row[j] = row[n - s - 1];
          }
        } else {
          uint32_t* bits = reinterpret_cast<uint32_t*>(row);
          for (int z = 0; z < (n + 31) / 32; ++z) bits[z] = 0;
          for (int s = 0; s < k; ++s) {
            int j = (int)mt_randbelow(rng, (uint32_t)n);
            while ((bits[j >> 5] >> (j & 31)) & 1u) j = (int)mt_randbelow(rng, (uint32_t)n);
            bits[j >> 5] |= 1u << (j & 31);
            consider(j);
          }
        }
      } else {
      int32_t slot[BIG ? 1 : kMaxBudget], sval[BIG ? 1 : kMaxBudget];
      int ns = 0;
      if ((int64_t)n <= P.setsize) {
        // pool branch: pool[j] read / pool[j] = pool[n-i-1]; only overwritten slots are stored
        for (int s = 0; s < k; ++s) {
          const int j = (int)mt_randbelow(rng, (uint32_t)(n - s));
          const int last = n - s - 1;
          int val = j, lval = last, jslot = -1;
          for (int z = 0; z < ns; ++z) {
            if (slot[z] == j) val = sval[z], jslot = z;
            if (slot[z] == last) lval = sval[z];
          }
          consider(val);
          if (jslot < 0) jslot = ns++, slot[jslot] = j;
          sval[jslot] = lval;
        }
      } else {
        // set branch: redraw until a position not yet selected
        for (int s = 0; s < k; ++s) {
          int j;
          bool dup;
          do {
            j = (int)mt_randbelow(rng, (uint32_t)n);
            dup = false;
            for (int z = 0; z < ns; ++z) dup |= slot[z] == j;
          } while (dup);
          slot[ns++] = j;
          consider(j);
        }
      }
      }
      cur = cs[best];
      // hill climb: best feasible strictly-better present neighbour, until none (policy.py:255-266)
      for (int64_t rr = 0; rr < P.rounds; ++rr) {
        const int* nb = tb.nbr + (size_t)(base + cur) * 4;
        const double cthr = tb.e_thr[base + cur];
        int move = -1;
        for (int z = 0; z < 4; ++z) {
          const int e = nb[z];
          if (e < 0) break;
          if (tb.e_pw[base + e] > cap || tb.e_thr[base + e] <= cthr) continue;
          if (move < 0 || !prefer_a(tb, base, move, e)) move = e;
        }
        if (move < 0) break;
        cur = move;
      }
    }
    P.out_entry[q] = cur;
    if (P.out_count) P.out_count[q] = n;
  }
}

}  // namespace

void set_last_launches(int n);

// Random.sample's table-size rule (Lib/random.py): 21, plus 4 ** ceil(log(3k, 4)) when k > 5.
// 3k is never a power of 4, so the smallest power of 4 >= 3k is exactly that ceiling.
int64_t sample_setsize(int64_t k) {
  int64_t s = 21;
  if (k > 5) {
    int64_t p = 1;
    while (p < 3 * k) p *= 4;
    s += p;
  }
  return s;
}

std::string launch_sampling(const DevTables& v, int g, const double* caps, int64_t T, int64_t S, int64_t ld,
                            int64_t budget, int64_t rounds, unsigned long long seed_lo, long long seed_hi,
                            int32_t* out_entry, int32_t* out_count, int n_entries, int sm_count, cudaStream_t st) {
  if (T <= 0 || S <= 0) return std::string();
  SampleParams P;
  P.tb = v;
  P.g = g;
  P.caps = caps;
  P.T = T;
  P.S = S;
  P.ld = ld;
  P.budget = budget;
  P.rounds = rounds;
  P.setsize = sample_setsize(budget < n_entries ? budget : n_entries);
  P.seed_lo = seed_lo;
  P.seed_hi = seed_hi;
  P.out_entry = out_entry;
  P.out_count = out_count;
  P.scratch = nullptr;
  P.scratch_stride = 0;
  const int threads = 128;
  const int64_t want = (T * S + threads - 1) / threads;
  const bool big = budget > kMaxBudget && budget < n_entries;
  if (!big) {
    const int64_t cap_blocks = (int64_t)sm_count * 16;
    sampling_kernel<false><<<(unsigned)(want < cap_blocks ? want : cap_blocks), threads, 0, st>>>(P);
  } else {
    // one CTA per SM; scratch rows hold n uint16 pool slots (>= the n-bit bitmap), 16-B aligned
    const int64_t blocks = want < sm_count ? want : sm_count;
    P.scratch_stride = ((int64_t)n_entries + 63) / 64 * 64;
    void* scratch = nullptr;
    cudaError_t e = cudaMallocAsync(&scratch, (size_t)blocks * threads * P.scratch_stride * 2, st);
    if (e != cudaSuccess) return std::string("CUDA error: ") + cudaGetErrorString(e);
    P.scratch = static_cast<uint16_t*>(scratch);
    sampling_kernel<true><<<(unsigned)blocks, threads, 0, st>>>(P);
    e = cudaGetLastError();
    cudaFreeAsync(scratch, st);
    if (e != cudaSuccess) return std::string("CUDA error: ") + cudaGetErrorString(e);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return std::string("CUDA error: ") + cudaGetErrorString(e);
  set_last_launches(1);
  return std::string();
}

// _aggregate (sim.py:104-127) over per-step entry selections (the sampling selector's output):
// one warp per trace. Every per-step value comes from a small per-entry table whose values the
// host pre-split into {hi, lo} (hi on a quantum grid so that the sum of hi is exact in fp64, like
// prep_kernel's split), so the result equals the reference's math.fsum up to the lo parts.
//   vals[j * (n + 1) + e], j = 0 thr, 1 penalised thr (thr * (1 - pf)), 2 energy; e = n: idle
__global__ void __launch_bounds__(256) entries_agg_kernel(const int32_t* ent, int64_t T, int64_t S, int64_t ld,
                                                          const double2* vals, int n, double pf, double* avg,
                                                          double* energy, int64_t* idle) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= T) return;
  const int32_t* row = ent + t * ld;
  double th = 0.0, tl = 0.0, eh = 0.0, el = 0.0;
  uint32_t id = 0;
  for (int64_t i = lane; i < S; i += 32) {
    const int32_t e = row[i];
    const int k = e < 0 ? n : e;
    const bool sw = pf > 0.0 && i > 0 && row[i - 1] != e;  // sim.py:119 (None vs config counts)
    const double2 v = vals[(sw ? 1 : 0) * (n + 1) + k];
    const double2 w = vals[2 * (n + 1) + k];
    th = __dadd_rn(th, v.x);
    tl = __dadd_rn(tl, v.y);
    eh = __dadd_rn(eh, w.x);
    el = __dadd_rn(el, w.y);
    id += e < 0 ? 1u : 0u;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    th = __dadd_rn(th, __shfl_xor_sync(0xffffffffu, th, o));
    tl = __dadd_rn(tl, __shfl_xor_sync(0xffffffffu, tl, o));
    eh = __dadd_rn(eh, __shfl_xor_sync(0xffffffffu, eh, o));
    el = __dadd_rn(el, __shfl_xor_sync(0xffffffffu, el, o));
  }
  id = __reduce_add_sync(0xffffffffu, id);
  if (lane == 0) {
    avg[t] = __ddiv_rn(__dadd_rn(th, tl), (double)S);  // fsum(ips) / n
    energy[t] = __dadd_rn(eh, el);
    idle[t] = id;
  }
}

std::string launch_entries_agg(const int32_t* ent, int64_t T, int64_t S, int64_t ld, const double2* vals, int n,
                               double pf, double* avg, double* energy, int64_t* idle, cudaStream_t st) {
  if (T <= 0) return std::string();
  const int64_t blocks = (T + 7) / 8;
  entries_agg_kernel<<<(unsigned)blocks, 256, 0, st>>>(ent, T, S, ld, vals, n, pf, avg, energy, idle);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return std::string("CUDA error: ") + cudaGetErrorString(e);
  set_last_launches(1);
  return std::string();
}

}  // namespace cs
