/*
 * capsim_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C, scalar restatement of the reference's trace-driven policy-evaluation hot
 * path (capsim 0.1.0, /root/reference/pkg/src/capsim). Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 *
 * Pinned against the reference itself: the JSON fixtures under tests/golden were produced by importing the
 * reference package in the build container (tests/golden/make_golden.py) and
 * tests/test_oracle_golden.py checks every vector against this file.
 *
 * Every function names the reference lines it restates:
 *   ora_regime_member   policy.py:100-107   (_regime_entries)
 *   ora_prefer          policy.py:90-97     (_prefer: higher ips, then lower (power, mtl, bs))
 *   ora_index_build     policy.py:118-134   (PolicyIndex.__init__: sort by (power,mtl,bs) + prefix best)
 *   ora_index_select    policy.py:136-148   (PolicyIndex.select: bisect_right, idle when 0)
 *   ora_bruteforce      tests/conftest.py:100-129 (independent linear-scan argmax)
 *   ora_fsum            CPython math.fsum   (exactly rounded sum; used by sim.py:126-127)
 *   ora_aggregate       sim.py:104-127      (_aggregate: switch penalty, energy proxy, idle count)
 *   ora_simulate        sim.py:130-188      (simulate: per-step selection + aggregate)
 *   ora_simulate_batch  loops ora_simulate over (trace, grid, policy) with pthreads — the
 *                       CPU baseline ("port") the bench times beside the GPU.
 *   ora_generate_traces not a reference function: host port of the bench's synthetic trace
 *                       generator, so the reference arm runs on the engine arm's exact caps.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORA_BATCHING 0
#define ORA_MULTI_TENANT 1
#define ORA_COMBINATION 2

typedef struct {
  int32_t mtl, bs;
  double thr, pw;
  int32_t idx; /* position in the caller's entry arrays */
} ora_entry;

/* policy.py:100-107 */
static int ora_regime_member(int regime, int32_t mtl, int32_t bs, int batching_mtl, int mt_bs) {
  if (regime == ORA_BATCHING) return mtl == batching_mtl;
  if (regime == ORA_MULTI_TENANT) return bs == mt_bs;
  return 1;
}

/* lexicographic (power, mtl, bs) comparison used by both the sort key (policy.py:129)
 * and the tie-break of _prefer (policy.py:95-97). */
static int ora_key_cmp(const ora_entry* a, const ora_entry* b) {
  if (a->pw < b->pw) return -1;
  if (a->pw > b->pw) return 1;
  if (a->mtl != b->mtl) return a->mtl < b->mtl ? -1 : 1;
  if (a->bs != b->bs) return a->bs < b->bs ? -1 : 1;
  return 0;
}

static int ora_qsort_cmp(const void* a, const void* b) {
  return ora_key_cmp((const ora_entry*)a, (const ora_entry*)b);
}

/* policy.py:90-97: returns 1 when a is preferred over b */
static int ora_prefer_a(const ora_entry* a, const ora_entry* b) {
  if (a->thr != b->thr) return a->thr > b->thr;
  return ora_key_cmp(a, b) <= 0;
}

/*
 * policy.py:118-134. Fills, for the regime's entries sorted by (power, mtl, bs):
 *   powers[i]   = power of the i-th sorted entry
 *   best_idx[i] = caller index of the prefix-best entry among sorted[0..i]
 * Returns the regime size n_reg (<= n).
 */
int ora_index_build(const int32_t* mtl, const int32_t* bs, const double* thr, const double* pw, int n,
                    int regime, int batching_mtl, int mt_bs, double* powers, int32_t* best_idx) {
  ora_entry* e = (ora_entry*)malloc(sizeof(ora_entry) * (size_t)(n > 0 ? n : 1));
  int m = 0;
  for (int i = 0; i < n; ++i) {
    if (!ora_regime_member(regime, mtl[i], bs[i], batching_mtl, mt_bs)) continue;
    e[m].mtl = mtl[i]; e[m].bs = bs[i]; e[m].thr = thr[i]; e[m].pw = pw[i]; e[m].idx = i;
    ++m;
  }
  /* (mtl, bs) are unique in a grid, so the key is a strict total order and an unstable
   * sort gives the same result as Python's stable sort. */
  qsort(e, (size_t)m, sizeof(ora_entry), ora_qsort_cmp);
  int best = -1;
  for (int i = 0; i < m; ++i) {
    powers[i] = e[i].pw;
    if (best < 0 || !ora_prefer_a(&e[best], &e[i])) best = i;
    best_idx[i] = e[best].idx;
  }
  free(e);
  return m;
}

/* policy.py:136-148 (caller has already rejected cap < 0). Returns feasible_count;
 * *sel = caller index of the selection or -1 for IDLE_SELECTION. */
int64_t ora_index_select(const double* powers, const int32_t* best_idx, int n_reg, double cap, int32_t* sel) {
  /* bisect.bisect_right: first position whose power is > cap */
  int lo = 0, hi = n_reg;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (cap < powers[mid]) hi = mid; else lo = mid + 1;
  }
  *sel = lo == 0 ? -1 : best_idx[lo - 1];
  return lo;
}

/* tests/conftest.py:100-129: independent brute-force argmax (no shared code with the index). */
int32_t ora_bruteforce(const int32_t* mtl, const int32_t* bs, const double* thr, const double* pw, int n,
                       int regime, int batching_mtl, int mt_bs, double cap) {
  int32_t best = -1;
  for (int i = 0; i < n; ++i) {
    if (pw[i] > cap) continue;
    if (!ora_regime_member(regime, mtl[i], bs[i], batching_mtl, mt_bs)) continue;
    if (best < 0) { best = i; continue; }
    if (thr[i] > thr[best]) best = i;
    else if (thr[i] == thr[best]) {
      if (pw[i] < pw[best]) best = i;
      else if (pw[i] == pw[best]) {
        if (mtl[i] < mtl[best]) best = i;
        else if (mtl[i] == mtl[best] && bs[i] < bs[best]) best = i;
      }
    }
  }
  return best;
}

/* CPython math.fsum (Shewchuk partials + half-even correction), finite inputs only. */
typedef struct { double* p; int n, cap; } ora_partials;

static void ora_partials_add(ora_partials* ps, double x) {
  int i = 0;
  for (int j = 0; j < ps->n; ++j) {
    double y = ps->p[j];
    if (fabs(x) < fabs(y)) { double t = x; x = y; y = t; }
    double hi = x + y;
    double lo = y - (hi - x);
    if (lo != 0.0) ps->p[i++] = lo;
    x = hi;
  }
  if (i >= ps->cap) {
    ps->cap = ps->cap ? ps->cap * 2 : 32;
    ps->p = (double*)realloc(ps->p, sizeof(double) * (size_t)ps->cap);
  }
  ps->p[i] = x;
  ps->n = i + 1;
}

static double ora_partials_result(const ora_partials* ps) {
  int n = ps->n;
  double hi = 0.0;
  if (n > 0) {
    double lo = 0.0;
    hi = ps->p[--n];
    while (n > 0) {
      double x = hi;
      double y = ps->p[--n];
      hi = x + y;
      double yr = hi - x;
      lo = y - yr;
      if (lo != 0.0) break;
    }
    if (n > 0 && ((lo < 0.0 && ps->p[n - 1] < 0.0) || (lo > 0.0 && ps->p[n - 1] > 0.0))) {
      double y = lo * 2.0;
      double x = hi + y;
      double yr = x - hi;
      if (y == yr) hi = x;
    }
  }
  return hi;
}

double ora_fsum(const double* x, int64_t n) {
  ora_partials ps = {0, 0, 0};
  for (int64_t i = 0; i < n; ++i) ora_partials_add(&ps, x[i]);
  double r = ora_partials_result(&ps);
  free(ps.p);
  return r;
}

/*
 * sim.py:104-127 over per-step selections. sel[i] = caller entry index or -1 (idle).
 * Outputs avg throughput, idle count and energy proxy exactly as the reference computes them.
 */
void ora_aggregate(const double* thr, const double* pw, const int32_t* sel, int64_t n_steps, int32_t step_seconds,
                   double idle_power_w, double switch_penalty_s, double* avg, int64_t* idle, double* energy) {
  double pen = switch_penalty_s < (double)step_seconds ? switch_penalty_s : (double)step_seconds;
  double pf = pen / (double)step_seconds;
  ora_partials pt = {0, 0, 0}, pe = {0, 0, 0};
  int64_t idle_count = 0;
  int32_t prev = -1;
  for (int64_t i = 0; i < n_steps; ++i) {
    int32_t s = sel[i];
    double ips = s < 0 ? 0.0 : thr[s];
    if (i > 0 && pf > 0.0 && s != prev) ips *= 1.0 - pf;
    ora_partials_add(&pt, ips);
    double p = s < 0 ? idle_power_w : pw[s];
    ora_partials_add(&pe, p * (double)step_seconds / 3600.0);
    if (s < 0) ++idle_count;
    prev = s;
  }
  *avg = ora_partials_result(&pt) / (double)n_steps;
  *idle = idle_count;
  *energy = ora_partials_result(&pe);
  free(pt.p);
  free(pe.p);
}

/*
 * sim.py:130-188 for one (grid, trace, exhaustive policy). caps are fp64 (fp32 caps are
 * widened exactly by the caller). step_sel / step_count (nullable) receive the per-step
 * selection index and feasible_count. Returns 0, or -1 on a negative cap (policy.py:137).
 */
int ora_simulate(const int32_t* mtl, const int32_t* bs, const double* thr, const double* pw, int n,
                 int regime, const double* caps, int64_t n_steps, int32_t step_seconds, double idle_power_w,
                 double switch_penalty_s, int32_t* step_sel, int64_t* step_count, double* avg, int64_t* idle,
                 double* energy) {
  double* powers = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  int32_t* best = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  int32_t* sel = step_sel ? step_sel : (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_steps > 0 ? n_steps : 1));
  int m = ora_index_build(mtl, bs, thr, pw, n, regime, 1, 1, powers, best);
  int rc = 0;
  for (int64_t i = 0; i < n_steps; ++i) {
    if (caps[i] < 0.0) { rc = -1; break; }
    int64_t c = ora_index_select(powers, best, m, caps[i], &sel[i]);
    if (step_count) step_count[i] = c;
  }
  if (rc == 0) ora_aggregate(thr, pw, sel, n_steps, step_seconds, idle_power_w, switch_penalty_s, avg, idle, energy);
  free(powers);
  free(best);
  if (!step_sel) free(sel);
  return rc;
}

/* ---- batch driver: the CPU baseline timed by bench.py (reference algorithm, all host threads) ---- */

typedef struct {
  const int32_t* mtl; const int32_t* bs; const double* thr; const double* pw; int n;
  double idle_power_w;
} ora_grid;

typedef struct {
  const ora_grid* grids; int n_grids;
  const float* caps; int64_t n_traces, n_steps;
  int32_t step_seconds; double switch_penalty_s;
  double* out_avg; int64_t* out_idle; double* out_energy; /* [trace][grid][policy] */
  int64_t next; pthread_mutex_t mu;
} ora_batch_job;

static void* ora_batch_worker(void* arg) {
  ora_batch_job* j = (ora_batch_job*)arg;
  double* caps64 = (double*)malloc(sizeof(double) * (size_t)j->n_steps);
  int32_t* sel = (int32_t*)malloc(sizeof(int32_t) * (size_t)j->n_steps);
  for (;;) {
    pthread_mutex_lock(&j->mu);
    int64_t t = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (t >= j->n_traces) break;
    const float* c = j->caps + t * j->n_steps;
    for (int64_t i = 0; i < j->n_steps; ++i) caps64[i] = (double)c[i];
    for (int g = 0; g < j->n_grids; ++g) {
      const ora_grid* gr = &j->grids[g];
      for (int p = 0; p < 3; ++p) {
        int64_t o = (t * j->n_grids + g) * 3 + p;
        ora_simulate(gr->mtl, gr->bs, gr->thr, gr->pw, gr->n, p, caps64, j->n_steps, j->step_seconds,
                     gr->idle_power_w, j->switch_penalty_s, sel, NULL, &j->out_avg[o], &j->out_idle[o],
                     &j->out_energy[o]);
      }
    }
  }
  free(caps64);
  free(sel);
  return NULL;
}

/* grids_* are flattened: entries of grid g live at [offs[g], offs[g+1]). Policy order in the
 * output is (batching, multi-tenant, combination). Returns the thread count used. */
int ora_simulate_batch(const int32_t* mtl, const int32_t* bs, const double* thr, const double* pw,
                       const int64_t* offs, const double* idle_power_w, int n_grids, const float* caps,
                       int64_t n_traces, int64_t n_steps, int32_t step_seconds, double switch_penalty_s,
                       int n_threads, double* out_avg, int64_t* out_idle, double* out_energy) {
  ora_grid* grids = (ora_grid*)malloc(sizeof(ora_grid) * (size_t)n_grids);
  for (int g = 0; g < n_grids; ++g) {
    grids[g].mtl = mtl + offs[g]; grids[g].bs = bs + offs[g];
    grids[g].thr = thr + offs[g]; grids[g].pw = pw + offs[g];
    grids[g].n = (int)(offs[g + 1] - offs[g]);
    grids[g].idle_power_w = idle_power_w[g];
  }
  ora_batch_job j;
  j.grids = grids; j.n_grids = n_grids; j.caps = caps; j.n_traces = n_traces; j.n_steps = n_steps;
  j.step_seconds = step_seconds; j.switch_penalty_s = switch_penalty_s;
  j.out_avg = out_avg; j.out_idle = out_idle; j.out_energy = out_energy; j.next = 0;
  pthread_mutex_init(&j.mu, NULL);
  if (n_threads < 1) n_threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
  for (int i = 0; i < n_threads; ++i) pthread_create(&th[i], NULL, ora_batch_worker, &j);
  for (int i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
  pthread_mutex_destroy(&j.mu);
  free(th);
  free(grids);
  return n_threads;
}

/* ---- online controller replay (controller.py:96-231), the §8(f) extension ----------------- */

/* CPython's MT19937 (Modules/_randommodule.c): init_by_array seeding, genrand_uint32 and
 * random() = (a*2^26 + b) / 2^53 from two draws; uniform(a, b) = a + (b - a) * random()
 * (Lib/random.py). random.Random(seed) for an int seed keys init_by_array with the 32-bit
 * little-endian words of abs(seed) (at least one word). */
typedef struct { uint32_t mt[624]; int mti; } ora_mt;

static void ora_mt_init_genrand(ora_mt* s, uint32_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 624; ++i) s->mt[i] = 1812433253u * (s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) + (uint32_t)i;
  s->mti = 624;
}

void ora_mt_seed(ora_mt* s, const uint32_t* key, int key_len) {
  ora_mt_init_genrand(s, 19650218u);
  int i = 1, j = 0;
  for (int k = (624 > key_len ? 624 : key_len); k; --k) {
    s->mt[i] = (s->mt[i] ^ ((s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
    ++i, ++j;
    if (i >= 624) { s->mt[0] = s->mt[623]; i = 1; }
    if (j >= key_len) j = 0;
  }
  for (int k = 623; k; --k) {
    s->mt[i] = (s->mt[i] ^ ((s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
    ++i;
    if (i >= 624) { s->mt[0] = s->mt[623]; i = 1; }
  }
  s->mt[0] = 0x80000000u;
  s->mti = 624;
}

static uint32_t ora_mt_next(ora_mt* s) {
  static const uint32_t mag01[2] = {0u, 0x9908b0dfu};
  if (s->mti >= 624) {
    int kk;
    uint32_t y;
    for (kk = 0; kk < 624 - 397; ++kk) {
      y = (s->mt[kk] & 0x80000000u) | (s->mt[kk + 1] & 0x7fffffffu);
      s->mt[kk] = s->mt[kk + 397] ^ (y >> 1) ^ mag01[y & 1u];
    }
    for (; kk < 623; ++kk) {
      y = (s->mt[kk] & 0x80000000u) | (s->mt[kk + 1] & 0x7fffffffu);
      s->mt[kk] = s->mt[kk + (397 - 624)] ^ (y >> 1) ^ mag01[y & 1u];
    }
    y = (s->mt[623] & 0x80000000u) | (s->mt[0] & 0x7fffffffu);
    s->mt[623] = s->mt[396] ^ (y >> 1) ^ mag01[y & 1u];
    s->mti = 0;
  }
  uint32_t y = s->mt[s->mti++];
  y ^= (y >> 11);
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= (y >> 18);
  return y;
}

double ora_mt_random(ora_mt* s) {
  uint32_t a = ora_mt_next(s) >> 5, b = ora_mt_next(s) >> 6;
  return ((double)a * 67108864.0 + (double)b) * (1.0 / 9007199254740992.0);
}

/* One replay (controller.py:161-231). mode: 0 reactive, 1 proactive(window_k).
 * initial: caller entry index, or -1 for select_config(first cap).
 * Per-step outputs (nullable, [n_steps]):
 *   kind_bits: bit0 violation (VIOLATION_DETECTED + RECONFIGURED), bit1 preemptive reselection
 *   measured:  measured power fed to the step
 *   sel_r / cnt_r: selection (+ feasible_count) after the reactive part (current before the
 *                  step when nothing happened)
 *   sel_f / cnt_f: selection after the step
 * Aggregates: violations, reconfigs, avg throughput (fsum/n). Returns 0, or -1 on bad args. */
int ora_replay(const int32_t* mtl, const int32_t* bs, const double* thr, const double* pw, int n, const double* caps,
               int64_t n_steps, int mode, int window_k, int32_t initial, double noise_pct, const uint32_t* key,
               int key_len, uint8_t* kind_bits, double* measured_out, int32_t* sel_r, int64_t* cnt_r,
               int32_t* sel_f, int64_t* cnt_f, int64_t* violations, int64_t* reconfigs, double* avg) {
  if (n_steps < 1 || window_k < 1) return -1;
  double* powers = (double*)malloc(sizeof(double) * (size_t)n);
  int32_t* best = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int m = ora_index_build(mtl, bs, thr, pw, n, ORA_COMBINATION, 1, 1, powers, best);
  ora_mt rng;
  ora_mt_seed(&rng, key, key_len);
  double* hist = (double*)malloc(sizeof(double) * (size_t)window_k);
  int hlen = 0, hpos = 0;
  int32_t cur;
  int64_t cur_cnt;
  if (initial >= 0) {
    cur = initial;
    cur_cnt = 0; /* Selection(config, thr, pw): feasible_count defaults to 0 (controller.py:187-189) */
  } else {
    cur_cnt = ora_index_select(powers, best, m, caps[0], &cur);
  }
  ora_partials tp = {0, 0, 0};
  int64_t viol = 0, rec = 0;
  for (int64_t i = 0; i < n_steps; ++i) {
    const double cap = caps[i];
    double meas = cur < 0 ? 0.0 : pw[cur];
    if (noise_pct > 0 && cur >= 0) meas *= 1.0 + ((-noise_pct) + (noise_pct - (-noise_pct)) * ora_mt_random(&rng)) / 100.0;
    uint8_t kb = 0;
    if (meas > cap) { /* _reactive_core */
      kb |= 1;
      ++viol;
      cur_cnt = ora_index_select(powers, best, m, cap, &cur);
      ++rec;
    }
    if (sel_r) sel_r[i] = cur;
    if (cnt_r) cnt_r[i] = cur_cnt;
    /* cap history (deque maxlen k), appended in both modes */
    hist[hpos] = cap;
    hpos = (hpos + 1) % window_k;
    if (hlen < window_k) ++hlen;
    if (mode == 1) {
      /* fmean(history) = fsum(history) / len, oldest first (deque order) */
      ora_partials ps = {0, 0, 0};
      int start = hlen < window_k ? 0 : hpos;
      for (int q = 0; q < hlen; ++q) ora_partials_add(&ps, hist[(start + q) % window_k]);
      const double predicted = ora_partials_result(&ps) / (double)hlen;
      free(ps.p);
      if (cur >= 0 && predicted < pw[cur]) {
        kb |= 2;
        cur_cnt = ora_index_select(powers, best, m, predicted, &cur);
        ++rec;
      }
    }
    if (kind_bits) kind_bits[i] = kb;
    if (measured_out) measured_out[i] = meas;
    if (sel_f) sel_f[i] = cur;
    if (cnt_f) cnt_f[i] = cur_cnt;
    ora_partials_add(&tp, cur < 0 ? 0.0 : thr[cur]);
  }
  *violations = viol;
  *reconfigs = rec;
  *avg = ora_partials_result(&tp) / (double)n_steps;
  free(tp.p);
  free(hist);
  free(powers);
  free(best);
  return 0;
}

/* ---- sampling selector (policy.py:191-273), the §8(f) rank-2 extension -------------------- */

/* Random._randbelow_with_getrandbits (Lib/random.py): k = n.bit_length(); r = getrandbits(k)
 * (= genrand_uint32() >> (32 - k) for k <= 32) until r < n. */
static uint32_t ora_randbelow(ora_mt* s, uint32_t n) {
  int k = 0;
  while (k < 32 && (n >> k)) ++k;
  uint32_t r = ora_mt_next(s) >> (32 - k);
  while (r >= n) r = ora_mt_next(s) >> (32 - k);
  return r;
}

/* Random.sample's table-size rule: setsize = 21 (+ 4 ** ceil(log(3k, 4)) when k > 5). */
static int64_t ora_sample_setsize(int64_t k) {
  int64_t setsize = 21;
  if (k > 5) {
    int64_t p = 1;
    while (p < 3 * k) p *= 4;
    setsize += p;
  }
  return setsize;
}

/* policy.py:191-197 _nearest_bs: present bs closest to target (excluding `exclude`), ties to
 * the smaller size; -1 when none. bs values are small integers, so |b - target| is exact. */
static int32_t ora_nearest_bs(const int32_t* mtl, const int32_t* bs, int n, int32_t at_mtl, double target,
                              int32_t exclude) {
  int32_t best = -1;
  double bd = 0.0;
  for (int i = 0; i < n; ++i) {
    if (mtl[i] != at_mtl || bs[i] == exclude) continue;
    const double d = fabs((double)bs[i] - target);
    if (best < 0 || d < bd || (d == bd && bs[i] < best)) best = bs[i], bd = d;
  }
  return best;
}

static int ora_find(const int32_t* mtl, const int32_t* bs, int n, int32_t m, int32_t b) {
  for (int i = 0; i < n; ++i)
    if (mtl[i] == m && bs[i] == b) return i;
  return -1;
}

/* policy.py:200-215 _neighbors: (mtl -/+ 1, same bs) then (same mtl, nearest bs to bs/2, bs*2). */
static int ora_neighbors(const int32_t* mtl, const int32_t* bs, int n, int c, int out[4]) {
  int k = 0;
  for (int d = -1; d <= 1; d += 2) {
    const int32_t m = mtl[c] + d;
    if (m < 1) continue;
    const int e = ora_find(mtl, bs, n, m, bs[c]);
    if (e >= 0) out[k++] = e;
  }
  const double targets[2] = {(double)bs[c] / 2.0, (double)bs[c] * 2.0};
  for (int q = 0; q < 2; ++q) {
    const int32_t b = ora_nearest_bs(mtl, bs, n, mtl[c], targets[q], bs[c]);
    if (b < 0) continue;
    const int e = ora_find(mtl, bs, n, mtl[c], b);
    int dup = 0;
    for (int j = 0; j < k; ++j) dup |= out[j] == e;
    if (e >= 0 && !dup) out[k++] = e;
  }
  return k;
}

/* policy.py:218-273 select_sampling for one cap (caller validated budget >= 1, rounds >= 0,
 * cap >= 0). key/key_len: random.Random(seed)'s init_by_array key (seed_key). Returns the
 * caller index of the selection or -1 (IDLE_SELECTION); *count = len(feasible). */
int32_t ora_select_sampling(const int32_t* mtl, const int32_t* bs, const double* thr, const double* pw, int n,
                            int64_t budget_m, int64_t rounds_r, double cap, const uint32_t* key, int key_len,
                            int64_t* count) {
  ora_entry* f = (ora_entry*)malloc(sizeof(ora_entry) * (size_t)(n > 0 ? n : 1));
  int nf = 0;
  for (int i = 0; i < n; ++i) {
    if (!(pw[i] <= cap)) continue;
    f[nf].mtl = mtl[i]; f[nf].bs = bs[i]; f[nf].thr = thr[i]; f[nf].pw = pw[i]; f[nf].idx = i;
    ++nf;
  }
  *count = nf;
  if (nf == 0) { free(f); return -1; }
  qsort(f, (size_t)nf, sizeof(ora_entry), ora_qsort_cmp); /* policy.py:246 */
  int best;
  if (budget_m >= nf) {
    best = 0;
    for (int i = 1; i < nf; ++i) if (!ora_prefer_a(&f[best], &f[i])) best = i;
  } else {
    /* rng.sample(feasible, budget_m) (Lib/random.py Random.sample) */
    ora_mt rng;
    ora_mt_seed(&rng, key, key_len);
    const int64_t k = budget_m;
    int32_t* picked = (int32_t*)calloc((size_t)(k > 0 ? k : 1), sizeof(int32_t));
    if (nf <= ora_sample_setsize(k)) {
      int32_t* pool = (int32_t*)malloc(sizeof(int32_t) * (size_t)nf);
      for (int i = 0; i < nf; ++i) pool[i] = i;
      for (int64_t i = 0; i < k; ++i) {
        const uint32_t j = ora_randbelow(&rng, (uint32_t)(nf - i));
        picked[i] = pool[j];
        pool[j] = pool[nf - i - 1];
      }
      free(pool);
    } else {
      uint8_t* sel = (uint8_t*)calloc((size_t)nf, 1);
      for (int64_t i = 0; i < k; ++i) {
        uint32_t j = ora_randbelow(&rng, (uint32_t)nf);
        while (sel[j]) j = ora_randbelow(&rng, (uint32_t)nf);
        sel[j] = 1;
        picked[i] = (int32_t)j;
      }
      free(sel);
    }
    best = picked[0];
    for (int64_t i = 1; i < k; ++i) if (!ora_prefer_a(&f[best], &f[picked[i]])) best = picked[i];
    free(picked);
  }
  int cur = f[best].idx;
  free(f);
  /* hill climb (policy.py:255-266): best feasible strictly-better neighbour, until none */
  for (int64_t r = 0; r < rounds_r; ++r) {
    int nb[4];
    const int k = ora_neighbors(mtl, bs, n, cur, nb);
    int move = -1;
    for (int q = 0; q < k; ++q) {
      const int e = nb[q];
      if (pw[e] > cap || thr[e] <= thr[cur]) continue;
      if (move < 0) { move = e; continue; }
      ora_entry a = {mtl[move], bs[move], thr[move], pw[move], move};
      ora_entry b = {mtl[e], bs[e], thr[e], pw[e], e};
      if (!ora_prefer_a(&a, &b)) move = e;
    }
    if (move < 0) break;
    cur = move;
  }
  return cur;
}

/* ---- bench input generator (not a reference function) ------------------------------------
 * Host restatement of gen_kernel (paper_2306_12247_b200/csrc/aux_kernels.cu): the synthetic
 * solar / wind / iid cap traces of BASELINE.json's configs, a pure function of
 * (seed, global trace id). Every operation is exactly rounded IEEE fp32 or integer (built with
 * -ffp-contract=off; the kernel with -fmad=false), so this produces the device's traces bit for
 * bit and bench.py's reference arm times the reference algorithm on the engine arm's inputs. */
#define ORA_TRACE_SOLAR 0
#define ORA_TRACE_WIND 1
#define ORA_TRACE_MIXED 2
#define ORA_TRACE_IID 3
#define ORA_GEN_CHUNK 4096

static uint64_t ora_splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
static float ora_u01(uint64_t h) { return (float)(h >> 40) * (1.0f / 16777216.0f); }
static float ora_gauss(uint64_t h) {
  const float s = ora_u01(h) + ora_u01(h * 0x9E3779B97F4A7C15ull) + ora_u01(ora_splitmix(h)) +
                  ora_u01(ora_splitmix(h ^ 0xABCDull));  /* Irwin-Hall(4), unit variance */
  return (s - 2.0f) * 1.7320508f;
}
static float ora_clear_sky(float x) {
  const float w = 2.0f * x - 1.0f, z = w * w;
  float p = -2.52020424e-05f;
  p = p * z + 9.19260275e-04f;
  p = p * z - 2.08634808e-02f;
  p = p * z + 2.53669508e-01f;
  p = p * z - 1.23370055f;
  return p * z + 1.0f;
}

static void ora_generate_one(float* row, int64_t S, int64_t tid, int32_t step_seconds, int32_t kind, float peak,
                             uint64_t seed, float a_cloud) {
  const uint64_t hk = ora_splitmix(seed ^ ora_splitmix((uint64_t)tid));
  int k = kind;
  if (k == ORA_TRACE_MIXED) k = (tid & 1) ? ORA_TRACE_WIND : ORA_TRACE_SOLAR;
  const float var = 0.1f + 0.7f * ora_u01(ora_splitmix(hk ^ 1));
  const float phase = 86400.0f * ora_u01(ora_splitmix(hk ^ 2));
  const float dt = (float)step_seconds;
  const float wind_mu = 5.0f + 5.0f * ora_u01(ora_splitmix(hk ^ 3));
  const float theta = 1.0f / 7200.0f;
  const float cloud_sd = var * 0.5f * sqrtf(fmaxf(1.0f - a_cloud * a_cloud, 1e-6f));
  const float sdt = fminf(theta * dt, 1.0f);
  const float wind_sd = var * 4.0f * sqrtf(2.0f * sdt);
  for (int64_t c0 = 0; c0 < S; c0 += ORA_GEN_CHUNK) {
    const int64_t c1 = c0 + ORA_GEN_CHUNK < S ? c0 + ORA_GEN_CHUNK : S;
    const uint64_t hc = ora_splitmix(hk ^ (0xC0FFEEull + (uint64_t)(c0 / ORA_GEN_CHUNK)));
    float cloud = fminf(fmaxf(0.7f + var * 0.5f * ora_gauss(hc), 0.2f), 1.0f);
    float wind = fmaxf(wind_mu + var * 4.0f * 0.7f * ora_gauss(ora_splitmix(hc)), 0.0f);
    for (int64_t s = c0; s < c1; ++s) {
      const uint64_t hs = ora_splitmix(hk ^ (uint64_t)(s * 0x632BE59BD9B4E019ull));
      float v;
      if (k == ORA_TRACE_IID) {
        v = peak * ora_u01(hs);
      } else if (k == ORA_TRACE_SOLAR) {
        const float tod = fmodf(phase + (float)s * dt, 86400.0f) / 3600.0f;
        const float clear = (tod > 6.0f && tod < 18.0f) ? ora_clear_sky((tod - 6.0f) / 12.0f) : 0.0f;
        cloud = a_cloud * cloud + (1.0f - a_cloud) * 0.7f + cloud_sd * ora_gauss(hs);
        cloud = fminf(fmaxf(cloud, 0.2f), 1.0f);
        v = peak * clear * cloud;
      } else {
        wind = wind + sdt * (wind_mu - wind) + wind_sd * ora_gauss(hs);
        wind = fmaxf(wind, 0.0f);
        float f = 0.0f;
        if (wind >= 3.0f && wind < 25.0f) {
          const float r = (wind - 3.0f) / 9.0f;
          f = wind >= 12.0f ? 1.0f : r * r * r;
        }
        v = peak * f;
      }
      row[s] = fminf(fmaxf(v, 0.0f), peak);
    }
  }
}

typedef struct {
  float* caps;
  int64_t T, S, ld, first_id, next;
  int32_t step_seconds, kind;
  float peak, a_cloud;
  uint64_t seed;
  pthread_mutex_t mu;
} ora_gen_job;

static void* ora_gen_worker(void* arg) {
  ora_gen_job* j = (ora_gen_job*)arg;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    const int64_t t = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (t >= j->T) break;
    ora_generate_one(j->caps + t * j->ld, j->S, j->first_id + t, j->step_seconds, j->kind, j->peak, j->seed,
                     j->a_cloud);
  }
  return NULL;
}

/* caps: [T][ld] fp32 (columns >= S untouched). Same arguments as cs_generate_traces. */
int ora_generate_traces(float* caps, int64_t T, int64_t S, int64_t ld, int64_t first_id, int32_t step_seconds,
                        int32_t kind, float peak, uint64_t seed, int n_threads) {
  if (T < 0 || S < 0 || ld < S || step_seconds <= 0 || kind < 0 || kind > 3) return -1;
  ora_gen_job j;
  j.caps = caps; j.T = T; j.S = S; j.ld = ld; j.first_id = first_id; j.next = 0;
  j.step_seconds = step_seconds; j.kind = kind; j.peak = peak; j.seed = seed;
  j.a_cloud = (float)exp(-(double)step_seconds / 3600.0);
  pthread_mutex_init(&j.mu, NULL);
  if (n_threads < 1) n_threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
  for (int i = 0; i < n_threads; ++i) pthread_create(&th[i], NULL, ora_gen_worker, &j);
  for (int i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
  pthread_mutex_destroy(&j.mu);
  free(th);
  return 0;
}
