/*
 * capsim_b200.h — C ABI of the B200-native policy-evaluation engine (libcapsim_b200.so).
 *
 * The reference (capsim 0.1.0, pure Python) has no FFI: its boundary for this path is the
 * Python API re-exported from pkg/src/capsim/__init__.py:8-116. Each entry point below names
 * the reference function it replaces; paper_2306_12247_b200/_native.py is the ctypes
 * binding and the package's policy.py / sim.py mirror the reference signatures on top of it.
 *
 * Conventions
 *   - Every function returns int status: 0 = ok, < 0 = error (CS_E_*); the message of the
 *     last error on the calling thread is cs_last_error().
 *   - Plain pointers and sizes only. "dev" pointers are CUDA device pointers owned by the
 *     caller (PyTorch tensors used as buffers); "host" pointers are host memory. No entry
 *     point allocates device memory inside an evaluation call except cs_engine_* which owns
 *     its pinned/device staging buffers for the host-buffer path.
 *   - stream is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Policy index order everywhere: 0 = batching, 1 = multi-tenant, 2 = combination
 *     (PolicyTag, policy.py:25-29).
 */
#ifndef CAPSIM_B200_H
#define CAPSIM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CS_ABI_VERSION 1

#define CS_OK 0
#define CS_E_INVALID -1   /* bad argument (maps to ValueError / ValidationError) */
#define CS_E_CUDA -2      /* CUDA runtime error */
#define CS_E_NODEVICE -3  /* no usable sm_100 device */
#define CS_E_UNSUPPORTED -4

#define CS_CAP_F32 0 /* synthetic traces: fp32 caps, 4 B/timestep */
#define CS_CAP_F64 1 /* drop-in PowerTrace values: fp64 caps, 8 B/timestep */

#define CS_BATCHING 0
#define CS_MULTI_TENANT 1
#define CS_COMBINATION 2

/* cs_eval flags */
#define CS_FLAG_CHECK_VIOLATIONS 1u /* per-step power <= cap self-check (StepRecord, sim.py:50-54) */
#define CS_FLAG_ACCUMULATE_HIST 2u  /* add into hist_out instead of overwriting it */
#define CS_FLAG_SEGMENT_EPILOGUE 4u /* diagnostics: keep the segment epilogue where the per-bin one applies */
#define CS_FLAG_PREPARED 8u         /* workspace already holds this launch's value tables: a previous cs_eval
                                       with the same tables, n_traces, n_steps, step_seconds, penalty and
                                       flags wrote them into this workspace (and re-armed its scheduling
                                       counters); skip the prep kernel (graph replays) */

/* One profiling grid (ProfileGrid, profile.py:57-106): n entries Config(mtl, bs) -> (ips, W). */
typedef struct {
  int32_t n_entries;
  const int32_t* mtl;
  const int32_t* bs;
  const double* throughput_ips;
  const double* power_w;
  double idle_power_w; /* gpu_idle_power_w, or NaN when None (energy then uses 0 W, sim.py:175) */
} cs_grid_desc;

/* Per (trace, grid, policy) aggregate: SimReport's aggregates (sim.py:57-83, _aggregate sim.py:104-127). */
typedef struct {
  double avg_throughput_ips; /* fsum(ips)/num_steps, switch penalty applied (sim.py:119-126) */
  double energy_proxy_wh;    /* fsum((power or idle) * step_seconds / 3600) (sim.py:122,127) */
  int64_t idle_steps;        /* steps with no feasible config (sim.py:123-124) */
  int64_t switches;          /* steps i>0 whose config differs from step i-1 (sim.py:119) */
  int64_t violations;        /* steps whose selected power exceeds the cap: must be 0 (sim.py:50-54) */
  int64_t num_steps;
} cs_agg;

typedef struct {
  int32_t cap_dtype;
  int32_t n_grids;
  int32_t n_union_bins;    /* distinct thresholds over all grids + 1 */
  int32_t max_grid_bins;
  int32_t lut_entries;     /* level-1 + sub-tables */
  int32_t lut_shift;
  int32_t lut_level1;
  int32_t lut_subtables;
  int64_t device_bytes;    /* size of the staged device blob */
  int32_t lut_unsafe_leaves; /* fp32: LUT leaves whose selections are NOT proven to fit every cap
                                they serve (0 for well-formed tables; such leaves take the exact
                                per-step power check) */
  int32_t n_segments;      /* selection segments over all grids x policies */
  int32_t lut_big_entries; /* fp32: finer LUT that cs_eval stages when shared memory allows (0: none) */
  int32_t lut_big_shift;
  int32_t lut_big_unsafe_leaves;
  int32_t lut_huge_entries; /* fp32: finer still, for thousands of union thresholds (0: none) */
  int32_t lut_huge_shift;
  int32_t lut_huge_unsafe_leaves;
} cs_tables_info;

typedef struct cs_tables cs_tables;
typedef struct cs_engine cs_engine;

/* Evaluation of an exhaustive-policy sweep over a [n_traces x n_steps] cap matrix
 * (simulate(), sim.py:130-188, for every (trace, grid, policy) at once). */
typedef struct {
  const void* caps;        /* dev, [n_traces][ld] fp32 or fp64 (cap_dtype of the tables), 16-B aligned */
  int64_t n_traces;
  int64_t n_steps;
  int64_t ld;              /* row pitch in elements: multiple of 4 (fp32) / 2 (fp64), >= n_steps */
  int32_t step_seconds;    /* PowerTrace.step_seconds (> 0) */
  double switch_penalty_s; /* simulate(switch_penalty_s=...) (>= 0) */
  uint32_t flags;          /* CS_FLAG_* */
  uint16_t* step_bins;     /* dev, nullable: [n_traces][ld_bins] union bin per step (per-step mode) */
  int64_t ld_bins;
  cs_agg* agg;             /* dev, nullable: [n_traces][n_grids][3] */
  uint64_t* hist;          /* dev, nullable: [n_union_bins] steps per union bin over all traces */
  void* workspace;         /* dev, cs_eval_workspace_size() bytes (may be NULL when that is 0) */
  size_t workspace_bytes;
} cs_eval_args;

/* ---- errors / version ---- */
const char* cs_last_error(void);
int cs_abi_version(void);
/* Fills props: SM count, sm major/minor, smem per block; fails with CS_E_NODEVICE off-GPU. */
int cs_device_query(int32_t device, int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);

/* ---- N1 table staging: PolicyIndex.__init__ (policy.py:118-134) for all 3 regimes of all
 *      grids at once, merged into one union-threshold rank table + bucketed LUT ---- */
int cs_tables_create(const cs_grid_desc* grids, int32_t n_grids, int32_t cap_dtype, int32_t batching_mtl,
                     int32_t multi_tenant_bs, cs_tables** out);
int cs_tables_destroy(cs_tables* t);
int cs_tables_get_info(const cs_tables* t, cs_tables_info* out);
/* Host copies of the decoded selection per grid bin (the drop-in turns per-step bins into
 * Selection records with these): sel = entry index in the caller's order or -1 (idle),
 * count = feasible_count (policy.py:139-148). Arrays hold max_grid_bins elements. */
int cs_tables_grid_bins(const cs_tables* t, int32_t grid, int32_t policy, int32_t* sel, int64_t* count,
                        int32_t* n_bins);
/* union bin -> grid bin map for one grid (n_union_bins uint16). */
int cs_tables_union_map(const cs_tables* t, int32_t grid, uint16_t* out);
/* Host restatement of the device bin lookup (for CPU tests of the staged LUT). */
int cs_tables_lookup_host(const cs_tables* t, const void* caps, int64_t n, int32_t* bins_out);
/* Same through a chosen LUT size: which = 0 the default LUT, 1 the finer fp32 LUT cs_eval stages
 * when shared memory allows (CS_E_INVALID when the tables have none). */
int cs_tables_lookup_host_lut(const cs_tables* t, const void* caps, int64_t n, int32_t which, int32_t* bins_out);
/* Upload the staged blob to a device (idempotent per device). */
int cs_tables_upload(cs_tables* t, int32_t device);

/* ---- N2+N3 per-timestep policy kernel + accumulation (simulate + _aggregate) ---- */
int cs_eval_workspace_size(const cs_tables* t, const cs_eval_args* a, size_t* bytes);
int cs_eval(const cs_tables* t, const cs_eval_args* a, void* stream);
/* Device duration (ms) of the last cs_eval's main kernel launch on this thread, timed with
 * CUDA events on the launching stream (valid after that stream is synchronized). */
int cs_eval_last_kernel_ms(float* ms);
/* Number of kernels the last cs_eval launched. */
int cs_eval_last_launches(int32_t* n);
/* Launch plan of the last cs_eval on this thread (diagnostics / bench reporting). */
typedef struct {
  int32_t ctas, threads, warps_per_group, smem_bytes;
  int32_t trace_segments; /* > 1: long traces split across worker groups (+ finalize kernel) */
  int32_t lut_entries, lut_shift;
  int32_t epilogue;       /* 0 segment tables from global, 1 staged segment tables, 2 per-bin, 3/4 packed
                             penalty counters, per touched bin (segment values from global / staged) */
  int32_t redirect_uniform; /* 1: the warp-uniform redirect kernel variant (redirect-heavy fp32 LUTs) */
} cs_eval_plan;
int cs_eval_last_plan(cs_eval_plan* out);

/* ---- sweep totals (the aggregate statistics of a sharded Monte Carlo sweep) ----
 * Per (grid, policy) row of agg_dev [n_traces][n_rows] (n_rows = n_grids * 3), CS_SWEEP_WORDS u64:
 *   [0] steps  [1] idle steps  [2] switched steps  [3] violations
 *   [4..7]  sum over traces of avg_throughput_ips  } exact 128-bit fixed point (LSB 2^-50) as four
 *   [8..11] sum over traces of energy_proxy_wh     } 32-bit limbs, each summed separately in u64
 * Every word is an integer sum, so the cross-GPU reduction is one int64 SUM all-reduce (NCCL) or
 * peer-memory atomics, and the totals do not depend on how traces were sharded; the host
 * recombines value = (sum_k limb_k 2^(32k)) / 2^50 exactly and rounds once.
 * flags: CS_FLAG_ACCUMULATE_HIST adds into totals_dev instead of overwriting it (it may then
 * point into another device's memory with peer access enabled). */
#define CS_SWEEP_WORDS 12
int cs_sweep_totals(const cs_agg* agg_dev, int64_t n_traces, int32_t n_rows, uint64_t* totals_dev, uint32_t flags,
                    void* stream);

/* ---- single-process multi-GPU reduction of a sharded sweep (the
 *      survey's cs_nccl_init / cs_reduce / cs_nccl_destroy; north star (4): "a single NCCL reduce over
 *      NVLink for the aggregate statistics"). One NCCL communicator over this process's devices
 *      (ncclCommInitAll) and one grouped int64 SUM all-reduce, in place, of one buffer per device —
 *      the [union-bin histogram | cs_sweep_totals words] of that device's shard. NCCL is resolved at
 *      run time (libnccl.so.2); without it these return CS_E_UNSUPPORTED. The reference has no
 *      multi-GPU path: its sweeps are Python loops over (trace, grid, policy) (sim.py:130-188). ---- */
typedef struct cs_comm cs_comm;
int cs_comm_init_all(int32_t n_devices, const int32_t* devices, cs_comm** out);
int cs_comm_size(const cs_comm* c, int32_t* n_devices);
/* bufs[i] / streams[i] (nullable: default stream) belong to devices[i] of cs_comm_init_all */
int cs_comm_allreduce_i64(cs_comm* c, int64_t* const* bufs, int64_t count, void* const* streams);
int cs_comm_destroy(cs_comm* c);

/* ---- per-cap API: select_config (policy.py:172-188) and feasible_set (policy.py:151-169) as
 *      warp-per-query argmax (shuffle) / ballot kernels over the grid's raw entries ---- */
int cs_select_caps(const cs_tables* t, int32_t grid, int32_t policy, const double* caps_dev, int64_t n,
                   int32_t* sel_dev, int64_t* count_dev, void* stream);
/* words_per_cap = ceil(n_entries/32); bit j of word w set <=> entry 32w+j is feasible. */
int cs_feasible_caps(const cs_tables* t, int32_t grid, int32_t policy, const double* caps_dev, int64_t n,
                     uint32_t* mask_dev, void* stream);

/* ---- host-buffer end-to-end path: pinned staging, H2D/compute/D2H overlapped on 2 streams ---- */
int cs_engine_create(int32_t device, int64_t chunk_traces_max, int64_t n_steps_max, int32_t cap_dtype,
                     cs_engine** out);
int cs_engine_destroy(cs_engine* e);
/* caps_host: [n_traces][ld] host memory; agg_host: [n_traces][n_grids][3]; hist_host:
 * [n_union_bins] (nullable). Blocks until results are in host memory. */
int cs_engine_eval_host(cs_engine* e, const cs_tables* t, const void* caps_host, int64_t n_traces, int64_t n_steps,
                        int64_t ld, int32_t step_seconds, double switch_penalty_s, uint32_t flags, cs_agg* agg_host,
                        uint64_t* hist_host, int64_t* h2d_bytes, int64_t* d2h_bytes);

/* ---- online controller replay: controller.replay (controller.py:161-231), one thread per trace ---- */
#define CS_CTRL_REACTIVE 0
#define CS_CTRL_PROACTIVE 1
#define CS_CTRL_TIME_MAJOR 256 /* OR into mode: caps_dev is [n_steps][ld] (ld >= n_traces), coalesced per step */
typedef struct {
  double measured_power_w; /* power fed to the step (selection's power x seeded noise) */
  uint16_t bin_reactive;   /* grid bin of the selection after the reactive part (0xFFFF: initial config) */
  uint16_t bin_final;      /* grid bin of the selection after the step */
  uint8_t kind_bits;       /* bit0: VIOLATION_DETECTED + RECONFIGURED; bit1: PREEMPTIVE_RECONFIGURED */
  uint8_t pad[3];
} cs_replay_step;
typedef struct {
  int64_t violations;        /* ControllerReport.violations */
  int64_t reconfigs;         /* ControllerReport.reconfigs */
  double violation_fraction; /* violations / num_steps */
  double avg_throughput_ips; /* fsum(post-step throughput) / num_steps */
  int64_t num_steps;
} cs_replay_agg;
/* caps_dev: fp64 [n_traces][ld] (tables staged with CS_CAP_F64); initial_dev: nullable int32
 * [n_traces] entry index per trace (-1: select_config(first cap)); noise: random.Random(seed)
 * with seed = keys (abs(seed) 32-bit words, key_len words per trace) or, when keys is NULL,
 * seed_base + trace index. steps_dev nullable [n_traces][n_steps]. */
int cs_replay(const cs_tables* t, int32_t grid, const double* caps_dev, int64_t n_traces, int64_t n_steps, int64_t ld,
              int32_t mode, int32_t window_k, const int32_t* initial_dev, double noise_pct, const uint32_t* keys_dev,
              const int32_t* key_len_dev, int32_t key_stride, uint64_t seed_base, cs_replay_step* steps_dev,
              cs_replay_agg* agg_dev, void* stream);

/* ---- sampling selector: select_sampling (policy.py:218-273) at every (trace, step) ---- */
#define CS_SAMPLING_MAX_BUDGET 256
/* caps_dev: fp64 [n_traces][ld] (tables staged with CS_CAP_F64). Step i of every trace samples
 * with random.Random(seed_base + i), seed_base the signed 128-bit integer seed_hi:seed_lo;
 * simulate() passes seed * 1_000_003 (sim.py:159-163), select_sampling(seed) one step with
 * seed_base = seed. out_entry_dev: int32 [n_traces][n_steps] caller entry index or -1 (idle);
 * out_count_dev (nullable): int32 feasible_count. budget_m >= 1, rounds_r >= 0. Budgets up to
 * CS_SAMPLING_MAX_BUDGET keep the sample in registers/local memory; larger ones (below the grid
 * size) run a slower variant with a stream-ordered scratch pool (cudaMallocAsync). */
int cs_select_sampling(const cs_tables* t, int32_t grid, const double* caps_dev, int64_t n_traces, int64_t n_steps,
                       int64_t ld, int64_t budget_m, int64_t rounds_r, uint64_t seed_lo, int64_t seed_hi,
                       int32_t* out_entry_dev, int32_t* out_count_dev, void* stream);

/* _aggregate (sim.py:104-127) of per-step entry selections on the device (the summary reports of
 * simulate_many with a sampling policy): entry_dev int32 [n_traces][ld] caller entry index or -1
 * (idle); values_dev f64 [3][n_entries + 1][2] per entry {hi, lo} of thr, penalised thr
 * (thr * (1 - penalty_frac)) and energy ((power or idle power) * step / 3600), index n_entries =
 * idle, each split so that the sum of hi is exact; outputs per trace the
 * average throughput (fsum(ips) / n), the energy and the idle-step count. */
int cs_entries_aggregate(const int32_t* entry_dev, int64_t n_traces, int64_t n_steps, int64_t ld,
                         const double* values_dev, int32_t n_entries, double penalty_frac, double* avg_dev,
                         double* energy_dev, int64_t* idle_dev, void* stream);

/* ---- synthetic traces for benchmarks (counter-based, keyed by (seed, global trace id)) ---- */
#define CS_TRACE_SOLAR 0
#define CS_TRACE_WIND 1
#define CS_TRACE_MIXED 2   /* even global ids solar, odd wind */
#define CS_TRACE_IID 3     /* iid uniform(0, peak) adversarial variant */
int cs_generate_traces(float* caps_dev, int64_t n_traces, int64_t n_steps, int64_t ld, int64_t first_trace_id,
                       int32_t step_seconds, int32_t kind, float peak_w, uint64_t seed, void* stream);

/* ---- low-latency per-cap queries from host memory (the scalar drop-in API) ----
 * caps_host: n fp64 caps. CS_QUERY_BINS: out int32 [n] union bin per cap (PolicyIndex.select,
 * policy.py:136-148, decoded per regime with cs_tables_grid_bins); CS_QUERY_SELECT: out int32 [n]
 * entry or -1, out2 int64 [n] feasible_count (select_config, policy.py:172-188);
 * CS_QUERY_FEASIBLE: out uint32 [n][ceil(entries/32)] bitmask (feasible_set, policy.py:151-169).
 * One H2D, one kernel, one D2H and one sync per call through per-thread pinned staging buffers. */
#define CS_QUERY_BINS 0
#define CS_QUERY_SELECT 1
#define CS_QUERY_FEASIBLE 2
int cs_query_host(const cs_tables* t, int32_t query, int32_t grid, int32_t policy, const double* caps_host,
                  int64_t n, void* out_host, void* out2_host);

/* ---- trace ingestion fast path (load_trace, trace.py:87-169) ----
 * CSV text -> fp64 samples on the host with the reference's rules (header, blank rows, 2
 * fields, ISO-8601 UTC timestamps on the step grid, finite non-negative capacities, whole-step
 * gaps forward-filled only with gap_fill). The native grammar is narrow (ASCII; timestamps
 * YYYY-MM-DD(T| )HH:MM:SS[.f{1,6}][Z|z|+00:00|-00:00]; plain decimal capacities): a file inside
 * it parses to exactly the reference's samples (status CS_OK); anything else, including every
 * error, reports CS_E_UNSUPPORTED in its info and the caller applies the reference rules
 * itself (paper_2306_12247_b200/trace.py) to produce the identical outcome or exception. */
typedef struct cs_traces cs_traces; /* parsed traces (host memory, library-owned) */
typedef struct {
  int64_t n_values;      /* samples after forward-fill (len(PowerTrace.values)) */
  int64_t start_unix_us; /* first row's UTC timestamp (PowerTrace.start_time), us since 1970-01-01 */
  int32_t status;        /* CS_OK or CS_E_UNSUPPORTED (see above) */
  int32_t line;          /* 1-based line where the native parser stopped (status != CS_OK) */
} cs_trace_info;
/* n files, parsed on n_threads host threads (<= 0: all hardware threads). */
int cs_traces_parse_files(const char* const* paths, int32_t n, int64_t step_seconds, int32_t gap_fill,
                          int32_t n_threads, cs_traces** out);
int cs_traces_parse_text(const char* text, int64_t len, int64_t step_seconds, int32_t gap_fill, cs_traces** out);
int cs_traces_info(const cs_traces* t, int32_t i, cs_trace_info* info);
int cs_traces_copy(const cs_traces* t, int32_t i, double* out); /* n_values doubles */
/* All traces (each CS_OK with n_steps samples) into a row-major [n][ld] host matrix of CS_CAP_F32
 * (round to nearest) or CS_CAP_F64; columns n_steps..ld-1 are zeroed. */
int cs_traces_pack(const cs_traces* t, int32_t dtype, int64_t n_steps, int64_t ld, void* out, int32_t n_threads);
void cs_traces_destroy(cs_traces* t);

#ifdef __cplusplus
}
#endif

#endif /* CAPSIM_B200_H */
