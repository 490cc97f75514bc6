// C-ABI glue: error reporting, table upload, argument validation and the host-buffer engine.
// Each entry point's reference counterpart is documented in include/capsim_b200.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <new>
#include <string>

#include "cs_internal.h"

#include <vector_types.h>
namespace cs {
std::string launch_lookup(const DevTables& v, const double* caps, int64_t n, int32_t* bins, cudaStream_t st);
}  // namespace cs
namespace cs {
std::string launch_entries_agg(const int32_t* ent, int64_t T, int64_t S, int64_t ld, const double2* vals, int n,
                               double pf, double* avg, double* energy, int64_t* idle, cudaStream_t st);
}  // namespace cs

namespace cs {
std::string launch_eval(const Tables& t, const DevTables& view, const cs_eval_args* a, int dev, cudaStream_t st);
std::string eval_workspace(const Tables& t, const DevTables& view, const cs_eval_args* a, int dev, size_t* bytes);
std::string last_kernel_ms(float* ms);
int last_launches();
cs_eval_plan last_plan();
std::string launch_select(const DevTables& v, int g, int p, const double* caps, int64_t n, int32_t* sel, int64_t* cnt,
                          cudaStream_t st);
std::string launch_feasible(const DevTables& v, int g, int p, const double* caps, int64_t n, uint32_t* mask,
                            cudaStream_t st);
std::string launch_sampling(const DevTables& v, int g, const double* caps, int64_t T, int64_t S, int64_t ld,
                            int64_t budget, int64_t rounds, unsigned long long seed_lo, long long seed_hi,
                            int32_t* out_entry, int32_t* out_count, int n_entries, int sm_count, cudaStream_t st);
std::string launch_replay(const DevTables& v, int g, const double* caps, int64_t T, int64_t S, int64_t ld, int mode,
                          int window_k, const int32_t* initial, double noise_pct, const uint32_t* keys,
                          const int32_t* key_len, int key_stride, unsigned long long seed_base, cs_replay_step* steps,
                          cs_replay_agg* agg, cudaStream_t st);
std::string launch_sweep_totals(const cs_agg* agg, int64_t T, int rows, uint64_t* out, bool accumulate, int sms,
                                cudaStream_t st);
std::string launch_generate(float* caps, int64_t T, int64_t S, int64_t ld, int64_t first_id, int32_t step_seconds,
                            int32_t kind, float peak, uint64_t seed, cudaStream_t st);

namespace {
thread_local std::string g_err;
std::mutex g_upload_mu;
}  // namespace

void set_error(const std::string& msg) { g_err = msg; }

static int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

#define CS_CUDA_RET(x)                                                                            \
  do {                                                                                            \
    cudaError_t e_ = (x);                                                                         \
    if (e_ != cudaSuccess) return fail(CS_E_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + " (" #x ")"); \
  } while (0)

static size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

// Copies the staged tables into one device allocation and fills the DevTables view.
static int upload(Tables& t, int device, Tables::Dev** out) {
  std::lock_guard<std::mutex> lk(g_upload_mu);
  for (auto& d : t.devs)
    if (d.device == device) {
      *out = &d;
      return CS_OK;
    }
  const bool f64 = t.cap_dtype == CS_CAP_F64;
  struct Part {
    const void* src;
    size_t bytes;
    size_t off;
  };
  std::vector<uint64_t> thr64 = f64 ? t.thresholds : std::vector<uint64_t>(1, 0);
  Part parts[] = {
      {t.lut.data(), t.lut.size() * 4, 0},
      {thr64.data(), thr64.size() * 8, 0},
      {t.vio.data(), t.vio.size() * 8, 0},
      {t.sig.data(), t.sig.size() * 8, 0},
      {t.umap.data(), t.umap.size() * 2, 0},
      {t.sel.data(), t.sel.size() * 4, 0},
      {t.sthr.data(), t.sthr.size() * 8, 0},
      {t.spw.data(), t.spw.size() * 8, 0},
      {t.idle_pw.data(), t.idle_pw.size() * 8, 0},
      {t.e_off.data(), t.e_off.size() * 4, 0},
      {t.e_mtl.data(), t.e_mtl.size() * 4, 0},
      {t.e_bs.data(), t.e_bs.size() * 4, 0},
      {t.e_thr.data(), t.e_thr.size() * 8, 0},
      {t.e_pw.data(), t.e_pw.size() * 8, 0},
      {t.seg_off.data(), t.seg_off.size() * 4, 0},
      {t.seg.data(), t.seg.size() * 4, 0},
      {t.csort.data(), t.csort.size() * 4, 0},
      {t.ccnt.data(), t.ccnt.size() * 4, 0},
      {t.nbr.data(), t.nbr.size() * 4, 0},
      {t.lut_big.lut.data(), t.lut_big.lut.size() * 4, 0},
      {t.lut_huge.lut.data(), t.lut_huge.lut.size() * 4, 0},
  };
  size_t total = 0;
  for (auto& p : parts) {
    p.off = total;
    total += align16(p.bytes);
  }
  int prev = 0;
  CS_CUDA_RET(cudaGetDevice(&prev));
  CS_CUDA_RET(cudaSetDevice(device));
  std::vector<unsigned char> host(total, 0);
  for (auto& p : parts) std::memcpy(host.data() + p.off, p.src, p.bytes);
  void* blob = nullptr;
  cudaError_t e = cudaMalloc(&blob, total);
  if (e == cudaSuccess) e = cudaMemcpy(blob, host.data(), total, cudaMemcpyHostToDevice);
  // a pageable-source cudaMemcpy may return before its DMA lands, ordered only on the legacy
  // stream; the query / host-engine streams are non-blocking, so wait for it here (once per
  // device upload) — a select launched right after staging read a half-written blob
  if (e == cudaSuccess) e = cudaStreamSynchronize(cudaStreamLegacy);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    if (blob) cudaFree(blob);
    return fail(CS_E_CUDA, std::string("CUDA error uploading tables: ") + cudaGetErrorString(e));
  }
  auto* b = reinterpret_cast<unsigned char*>(blob);
  Tables::Dev d;
  d.device = device;
  d.blob = blob;
  d.bytes = total;
  DevTables& v = d.view;
  v.cap_dtype = t.cap_dtype;
  v.M = t.M;
  v.U = t.U;
  v.maxB = t.maxB;
  v.n_lut = (int32_t)t.lut.size();
  v.n_level1 = (int32_t)t.n_level1;
  v.batching_mtl = t.batching_mtl;
  v.mt_bs = t.mt_bs;
  v.lv.lo = t.lo;
  v.lv.hi = t.hi;
  v.lv.kbase = t.kbase;
  v.lv.shift1 = t.shift1;
  v.lv.sub0 = t.n_level1;
  v.lv.lut = reinterpret_cast<const uint32_t*>(b + parts[0].off);
  v.lv.thr64 = reinterpret_cast<const uint64_t*>(b + parts[1].off);
  v.vio = reinterpret_cast<const uint64_t*>(b + parts[2].off);
  v.sig = reinterpret_cast<const uint64_t*>(b + parts[3].off);
  v.umap = reinterpret_cast<const uint16_t*>(b + parts[4].off);
  v.sel = reinterpret_cast<const int32_t*>(b + parts[5].off);
  v.sthr = reinterpret_cast<const double*>(b + parts[6].off);
  v.spw = reinterpret_cast<const double*>(b + parts[7].off);
  v.idle_pw = reinterpret_cast<const double*>(b + parts[8].off);
  v.e_off = reinterpret_cast<const int32_t*>(b + parts[9].off);
  v.e_mtl = reinterpret_cast<const int32_t*>(b + parts[10].off);
  v.e_bs = reinterpret_cast<const int32_t*>(b + parts[11].off);
  v.e_thr = reinterpret_cast<const double*>(b + parts[12].off);
  v.e_pw = reinterpret_cast<const double*>(b + parts[13].off);
  v.seg_off = reinterpret_cast<const int32_t*>(b + parts[14].off);
  v.seg = reinterpret_cast<const int4*>(b + parts[15].off);
  v.csort = reinterpret_cast<const int32_t*>(b + parts[16].off);
  v.ccnt = reinterpret_cast<const int32_t*>(b + parts[17].off);
  v.nbr = reinterpret_cast<const int32_t*>(b + parts[18].off);
  v.n_lut_big = (int32_t)t.lut_big.lut.size();
  v.n_level1_big = (int32_t)t.lut_big.n_level1;
  v.lv_big = v.lv;
  if (v.n_lut_big) {
    v.lv_big.kbase = t.lut_big.kbase;
    v.lv_big.shift1 = t.lut_big.shift1;
    v.lv_big.sub0 = t.lut_big.n_level1;
    v.lv_big.lut = reinterpret_cast<const uint32_t*>(b + parts[19].off);
  }
  v.n_lut_huge = (int32_t)t.lut_huge.lut.size();
  v.n_level1_huge = (int32_t)t.lut_huge.n_level1;
  v.lv_huge = v.lv;
  if (v.n_lut_huge) {
    v.lv_huge.kbase = t.lut_huge.kbase;
    v.lv_huge.shift1 = t.lut_huge.shift1;
    v.lv_huge.sub0 = t.lut_huge.n_level1;
    v.lv_huge.lut = reinterpret_cast<const uint32_t*>(b + parts[20].off);
  }
  t.devs.push_back(d);
  *out = &t.devs.back();
  return CS_OK;
}

static int current_view(const cs_tables* tp, Tables::Dev** out, int* dev) {
  if (!tp) return fail(CS_E_INVALID, "null tables");
  Tables& t = *reinterpret_cast<Tables*>(const_cast<cs_tables*>(tp));
  int d = 0;
  CS_CUDA_RET(cudaGetDevice(&d));
  *dev = d;
  return upload(t, d, out);
}

}  // namespace cs

using cs::fail;
using cs::Tables;

extern "C" {

const char* cs_last_error(void) { return cs::g_err.c_str(); }

int cs_abi_version(void) { return CS_ABI_VERSION; }

int cs_device_query(int32_t device, int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return fail(CS_E_NODEVICE, "no CUDA device visible");
  if (device < 0 || device >= n) return fail(CS_E_INVALID, "device ordinal out of range");
  cudaDeviceProp p;
  CS_CUDA_RET(cudaGetDeviceProperties(&p, device));
  if (sm_count) *sm_count = p.multiProcessorCount;
  if (cc_major) *cc_major = p.major;
  if (cc_minor) *cc_minor = p.minor;
  if (p.major != 10) return fail(CS_E_NODEVICE, "libcapsim_b200 is built for sm_100a (B200); found sm_" +
                                                   std::to_string(p.major) + std::to_string(p.minor));
  return CS_OK;
}

int cs_tables_create(const cs_grid_desc* grids, int32_t n_grids, int32_t cap_dtype, int32_t batching_mtl,
                     int32_t multi_tenant_bs, cs_tables** out) {
  if (!out) return fail(CS_E_INVALID, "null output pointer");
  Tables* t = new (std::nothrow) Tables();
  if (!t) return fail(CS_E_INVALID, "out of host memory");
  std::string err = cs::build_tables(grids, n_grids, cap_dtype, batching_mtl, multi_tenant_bs, *t);
  if (!err.empty()) {
    delete t;
    return fail(CS_E_INVALID, err);
  }
  *out = reinterpret_cast<cs_tables*>(t);
  return CS_OK;
}

int cs_tables_destroy(cs_tables* tp) {
  if (!tp) return CS_OK;
  Tables* t = reinterpret_cast<Tables*>(tp);
  for (auto& d : t->devs) {
    int prev = 0;
    if (cudaGetDevice(&prev) == cudaSuccess && cudaSetDevice(d.device) == cudaSuccess) {
      cudaFree(d.blob);
      cudaSetDevice(prev);
    }
  }
  delete t;
  return CS_OK;
}

int cs_tables_get_info(const cs_tables* tp, cs_tables_info* o) {
  if (!tp || !o) return fail(CS_E_INVALID, "null argument");
  const Tables& t = *reinterpret_cast<const Tables*>(tp);
  o->cap_dtype = t.cap_dtype;
  o->n_grids = t.M;
  o->n_union_bins = t.U;
  o->max_grid_bins = t.maxB;
  o->lut_entries = (int32_t)t.lut.size();
  o->lut_shift = (int32_t)t.shift1;
  o->lut_level1 = (int32_t)t.n_level1;
  o->lut_subtables = (int32_t)t.n_sub;
  o->device_bytes = t.devs.empty() ? 0 : (int64_t)t.devs.front().bytes;
  o->lut_unsafe_leaves = (int32_t)t.n_unsafe;
  o->n_segments = (int32_t)(t.seg.size() / 4);
  o->lut_big_entries = (int32_t)t.lut_big.lut.size();
  o->lut_big_shift = (int32_t)t.lut_big.shift1;
  o->lut_big_unsafe_leaves = (int32_t)t.lut_big.n_unsafe;
  o->lut_huge_entries = (int32_t)t.lut_huge.lut.size();
  o->lut_huge_shift = (int32_t)t.lut_huge.shift1;
  o->lut_huge_unsafe_leaves = (int32_t)t.lut_huge.n_unsafe;
  return CS_OK;
}

int cs_tables_grid_bins(const cs_tables* tp, int32_t grid, int32_t policy, int32_t* sel, int64_t* count,
                        int32_t* n_bins) {
  if (!tp) return fail(CS_E_INVALID, "null tables");
  const Tables& t = *reinterpret_cast<const Tables*>(tp);
  if (grid < 0 || grid >= t.M || policy < 0 || policy > 2) return fail(CS_E_INVALID, "grid/policy out of range");
  const size_t o = ((size_t)grid * 3 + policy) * t.maxB;
  const int B = t.grid_bins[grid];
  if (sel) std::memcpy(sel, t.sel.data() + o, (size_t)B * 4);
  if (count) std::memcpy(count, t.cnt.data() + o, (size_t)B * 8);
  if (n_bins) *n_bins = B;
  return CS_OK;
}

int cs_tables_union_map(const cs_tables* tp, int32_t grid, uint16_t* out) {
  if (!tp || !out) return fail(CS_E_INVALID, "null argument");
  const Tables& t = *reinterpret_cast<const Tables*>(tp);
  if (grid < 0 || grid >= t.M) return fail(CS_E_INVALID, "grid out of range");
  std::memcpy(out, t.umap.data() + (size_t)grid * t.U, (size_t)t.U * 2);
  return CS_OK;
}

int cs_tables_lookup_host_lut(const cs_tables* tp, const void* caps, int64_t n, int32_t which, int32_t* bins_out) {
  if (!tp || (n > 0 && (!caps || !bins_out))) return fail(CS_E_INVALID, "null argument");
  const Tables& t = *reinterpret_cast<const Tables*>(tp);
  if (which == 0) return cs_tables_lookup_host(tp, caps, n, bins_out);
  const Tables::Lut& L = which == 2 ? t.lut_huge : t.lut_big;
  if ((which != 1 && which != 2) || L.lut.empty()) return fail(CS_E_INVALID, "no such LUT");
  if (t.cap_dtype == CS_CAP_F32) {
    const uint32_t* c = reinterpret_cast<const uint32_t*>(caps);
    for (int64_t i = 0; i < n; ++i)
      bins_out[i] = (int32_t)cs::bin_f32(c[i], L.shift1, (int32_t)L.kbase, (int32_t)L.n_level1, L.n_level1,
                                         L.lut.data());
  } else {
    const uint64_t* c = reinterpret_cast<const uint64_t*>(caps);
    for (int64_t i = 0; i < n; ++i)
      bins_out[i] = (int32_t)cs::bin_f64(c[i], t.lo, t.hi, L.shift1, L.kbase, L.n_level1, L.lut.data(),
                                         t.thresholds.data());
  }
  return CS_OK;
}

int cs_tables_lookup_host(const cs_tables* tp, const void* caps, int64_t n, int32_t* bins_out) {
  if (!tp || (n > 0 && (!caps || !bins_out))) return fail(CS_E_INVALID, "null argument");
  const Tables& t = *reinterpret_cast<const Tables*>(tp);
  if (t.cap_dtype == CS_CAP_F32) {
    const uint32_t* c = reinterpret_cast<const uint32_t*>(caps);
    for (int64_t i = 0; i < n; ++i)
      bins_out[i] = (int32_t)cs::bin_f32(c[i], t.shift1, (int32_t)t.kbase, (int32_t)t.n_level1, t.n_level1,
                                         t.lut.data());
  } else {
    const uint64_t* c = reinterpret_cast<const uint64_t*>(caps);
    for (int64_t i = 0; i < n; ++i)
      bins_out[i] =
          (int32_t)cs::bin_f64(c[i], t.lo, t.hi, t.shift1, t.kbase, t.n_level1, t.lut.data(), t.thresholds.data());
  }
  return CS_OK;
}

int cs_tables_upload(cs_tables* tp, int32_t device) {
  if (!tp) return fail(CS_E_INVALID, "null tables");
  Tables::Dev* d = nullptr;
  return cs::upload(*reinterpret_cast<Tables*>(tp), device, &d);
}

static int check_eval_args(const Tables& t, const cs_eval_args* a) {
  if (!a) return fail(CS_E_INVALID, "null args");
  if (a->n_traces < 0 || a->n_steps < 0) return fail(CS_E_INVALID, "negative sizes");
  if (a->n_traces > 0 && a->n_steps == 0) return fail(CS_E_INVALID, "cannot simulate an empty trace");
  if (a->step_seconds <= 0) return fail(CS_E_INVALID, "step_seconds must be positive");
  if (!(a->switch_penalty_s >= 0.0)) return fail(CS_E_INVALID, "switch_penalty_s must be >= 0");
  const int vec = t.cap_dtype == CS_CAP_F32 ? 4 : 2;
  if (a->ld < a->n_steps || a->ld % vec) return fail(CS_E_INVALID, "ld must be >= n_steps and a multiple of 16 bytes");
  if (a->n_traces > 0 && (!a->caps || (reinterpret_cast<uintptr_t>(a->caps) & 15)))
    return fail(CS_E_INVALID, "caps must be a 16-byte aligned device pointer");
  if (a->step_bins && (a->ld_bins < a->n_steps || a->ld_bins % 4 || (reinterpret_cast<uintptr_t>(a->step_bins) & 7)))
    return fail(CS_E_INVALID, "step_bins needs ld_bins >= n_steps, a multiple of 4, 8-byte alignment");
  return CS_OK;
}

int cs_eval_workspace_size(const cs_tables* tp, const cs_eval_args* a, size_t* bytes) {
  if (!bytes) return fail(CS_E_INVALID, "null argument");
  Tables::Dev* d = nullptr;
  int dev = 0;
  int rc = cs::current_view(tp, &d, &dev);
  if (rc) return rc;
  const Tables& t = *reinterpret_cast<const Tables*>(tp);
  if ((rc = check_eval_args(t, a))) return rc;
  std::string err = cs::eval_workspace(t, d->view, a, dev, bytes);
  if (!err.empty()) return fail(CS_E_INVALID, err);
  return CS_OK;
}

int cs_eval(const cs_tables* tp, const cs_eval_args* a, void* stream) {
  Tables::Dev* d = nullptr;
  int dev = 0;
  int rc = cs::current_view(tp, &d, &dev);
  if (rc) return rc;
  const Tables& t = *reinterpret_cast<const Tables*>(tp);
  if ((rc = check_eval_args(t, a))) return rc;
  if (a->n_traces == 0) {  // no work, but an overwritten histogram must still read all-zero
    if (a->hist && !(a->flags & CS_FLAG_ACCUMULATE_HIST))
      CS_CUDA_RET(cudaMemsetAsync(a->hist, 0, (size_t)t.U * 8, reinterpret_cast<cudaStream_t>(stream)));
    return CS_OK;
  }
  std::string err = cs::launch_eval(t, d->view, a, dev, reinterpret_cast<cudaStream_t>(stream));
  if (!err.empty()) return fail(err.rfind("CUDA", 0) == 0 ? CS_E_CUDA : CS_E_INVALID, err);
  return CS_OK;
}

int cs_sweep_totals(const cs_agg* agg_dev, int64_t n_traces, int32_t n_rows, uint64_t* totals_dev, uint32_t flags,
                    void* stream) {
  if (n_traces < 0 || n_rows < 1 || !totals_dev || (n_traces > 0 && !agg_dev))
    return fail(CS_E_INVALID, "bad sweep arguments");
  int dev = 0, sms = 148;
  CS_CUDA_RET(cudaGetDevice(&dev));
  CS_CUDA_RET(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  std::string err = cs::launch_sweep_totals(agg_dev, n_traces, n_rows, totals_dev,
                                            (flags & CS_FLAG_ACCUMULATE_HIST) != 0, sms,
                                            reinterpret_cast<cudaStream_t>(stream));
  if (!err.empty()) return fail(CS_E_CUDA, err);
  return CS_OK;
}

int cs_eval_last_kernel_ms(float* ms) {
  if (!ms) return fail(CS_E_INVALID, "null argument");
  std::string err = cs::last_kernel_ms(ms);
  if (!err.empty()) return fail(CS_E_CUDA, err);
  return CS_OK;
}

int cs_eval_last_launches(int32_t* n) {
  if (!n) return fail(CS_E_INVALID, "null argument");
  *n = cs::last_launches();
  return CS_OK;
}

int cs_eval_last_plan(cs_eval_plan* out) {
  if (!out) return fail(CS_E_INVALID, "null argument");
  *out = cs::last_plan();
  return CS_OK;
}

int cs_select_caps(const cs_tables* tp, int32_t grid, int32_t policy, const double* caps_dev, int64_t n,
                   int32_t* sel_dev, int64_t* count_dev, void* stream) {
  Tables::Dev* d = nullptr;
  int dev = 0;
  int rc = cs::current_view(tp, &d, &dev);
  if (rc) return rc;
  if (grid < 0 || grid >= d->view.M || policy < 0 || policy > 2) return fail(CS_E_INVALID, "grid/policy out of range");
  std::string err = cs::launch_select(d->view, grid, policy, caps_dev, n, sel_dev, count_dev,
                                      reinterpret_cast<cudaStream_t>(stream));
  if (!err.empty()) return fail(CS_E_CUDA, err);
  return CS_OK;
}

// Low-latency host-buffer queries for the per-cap API: the caps go through a per-thread pinned
// staging buffer on a per-thread stream (one H2D, one launch, one D2H, one sync per call).
namespace {
struct QueryStage {
  int device = -1;
  cudaStream_t st = nullptr;
  unsigned char* hpin = nullptr;
  unsigned char* dbuf = nullptr;
  size_t cap = 0;  // (not freed at thread exit: the CUDA runtime may already be torn down)
};
thread_local QueryStage g_qs;

int query_stage(int dev, size_t bytes) {
  if (g_qs.device != dev) {
    if (g_qs.st) cudaStreamDestroy(g_qs.st), g_qs.st = nullptr;
    if (g_qs.hpin) cudaFreeHost(g_qs.hpin), g_qs.hpin = nullptr;
    if (g_qs.dbuf) cudaFree(g_qs.dbuf), g_qs.dbuf = nullptr;
    g_qs.cap = 0;
    CS_CUDA_RET(cudaStreamCreateWithFlags(&g_qs.st, cudaStreamNonBlocking));
    g_qs.device = dev;
  }
  if (g_qs.cap < bytes) {
    size_t c = std::max<size_t>(bytes, 1 << 16);
    if (g_qs.hpin) cudaFreeHost(g_qs.hpin), g_qs.hpin = nullptr;
    if (g_qs.dbuf) cudaFree(g_qs.dbuf), g_qs.dbuf = nullptr;
    g_qs.cap = 0;
    CS_CUDA_RET(cudaMallocHost(&g_qs.hpin, c));
    CS_CUDA_RET(cudaMalloc(&g_qs.dbuf, c));
    g_qs.cap = c;
  }
  return CS_OK;
}
}  // namespace

int cs_query_host(const cs_tables* tp, int32_t query, int32_t grid, int32_t policy, const double* caps_host,
                  int64_t n, void* out_host, void* out2_host) {
  if (n < 0 || (n > 0 && (!caps_host || !out_host))) return fail(CS_E_INVALID, "null argument");
  if (n == 0) return CS_OK;
  Tables::Dev* d = nullptr;
  int dev = 0;
  int rc = cs::current_view(tp, &d, &dev);
  if (rc) return rc;
  const Tables& t = *reinterpret_cast<const Tables*>(tp);
  if (query != CS_QUERY_BINS && (grid < 0 || grid >= d->view.M || policy < 0 || policy > 2))
    return fail(CS_E_INVALID, "grid/policy out of range");
  const int64_t ne = query == CS_QUERY_FEASIBLE ? t.e_off[grid + 1] - t.e_off[grid] : 0;
  const int64_t words = (ne + 31) / 32;
  size_t out_b = 0, out2_b = 0;
  if (query == CS_QUERY_BINS) out_b = (size_t)n * 4;
  else if (query == CS_QUERY_SELECT) out_b = (size_t)n * 4, out2_b = (size_t)n * 8;
  else if (query == CS_QUERY_FEASIBLE) out_b = (size_t)n * words * 4;
  else return fail(CS_E_INVALID, "unknown query");
  auto a16 = [](size_t x) { return (x + 15) & ~(size_t)15; };
  const size_t in_b = a16((size_t)n * 8), o1 = a16(out_b);
  rc = query_stage(dev, in_b + o1 + a16(out2_b));
  if (rc) return rc;
  std::memcpy(g_qs.hpin, caps_host, (size_t)n * 8);
  cudaStream_t st = g_qs.st;
  CS_CUDA_RET(cudaMemcpyAsync(g_qs.dbuf, g_qs.hpin, (size_t)n * 8, cudaMemcpyHostToDevice, st));
  const double* cd = reinterpret_cast<const double*>(g_qs.dbuf);
  std::string err;
  if (query == CS_QUERY_BINS)
    err = cs::launch_lookup(d->view, cd, n, reinterpret_cast<int32_t*>(g_qs.dbuf + in_b), st);
  else if (query == CS_QUERY_SELECT)
    err = cs::launch_select(d->view, grid, policy, cd, n, reinterpret_cast<int32_t*>(g_qs.dbuf + in_b),
                            reinterpret_cast<int64_t*>(g_qs.dbuf + in_b + o1), st);
  else
    err = cs::launch_feasible(d->view, grid, policy, cd, n, reinterpret_cast<uint32_t*>(g_qs.dbuf + in_b), st);
  if (!err.empty()) return fail(CS_E_CUDA, err);
  CS_CUDA_RET(cudaMemcpyAsync(g_qs.hpin + in_b, g_qs.dbuf + in_b, o1 + a16(out2_b), cudaMemcpyDeviceToHost, st));
  CS_CUDA_RET(cudaStreamSynchronize(st));
  std::memcpy(out_host, g_qs.hpin + in_b, out_b);
  if (out2_b && out2_host) std::memcpy(out2_host, g_qs.hpin + in_b + o1, out2_b);
  return CS_OK;
}

int cs_feasible_caps(const cs_tables* tp, int32_t grid, int32_t policy, const double* caps_dev, int64_t n,
                     uint32_t* mask_dev, void* stream) {
  Tables::Dev* d = nullptr;
  int dev = 0;
  int rc = cs::current_view(tp, &d, &dev);
  if (rc) return rc;
  if (grid < 0 || grid >= d->view.M || policy < 0 || policy > 2) return fail(CS_E_INVALID, "grid/policy out of range");
  std::string err = cs::launch_feasible(d->view, grid, policy, caps_dev, n, mask_dev,
                                        reinterpret_cast<cudaStream_t>(stream));
  if (!err.empty()) return fail(CS_E_CUDA, err);
  return CS_OK;
}

int cs_replay(const cs_tables* tp, int32_t grid, const double* caps_dev, int64_t n_traces, int64_t n_steps, int64_t ld,
              int32_t mode, int32_t window_k, const int32_t* initial_dev, double noise_pct, const uint32_t* keys_dev,
              const int32_t* key_len_dev, int32_t key_stride, uint64_t seed_base, cs_replay_step* steps_dev,
              cs_replay_agg* agg_dev, void* stream) {
  Tables::Dev* d = nullptr;
  int dev = 0;
  int rc = cs::current_view(tp, &d, &dev);
  if (rc) return rc;
  if (d->view.cap_dtype != CS_CAP_F64) return fail(CS_E_INVALID, "cs_replay needs tables staged for fp64 caps");
  if (grid < 0 || grid >= d->view.M) return fail(CS_E_INVALID, "grid out of range");
  if (n_steps < 1 && n_traces > 0) return fail(CS_E_INVALID, "cannot replay an empty trace");
  const int32_t base_mode = mode & 0xFF;
  const bool tmaj = (mode & CS_CTRL_TIME_MAJOR) != 0;
  if ((tmaj ? ld < n_traces : ld < n_steps) || (base_mode != CS_CTRL_REACTIVE && base_mode != CS_CTRL_PROACTIVE) ||
      (mode & ~(0xFF | CS_CTRL_TIME_MAJOR)) || !(noise_pct >= 0.0) || !agg_dev)
    return fail(CS_E_INVALID, "bad replay arguments");
  if (keys_dev && !key_len_dev) return fail(CS_E_INVALID, "keys need key lengths");
  std::string err = cs::launch_replay(d->view, grid, caps_dev, n_traces, n_steps, ld, mode, window_k, initial_dev,
                                      noise_pct, keys_dev, key_len_dev, key_stride, seed_base, steps_dev, agg_dev,
                                      reinterpret_cast<cudaStream_t>(stream));
  if (!err.empty()) return fail(err.rfind("CUDA", 0) == 0 ? CS_E_CUDA : CS_E_INVALID, err);
  return CS_OK;
}

int cs_select_sampling(const cs_tables* tp, int32_t grid, const double* caps_dev, int64_t n_traces, int64_t n_steps,
                       int64_t ld, int64_t budget_m, int64_t rounds_r, uint64_t seed_lo, int64_t seed_hi,
                       int32_t* out_entry_dev, int32_t* out_count_dev, void* stream) {
  Tables::Dev* d = nullptr;
  int dev = 0;
  int rc = cs::current_view(tp, &d, &dev);
  if (rc) return rc;
  const Tables& t = *reinterpret_cast<const Tables*>(tp);
  if (d->view.cap_dtype != CS_CAP_F64) return fail(CS_E_INVALID, "cs_select_sampling needs tables staged for fp64 caps");
  if (grid < 0 || grid >= d->view.M) return fail(CS_E_INVALID, "grid out of range");
  if (budget_m < 1) return fail(CS_E_INVALID, "budget_m must be >= 1, got " + std::to_string(budget_m));
  if (rounds_r < 0) return fail(CS_E_INVALID, "rounds_r must be >= 0, got " + std::to_string(rounds_r));
  if (n_traces < 0 || n_steps < 0 || ld < n_steps || (!caps_dev && n_traces * n_steps > 0) ||
      (!out_entry_dev && n_traces * n_steps > 0))
    return fail(CS_E_INVALID, "bad sampling arguments");
  const int64_t n_entries = t.e_off[grid + 1] - t.e_off[grid];
  if (n_entries > 65535) return fail(CS_E_UNSUPPORTED, "sampling over grids of more than 65535 entries");
  int sms = 0;
  CS_CUDA_RET(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  std::string err = cs::launch_sampling(d->view, grid, caps_dev, n_traces, n_steps, ld, budget_m, rounds_r, seed_lo,
                                        seed_hi, out_entry_dev, out_count_dev, (int)n_entries, sms,
                                        reinterpret_cast<cudaStream_t>(stream));
  if (!err.empty()) return fail(CS_E_CUDA, err);
  return CS_OK;
}

int cs_entries_aggregate(const int32_t* entry_dev, int64_t n_traces, int64_t n_steps, int64_t ld,
                         const double* values_dev, int32_t n_entries, double penalty_frac, double* avg_dev,
                         double* energy_dev, int64_t* idle_dev, void* stream) {
  if (n_traces < 0 || n_steps < 1 || ld < n_steps || n_entries < 1 || !(penalty_frac >= 0.0 && penalty_frac <= 1.0) ||
      (n_traces > 0 && (!entry_dev || !values_dev || !avg_dev || !energy_dev || !idle_dev)))
    return fail(CS_E_INVALID, "bad aggregate arguments");
  std::string err = cs::launch_entries_agg(entry_dev, n_traces, n_steps, ld,
                                           reinterpret_cast<const double2*>(values_dev), n_entries, penalty_frac,
                                           avg_dev, energy_dev, idle_dev, reinterpret_cast<cudaStream_t>(stream));
  if (!err.empty()) return fail(CS_E_CUDA, err);
  return CS_OK;
}

int cs_generate_traces(float* caps_dev, int64_t n_traces, int64_t n_steps, int64_t ld, int64_t first_trace_id,
                       int32_t step_seconds, int32_t kind, float peak_w, uint64_t seed, void* stream) {
  if (ld < n_steps || n_traces < 0 || n_steps < 0 || step_seconds <= 0 || kind < 0 || kind > 3)
    return fail(CS_E_INVALID, "bad generator arguments");
  std::string err = cs::launch_generate(caps_dev, n_traces, n_steps, ld, first_trace_id, step_seconds, kind, peak_w,
                                        seed, reinterpret_cast<cudaStream_t>(stream));
  if (!err.empty()) return fail(CS_E_CUDA, err);
  return CS_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// host-buffer engine: chunked H2D -> eval -> D2H on three streams, double-buffered
// ---------------------------------------------------------------------------------------------
struct cs_engine {
  int device = 0;
  int cap_dtype = CS_CAP_F32;
  int64_t chunk = 0, smax = 0;
  int64_t ld_dev = 0;  // row pitch (elements) of the device cap buffers
  int64_t agg_rows = 0;  // grids x policies the aggregate buffers hold per trace
  cudaStream_t s_in = nullptr, s_cmp = nullptr, s_out = nullptr;
  void* dcaps[2] = {nullptr, nullptr};
  cs_agg* dagg[2] = {nullptr, nullptr};
  uint64_t* dhist = nullptr;
  void* dws = nullptr;
  size_t ws_bytes = 0;
  int32_t hist_bins = 0;
  cudaEvent_t in_done[2], cmp_done[2], out_done[2];
};

extern "C" {

int cs_engine_create(int32_t device, int64_t chunk_traces_max, int64_t n_steps_max, int32_t cap_dtype,
                     cs_engine** out) {
  if (!out || chunk_traces_max < 1 || n_steps_max < 1) return fail(CS_E_INVALID, "bad engine arguments");
  cs_engine* e = new (std::nothrow) cs_engine();
  if (!e) return fail(CS_E_INVALID, "out of host memory");
  e->device = device;
  e->cap_dtype = cap_dtype;
  e->chunk = chunk_traces_max;
  e->smax = n_steps_max;
  int prev = 0;
  CS_CUDA_RET(cudaGetDevice(&prev));
  CS_CUDA_RET(cudaSetDevice(device));
  const size_t esz = cap_dtype == CS_CAP_F32 ? 4 : 8;
  const int vec = cap_dtype == CS_CAP_F32 ? 4 : 2;
  const int64_t ld = (n_steps_max + vec - 1) / vec * vec;
  e->ld_dev = ld;
  cudaError_t err = cudaSuccess;
  for (int i = 0; i < 2 && err == cudaSuccess; ++i) {
    err = cudaMalloc(&e->dcaps[i], (size_t)chunk_traces_max * ld * esz);
    if (err == cudaSuccess) err = cudaEventCreateWithFlags(&e->in_done[i], cudaEventDisableTiming);
    if (err == cudaSuccess) err = cudaEventCreateWithFlags(&e->cmp_done[i], cudaEventDisableTiming);
    if (err == cudaSuccess) err = cudaEventCreateWithFlags(&e->out_done[i], cudaEventDisableTiming);
  }
  if (err == cudaSuccess) err = cudaStreamCreateWithFlags(&e->s_in, cudaStreamNonBlocking);
  if (err == cudaSuccess) err = cudaStreamCreateWithFlags(&e->s_cmp, cudaStreamNonBlocking);
  if (err == cudaSuccess) err = cudaStreamCreateWithFlags(&e->s_out, cudaStreamNonBlocking);
  cudaSetDevice(prev);
  if (err != cudaSuccess) {
    cs_engine_destroy(e);
    return fail(CS_E_CUDA, std::string("CUDA error creating engine: ") + cudaGetErrorString(err));
  }
  *out = e;
  return CS_OK;
}

int cs_engine_destroy(cs_engine* e) {
  if (!e) return CS_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(e->device);
  for (int i = 0; i < 2; ++i) {
    if (e->dcaps[i]) cudaFree(e->dcaps[i]);
    if (e->dagg[i]) cudaFree(e->dagg[i]);
  }
  if (e->dhist) cudaFree(e->dhist);
  if (e->dws) cudaFree(e->dws);
  if (e->s_in) cudaStreamDestroy(e->s_in);
  if (e->s_cmp) cudaStreamDestroy(e->s_cmp);
  if (e->s_out) cudaStreamDestroy(e->s_out);
  cudaSetDevice(prev);
  delete e;
  return CS_OK;
}

int cs_engine_eval_host(cs_engine* e, const cs_tables* tp, const void* caps_host, int64_t n_traces, int64_t n_steps,
                        int64_t ld, int32_t step_seconds, double switch_penalty_s, uint32_t flags, cs_agg* agg_host,
                        uint64_t* hist_host, int64_t* h2d_bytes, int64_t* d2h_bytes) {
  if (!e || !tp || !caps_host || !agg_host) return fail(CS_E_INVALID, "null argument");
  const Tables& t = *reinterpret_cast<const Tables*>(tp);
  if (t.cap_dtype != e->cap_dtype) return fail(CS_E_INVALID, "engine and tables cap dtype differ");
  if (n_traces < 0 || n_steps < 1) return fail(CS_E_INVALID, "bad sizes");
  if (n_steps > e->smax) return fail(CS_E_INVALID, "n_steps exceeds the engine's n_steps_max");
  if (ld < n_steps) return fail(CS_E_INVALID, "ld must be >= n_steps");
  int prev = 0;
  CS_CUDA_RET(cudaGetDevice(&prev));
  CS_CUDA_RET(cudaSetDevice(e->device));
  const size_t esz = e->cap_dtype == CS_CAP_F32 ? 4 : 8;
  const int64_t M = t.M;
  const size_t agg_chunk = (size_t)e->chunk * M * 3;
  int rc = CS_OK;
  auto done = [&](int r) {
    cudaSetDevice(prev);
    return r;
  };
  if (e->agg_rows < M * 3) {  // sized for the tables of this call (more grids: grow)
    for (int i = 0; i < 2; ++i) {
      if (e->dagg[i]) cudaFree(e->dagg[i]), e->dagg[i] = nullptr;
      CS_CUDA_RET(cudaMalloc(&e->dagg[i], agg_chunk * sizeof(cs_agg)));
    }
    e->agg_rows = M * 3;
  }
  if (e->hist_bins < t.U) {
    if (e->dhist) cudaFree(e->dhist);
    CS_CUDA_RET(cudaMalloc(&e->dhist, (size_t)t.U * 8));
    e->hist_bins = t.U;
  }
  CS_CUDA_RET(cudaMemsetAsync(e->dhist, 0, (size_t)t.U * 8, e->s_cmp));
  // workspace for the largest chunk
  cs_eval_args probe{};
  probe.caps = e->dcaps[0];
  probe.n_traces = std::min(n_traces, e->chunk);
  probe.n_steps = n_steps;
  probe.ld = e->ld_dev;  // device rows keep the engine's pitch whatever the host pitch
  probe.step_seconds = step_seconds;
  probe.switch_penalty_s = switch_penalty_s;
  probe.flags = flags;
  probe.hist = e->dhist;
  size_t need = 0;
  if ((rc = cs_eval_workspace_size(tp, &probe, &need))) return done(rc);
  if (n_traces > e->chunk && n_traces % e->chunk) {  // the tail chunk may take the split-trace path
    cs_eval_args tail = probe;
    tail.n_traces = n_traces % e->chunk;
    size_t need_tail = 0;
    if ((rc = cs_eval_workspace_size(tp, &tail, &need_tail))) return done(rc);
    need = std::max(need, need_tail);
  }
  if (need > e->ws_bytes) {
    if (e->dws) cudaFree(e->dws);
    CS_CUDA_RET(cudaMalloc(&e->dws, need));
    e->ws_bytes = need;
  }
  int64_t h2d = 0, d2h = 0;
  const int64_t nchunks = (n_traces + e->chunk - 1) / e->chunk;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int b = (int)(c & 1);
    const int64_t t0 = c * e->chunk;
    const int64_t nt = std::min(e->chunk, n_traces - t0);
    // H2D into buffer b once the eval that last read it is done
    if (c >= 2) CS_CUDA_RET(cudaStreamWaitEvent(e->s_in, e->cmp_done[b], 0));
    const unsigned char* src = reinterpret_cast<const unsigned char*>(caps_host) + (size_t)t0 * ld * esz;
    size_t bytes;
    if (ld == e->ld_dev) {  // same pitch: one contiguous copy of whole rows
      bytes = (size_t)nt * ld * esz;
      CS_CUDA_RET(cudaMemcpyAsync(e->dcaps[b], src, bytes, cudaMemcpyHostToDevice, e->s_in));
    } else {  // padded / strided host rows: copy the n_steps samples of each row into the engine's pitch
      bytes = (size_t)nt * n_steps * esz;
      CS_CUDA_RET(cudaMemcpy2DAsync(e->dcaps[b], (size_t)e->ld_dev * esz, src, (size_t)ld * esz, (size_t)n_steps * esz,
                                    (size_t)nt, cudaMemcpyHostToDevice, e->s_in));
    }
    h2d += (int64_t)bytes;
    CS_CUDA_RET(cudaEventRecord(e->in_done[b], e->s_in));
    // eval once the copy landed and the previous D2H of agg[b] drained
    CS_CUDA_RET(cudaStreamWaitEvent(e->s_cmp, e->in_done[b], 0));
    if (c >= 2) CS_CUDA_RET(cudaStreamWaitEvent(e->s_cmp, e->out_done[b], 0));
    cs_eval_args a = probe;
    a.caps = e->dcaps[b];
    a.n_traces = nt;
    a.agg = e->dagg[b];
    a.flags = flags | CS_FLAG_ACCUMULATE_HIST;
    a.workspace = e->dws;
    a.workspace_bytes = e->ws_bytes;
    if ((rc = cs_eval(tp, &a, e->s_cmp))) return done(rc);
    CS_CUDA_RET(cudaEventRecord(e->cmp_done[b], e->s_cmp));
    // D2H of this chunk's aggregates
    CS_CUDA_RET(cudaStreamWaitEvent(e->s_out, e->cmp_done[b], 0));
    const size_t abytes = (size_t)nt * M * 3 * sizeof(cs_agg);
    CS_CUDA_RET(cudaMemcpyAsync(agg_host + (size_t)t0 * M * 3, e->dagg[b], abytes, cudaMemcpyDeviceToHost, e->s_out));
    d2h += (int64_t)abytes;
    CS_CUDA_RET(cudaEventRecord(e->out_done[b], e->s_out));
  }
  CS_CUDA_RET(cudaStreamSynchronize(e->s_cmp));
  if (hist_host) {
    CS_CUDA_RET(cudaMemcpyAsync(hist_host, e->dhist, (size_t)t.U * 8, cudaMemcpyDeviceToHost, e->s_out));
    d2h += (int64_t)t.U * 8;
  }
  CS_CUDA_RET(cudaStreamSynchronize(e->s_out));
  CS_CUDA_RET(cudaStreamSynchronize(e->s_in));
  if (h2d_bytes) *h2d_bytes = h2d;
  if (d2h_bytes) *d2h_bytes = d2h;
  return done(CS_OK);
}

}  // extern "C"
