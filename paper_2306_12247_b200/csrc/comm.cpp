// Single-process multi-GPU reduction of a sharded sweep (north star (4): "a single
// NCCL reduce over NVLink for the aggregate statistics"). One communicator over the devices of
// this process (ncclCommInitAll) and one grouped int64 SUM all-reduce of every device's
// [union-bin histogram | sweep totals] buffer: integer words, so the result is identical at any
// device count and in any reduction order.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2 — the copy a PyTorch process has already
// loaded, else the system one), so the library loads and every other entry point works on hosts
// without NCCL; these calls then report CS_E_UNSUPPORTED.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <mutex>
#include <string>
#include <vector>

#include "capsim_b200.h"
#include "cs_internal.h"

namespace {

// the subset of nccl.h used here (ABI-stable since NCCL 2.0)
typedef struct ncclComm* ncclComm_t;
typedef int ncclResult_t;
constexpr int kNcclInt64 = 4, kNcclSum = 0;

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string err;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (n.h) break;
    }
    if (!n.h) {
      n.err = "NCCL (libnccl.so.2) not found";
      return;
    }
    n.comm_init_all = reinterpret_cast<decltype(n.comm_init_all)>(dlsym(n.h, "ncclCommInitAll"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(n.h, "ncclCommDestroy"));
    n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(n.h, "ncclAllReduce"));
    n.group_start = reinterpret_cast<decltype(n.group_start)>(dlsym(n.h, "ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(n.group_end)>(dlsym(n.h, "ncclGroupEnd"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(n.h, "ncclGetErrorString"));
    if (!n.comm_init_all || !n.comm_destroy || !n.all_reduce || !n.group_start || !n.group_end || !n.error_string)
      n.err = "libnccl.so.2 lacks the collective entry points";
  });
  return n;
}

int fail(int code, const std::string& msg) {
  cs::set_error(msg);
  return code;
}

std::string nccl_msg(const Nccl& n, ncclResult_t r) { return std::string("NCCL error: ") + n.error_string(r); }

}  // namespace

struct cs_comm {
  std::vector<int> devices;
  std::vector<ncclComm_t> comms;
};

extern "C" {

int cs_comm_init_all(int32_t n_devices, const int32_t* devices, cs_comm** out) {
  if (!out || n_devices < 1 || !devices) return fail(CS_E_INVALID, "cs_comm_init_all: need >= 1 device");
  Nccl& n = nccl();
  if (!n.err.empty()) return fail(CS_E_UNSUPPORTED, n.err);
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) return fail(CS_E_NODEVICE, "no CUDA device");
  for (int i = 0; i < n_devices; ++i) {
    if (devices[i] < 0 || devices[i] >= count) return fail(CS_E_INVALID, "device ordinal out of range");
    for (int j = 0; j < i; ++j)
      if (devices[j] == devices[i]) return fail(CS_E_INVALID, "a device may appear once per communicator");
  }
  auto* c = new cs_comm;
  c->devices.assign(devices, devices + n_devices);
  c->comms.resize(n_devices);
  const ncclResult_t r = n.comm_init_all(c->comms.data(), n_devices, c->devices.data());
  if (r != 0) {
    delete c;
    return fail(CS_E_CUDA, nccl_msg(n, r));
  }
  *out = c;
  return CS_OK;
}

int cs_comm_size(const cs_comm* c, int32_t* n_devices) {
  if (!c || !n_devices) return fail(CS_E_INVALID, "null argument");
  *n_devices = (int32_t)c->devices.size();
  return CS_OK;
}

int cs_comm_allreduce_i64(cs_comm* c, int64_t* const* bufs, int64_t count, void* const* streams) {
  if (!c || !bufs || count < 0) return fail(CS_E_INVALID, "bad all-reduce arguments");
  Nccl& n = nccl();
  if (!n.err.empty()) return fail(CS_E_UNSUPPORTED, n.err);
  if (count == 0) return CS_OK;
  for (size_t i = 0; i < c->devices.size(); ++i)
    if (!bufs[i]) return fail(CS_E_INVALID, "null device buffer");
  int prev = 0;
  cudaGetDevice(&prev);
  ncclResult_t r = n.group_start();
  for (size_t i = 0; r == 0 && i < c->devices.size(); ++i) {
    cudaSetDevice(c->devices[i]);
    r = n.all_reduce(bufs[i], bufs[i], (size_t)count, kNcclInt64, kNcclSum, c->comms[i],
                     streams ? reinterpret_cast<cudaStream_t>(streams[i]) : nullptr);
  }
  const ncclResult_t r2 = n.group_end();
  cudaSetDevice(prev);
  if (r != 0) return fail(CS_E_CUDA, nccl_msg(n, r));
  if (r2 != 0) return fail(CS_E_CUDA, nccl_msg(n, r2));
  return CS_OK;
}

int cs_comm_destroy(cs_comm* c) {
  if (!c) return CS_OK;
  Nccl& n = nccl();
  if (n.err.empty())
    for (ncclComm_t x : c->comms)
      if (x) n.comm_destroy(x);
  delete c;
  return CS_OK;
}

}  // extern "C"
