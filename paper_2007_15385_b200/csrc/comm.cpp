// comm.cpp -- the path's one collective: a sum of the per-GPU inside counts
// (the reference is single-node CPU code with no collective).
//
// NCCL is resolved at run time with dlopen so libvpipg.so loads on hosts
// without it (the CPU test suite, the build container) and shares the copy a
// host framework already loaded (torch's libnccl.so.2 has the same soname).
// nccl.h is included for its types only.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "vpipg.h"
#include "vpipg_internal.h"

struct vpipg_comm {
  ncclComm_t comm = nullptr;
  int nranks = 0;
  int rank = 0;
  int device = 0;
};

namespace {

struct Nccl {
  void* lib = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

template <class F>
bool sym(void* lib, const char* name, F& f) {
  f = reinterpret_cast<F>(dlsym(lib, name));
  return f != nullptr;
}

const Nccl* nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {std::getenv("VPIPG_NCCL_LIBRARY"), "libnccl.so.2", "libnccl.so"};
    for (const char* name : names) {
      if (!name || !*name) continue;
      n.lib = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (n.lib) break;
    }
    if (!n.lib) return;
    const bool ok = sym(n.lib, "ncclGetVersion", n.get_version) &&
                    sym(n.lib, "ncclGetUniqueId", n.get_unique_id) &&
                    sym(n.lib, "ncclCommInitRank", n.comm_init_rank) &&
                    sym(n.lib, "ncclCommInitAll", n.comm_init_all) &&
                    sym(n.lib, "ncclAllReduce", n.all_reduce) &&
                    sym(n.lib, "ncclGroupStart", n.group_start) &&
                    sym(n.lib, "ncclGroupEnd", n.group_end) &&
                    sym(n.lib, "ncclCommDestroy", n.comm_destroy) &&
                    sym(n.lib, "ncclGetErrorString", n.error_string);
    if (!ok) {
      dlclose(n.lib);
      n.lib = nullptr;
    }
  });
  return n.lib ? &n : nullptr;
}

int nccl_code(ncclResult_t r) { return r == ncclSuccess ? 0 : VPIPG_ERR_NCCL + static_cast<int>(r); }
int cuda_code(cudaError_t e) { return e == cudaSuccess ? 0 : VPIPG_ERR_CUDA + static_cast<int>(e); }

constexpr int kInvalid = 6;

}  // namespace

const char* vpipg_nccl_error_string(int code) {
  const Nccl* n = nccl();
  if (!n) return "NCCL error (libnccl not loaded)";
  return n->error_string(static_cast<ncclResult_t>(code - VPIPG_ERR_NCCL));
}

extern "C" {

int vpipg_nccl_version(int* version) {
  const Nccl* n = nccl();
  if (!n) return VPIPG_ERR_NCCL_MISSING;
  if (!version) return kInvalid;
  return nccl_code(n->get_version(version));
}

int vpipg_comm_unique_id(uint8_t id[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  const Nccl* n = nccl();
  if (!n) return VPIPG_ERR_NCCL_MISSING;
  if (!id) return kInvalid;
  ncclUniqueId u;
  const int rc = nccl_code(n->get_unique_id(&u));
  if (rc == 0) std::memcpy(id, &u, sizeof u);
  return rc;
}

int vpipg_comm_init(const uint8_t id[128], int nranks, int rank, int device, vpipg_comm** out) {
  if (!out) return kInvalid;
  *out = nullptr;
  if (!id || nranks < 1 || rank < 0 || rank >= nranks || device < 0) return kInvalid;
  const Nccl* n = nccl();
  if (!n) return VPIPG_ERR_NCCL_MISSING;
  int prev = 0;
  int rc = cuda_code(cudaGetDevice(&prev));
  if (rc) return rc;
  if ((rc = cuda_code(cudaSetDevice(device)))) return rc;
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof u);
  ncclComm_t c = nullptr;
  rc = nccl_code(n->comm_init_rank(&c, nranks, u, rank));
  cudaSetDevice(prev);
  if (rc) return rc;
  auto* h = new (std::nothrow) vpipg_comm{c, nranks, rank, device};
  if (!h) {
    n->comm_destroy(c);
    return kInvalid;
  }
  *out = h;
  return 0;
}

int vpipg_comm_init_all(int ndev, const int* devices, vpipg_comm** comms) {
  if (ndev < 1 || !devices || !comms) return kInvalid;
  const Nccl* n = nccl();
  if (!n) return VPIPG_ERR_NCCL_MISSING;
  std::vector<ncclComm_t> c(ndev, nullptr);
  const int rc = nccl_code(n->comm_init_all(c.data(), ndev, devices));
  if (rc) return rc;
  for (int i = 0; i < ndev; ++i) {
    comms[i] = new (std::nothrow) vpipg_comm{c[i], ndev, i, devices[i]};
    if (!comms[i]) {
      for (int j = 0; j < ndev; ++j) {
        if (j < i) delete comms[j];
        n->comm_destroy(c[j]);
        comms[j] = nullptr;
      }
      return kInvalid;
    }
  }
  return 0;
}

int vpipg_comm_info(const vpipg_comm* comm, int* nranks, int* rank, int* device) {
  if (!comm) return kInvalid;
  if (nranks) *nranks = comm->nranks;
  if (rank) *rank = comm->rank;
  if (device) *device = comm->device;
  return 0;
}

int vpipg_allreduce_counts(vpipg_comm* comm, unsigned long long* d_counts, int n, void* stream) {
  if (!comm || n < 0 || (n > 0 && !d_counts)) return kInvalid;
  if (n == 0) return 0;
  const Nccl* lib = nccl();
  if (!lib) return VPIPG_ERR_NCCL_MISSING;
  return nccl_code(lib->all_reduce(d_counts, d_counts, static_cast<size_t>(n), ncclUint64, ncclSum,
                                   comm->comm, static_cast<cudaStream_t>(stream)));
}

int vpipg_allreduce_counts_group(int ncomms, vpipg_comm* const* comms,
                                 unsigned long long* const* d_counts, int n,
                                 void* const* streams) {
  if (ncomms < 1 || !comms || !d_counts || !streams || n < 0) return kInvalid;
  for (int i = 0; i < ncomms; ++i)
    if (!comms[i] || (n > 0 && !d_counts[i])) return kInvalid;
  if (n == 0) return 0;
  const Nccl* lib = nccl();
  if (!lib) return VPIPG_ERR_NCCL_MISSING;
  int rc = nccl_code(lib->group_start());
  if (rc) return rc;
  for (int i = 0; i < ncomms && !rc; ++i)
    rc = nccl_code(lib->all_reduce(d_counts[i], d_counts[i], static_cast<size_t>(n), ncclUint64,
                                   ncclSum, comms[i]->comm, static_cast<cudaStream_t>(streams[i])));
  const int rc_end = nccl_code(lib->group_end());
  return rc ? rc : rc_end;
}

int vpipg_comm_destroy(vpipg_comm* comm) {
  if (!comm) return 0;
  const Nccl* n = nccl();
  int rc = 0;
  if (n && comm->comm) rc = nccl_code(n->comm_destroy(comm->comm));
  delete comm;
  return rc;
}

}  // extern "C"
