// Communicator of the slab-decomposed solve (wd_comm_init).
//
// One process per GPU.  The production backend is NCCL over NVLink/NVSwitch,
// loaded with dlopen at wd_comm_init time (the library itself has no NCCL link
// dependency: a single-GPU user never needs it; torch's bundled libnccl.so.2 is
// reused when it is already mapped into the process).  Every operation is
// enqueued on the caller's stream and is CUDA-graph capturable.  The second
// backend forwards the four collectives to host callbacks; it exists so the
// SAME step program can be driven by another transport (torch.distributed /
// gloo with host staging, or P logical ranks in one process) in tests on a
// single GPU -- callbacks synchronise on the host, so it is not capturable.
// With one rank both backends degenerate to device copies.  A third, "solo"
// backend lets ONE rank of a P-rank decomposition run alone (its collectives
// are device copies of the same volume, the slab wraps onto itself): the
// per-GPU kernel time of a P-way split measured on a single GPU, graph
// captured like the NCCL program (bench.py --dist --as-ranks P).
#pragma once

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/walldist_b200.h"

namespace wd {

// Minimal NCCL declarations (ABI-stable since NCCL 2.x): the functions are
// resolved with dlsym, so nccl.h is not needed to build.
struct NcclUniqueId {
  char internal[128];
};
typedef void* NcclComm;
constexpr int kNcclInt64 = 4;
constexpr int kNcclFloat64 = 8;
constexpr int kNcclMax = 2;

struct NcclApi {
  void* handle = nullptr;
  int (*GetUniqueId)(NcclUniqueId*) = nullptr;
  int (*CommInitRank)(NcclComm*, int, NcclUniqueId, int) = nullptr;
  int (*CommDestroy)(NcclComm) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*Send)(const void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, NcclComm, cudaStream_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  int (*GetVersion)(int*) = nullptr;
};

inline NcclApi* nccl_api(std::string& err) {
  static NcclApi api;
  static bool tried = false;
  if (api.handle) return &api;
  if (tried) {
    err = "NCCL is not loadable (libnccl.so.2)";
    return nullptr;
  }
  tried = true;
  void* h = nullptr;
  if (const char* p = getenv("WD_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
  // the copy torch (or the host application) already mapped, else the system's
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    err = std::string("cannot load NCCL: ") + dlerror();
    return nullptr;
  }
  bool ok = true;
  auto sym = [&](const char* name) {
    void* s = dlsym(h, name);
    if (!s) ok = false;
    return s;
  };
  api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
  api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
  api.Send = (decltype(api.Send))sym("ncclSend");
  api.Recv = (decltype(api.Recv))sym("ncclRecv");
  api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
  api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
  api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
  api.GetVersion = (decltype(api.GetVersion))sym("ncclGetVersion");
  if (!ok) {
    err = "libnccl.so.2 lacks a required symbol";
    return nullptr;
  }
  api.handle = h;
  return &api;
}

}  // namespace wd

struct wd_comm {
  int rank = 0;
  int P = 1;
  int kind = 0;  // 0: NCCL, 1: host callbacks, 2: solo (one rank of P timed alone)
  int decomposition = 0;
  wd::NcclApi* api = nullptr;
  wd::NcclComm nccl = nullptr;
  wd_comm_callbacks cb{};
  std::string err;

  int left() const { return (rank + P - 1) % P; }
  int right() const { return (rank + 1) % P; }
  bool capturable() const { return kind != 1; }

  int nccl_rc(int rc, const char* what) {
    if (rc == 0) return WD_OK;
    err = std::string(what) + ": " + (api && api->GetErrorString ? api->GetErrorString(rc) : "?");
    return WD_ERR_CUDA;
  }
  int cuda_rc(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return WD_OK;
    err = std::string(what) + ": " + cudaGetErrorString(e);
    return WD_ERR_CUDA;
  }

  // Ghost planes of a slab stored as (nl + 2G) planes of `plane` doubles:
  // my top G interior planes -> right neighbour's low ghosts, my bottom G
  // interior planes -> left neighbour's high ghosts (periodic ring),
  // received straight into the ghost planes.
  int halo(double* t, long long plane, int nl, int G, cudaStream_t s) {
    const size_t cnt = (size_t)G * plane;
    double* lo_ghost = t;
    double* lo_int = t + (size_t)G * plane;
    double* hi_int = t + (size_t)nl * plane;
    double* hi_ghost = t + (size_t)(nl + G) * plane;
    if ((P == 1 && !nccl) || kind == 2) {
      if (int rc = cuda_rc(cudaMemcpyAsync(lo_ghost, hi_int, cnt * 8, cudaMemcpyDeviceToDevice, s),
                           "halo copy"))
        return rc;
      return cuda_rc(cudaMemcpyAsync(hi_ghost, lo_int, cnt * 8, cudaMemcpyDeviceToDevice, s),
                     "halo copy");
    }
    if (kind == 1) {
      if (cb.halo(cb.user, t, plane, nl, G, (void*)s)) {
        err = "halo callback failed";
        return WD_ERR_CUDA;
      }
      return WD_OK;
    }
    // posting order matters when left == right (P = 2): point-to-point
    // operations between one pair of ranks match in posting order
    int rc = api->GroupStart();
    if (!rc) rc = api->Send(hi_int, cnt, wd::kNcclFloat64, right(), nccl, s);
    if (!rc) rc = api->Recv(lo_ghost, cnt, wd::kNcclFloat64, left(), nccl, s);
    if (!rc) rc = api->Send(lo_int, cnt, wd::kNcclFloat64, left(), nccl, s);
    if (!rc) rc = api->Recv(hi_ghost, cnt, wd::kNcclFloat64, right(), nccl, s);
    const int rc2 = api->GroupEnd();
    return nccl_rc(rc ? rc : rc2, "ncclSend/Recv (halo)");
  }

  // all[q * count ..] <- rank q's mine[0 .. count)
  int allgather(const double* mine, double* all, size_t count, cudaStream_t s) {
    if (P == 1 && !nccl)
      return cuda_rc(cudaMemcpyAsync(all, mine, count * 8, cudaMemcpyDeviceToDevice, s),
                     "allgather copy");
    if (kind == 2) {  // every slot <- mine: the received volume of a real all_gather
      for (int q = 0; q < P; ++q)
        if (int rc = cuda_rc(cudaMemcpyAsync(all + (size_t)q * count, mine, count * 8,
                                             cudaMemcpyDeviceToDevice, s), "allgather copy"))
          return rc;
      return WD_OK;
    }
    if (kind == 1) {
      if (cb.allgather(cb.user, mine, all, (long long)count, (void*)s)) {
        err = "allgather callback failed";
        return WD_ERR_CUDA;
      }
      return WD_OK;
    }
    return nccl_rc(api->AllGather(mine, all, count, wd::kNcclFloat64, nccl, s), "ncclAllGather");
  }

  // recv[q * count ..] <- rank q's send[rank * count ..]  (slab <-> pencil)
  int alltoall(const double* send, double* recv, size_t count, cudaStream_t s) {
    if ((P == 1 && !nccl) || kind == 2)
      return cuda_rc(cudaMemcpyAsync(recv, send, count * 8 * P, cudaMemcpyDeviceToDevice, s),
                     "alltoall copy");
    if (kind == 1) {
      if (cb.alltoall(cb.user, send, recv, (long long)count, (void*)s)) {
        err = "alltoall callback failed";
        return WD_ERR_CUDA;
      }
      return WD_OK;
    }
    int rc = api->GroupStart();
    for (int q = 0; q < P && !rc; ++q) {
      rc = api->Send(send + (size_t)q * count, count, wd::kNcclFloat64, q, nccl, s);
      if (!rc) rc = api->Recv(recv + (size_t)q * count, count, wd::kNcclFloat64, q, nccl, s);
    }
    const int rc2 = api->GroupEnd();
    return nccl_rc(rc ? rc : rc2, "ncclSend/Recv (all_to_all)");
  }

  // element-wise max over the ranks of n int64 words, in place
  int allreduce_max(long long* buf, int n, cudaStream_t s) {
    if ((P == 1 && !nccl) || kind == 2) return WD_OK;
    if (kind == 1) {
      if (cb.allreduce_max(cb.user, buf, n, (void*)s)) {
        err = "allreduce callback failed";
        return WD_ERR_CUDA;
      }
      return WD_OK;
    }
    return nccl_rc(api->AllReduce(buf, buf, (size_t)n, wd::kNcclInt64, wd::kNcclMax, nccl, s),
                   "ncclAllReduce");
  }
};
