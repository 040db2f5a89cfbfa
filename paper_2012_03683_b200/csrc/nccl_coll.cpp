// Native NCCL collective for row-sharded registrations (C4):
// the per-round combination of the ranks' sums and maxima
// (kreg_register_clouds_rows, solver.cpp reduce_round) as NCCL calls on the
// context's stream instead of a host callback into Python.
//
// NCCL is dlopen'ed ("libnccl.so.2": the copy torch already loaded, else the
// system one), so the engine has no link-time NCCL dependency. The context's
// kreg_collective_fn is set to nccl_round below:
//   deterministic: ncclAllGather of every rank's [sums, maxes] (one call),
//                  sums added in rank order on every rank (bitwise independent
//                  of NCCL's algorithm: ring / tree / NVLS), max over ranks;
//   otherwise:     ncclAllReduce(sum) + ncclAllReduce(max) in one group.
// The round's values travel host -> device -> NCCL -> host on the context
// stream (a few hundred bytes: K x 7 sums + pair counts, K displacements).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <type_traits>
#include <vector>

#include "engine_host.hpp"

namespace kreg_host {

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [h](auto& fn, const char* name) { fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name)); };
    sym(api.get_unique_id, "ncclGetUniqueId");
    sym(api.comm_init_rank, "ncclCommInitRank");
    sym(api.comm_destroy, "ncclCommDestroy");
    sym(api.all_reduce, "ncclAllReduce");
    sym(api.all_gather, "ncclAllGather");
    sym(api.group_start, "ncclGroupStart");
    sym(api.group_end, "ncclGroupEnd");
    sym(api.error_string, "ncclGetErrorString");
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce && api.all_gather &&
             api.group_start && api.group_end && api.error_string;
  });
  return api;
}

void check_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(KREG_RUNTIME_ERROR, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

struct NcclState {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  bool deterministic = true;
  cudaStream_t stream = nullptr;
  DevBuf<double> send, recv;
  std::vector<double> host;  // gathered values (deterministic mode)
  long long calls = 0;
  ~NcclState() {
    if (comm) nccl().comm_destroy(comm);
  }
};

void nccl_unique_id(unsigned char out[128]) {
  const NcclApi& a = nccl();
  if (!a.ok) throw Error(KREG_RUNTIME_ERROR, "libnccl.so.2 not found");
  ncclUniqueId id;
  check_nccl(a.get_unique_id(&id), "ncclGetUniqueId");
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out, &id, sizeof(id));
}

// kreg_collective_fn over NCCL (user = the NcclState)
int32_t nccl_round(void* user, double* sums, int32_t n_sums, double* maxes, int32_t n_maxes) {
  auto* S = static_cast<NcclState*>(user);
  try {
    const NcclApi& a = nccl();
    const size_t n = static_cast<size_t>(n_sums) + static_cast<size_t>(n_maxes);
    if (n == 0) return 0;
    S->send.ensure(n, false, 2.0);
    S->recv.ensure(n * static_cast<size_t>(S->world), false, 2.0);
    std::vector<double> v(n);
    std::memcpy(v.data(), sums, sizeof(double) * n_sums);
    std::memcpy(v.data() + n_sums, maxes, sizeof(double) * n_maxes);
    KREG_CUDA(cudaMemcpyAsync(S->send.ptr, v.data(), sizeof(double) * n, cudaMemcpyHostToDevice, S->stream));
    if (S->deterministic) {
      check_nccl(a.all_gather(S->send.ptr, S->recv.ptr, n, ncclFloat64, S->comm, S->stream), "ncclAllGather");
      S->host.resize(n * static_cast<size_t>(S->world));
      KREG_CUDA(cudaMemcpyAsync(S->host.data(), S->recv.ptr, sizeof(double) * S->host.size(), cudaMemcpyDeviceToHost,
                                S->stream));
      KREG_CUDA(cudaStreamSynchronize(S->stream));
      for (int32_t k = 0; k < n_sums; ++k) {  // rank order
        double t = S->host[k];
        for (int r = 1; r < S->world; ++r) t += S->host[static_cast<size_t>(r) * n + k];
        sums[k] = t;
      }
      for (int32_t k = 0; k < n_maxes; ++k) {
        double m = S->host[n_sums + k];
        for (int r = 1; r < S->world; ++r) m = std::max(m, S->host[static_cast<size_t>(r) * n + n_sums + k]);
        maxes[k] = m;
      }
    } else {
      check_nccl(a.group_start(), "ncclGroupStart");
      if (n_sums)
        check_nccl(a.all_reduce(S->send.ptr, S->recv.ptr, n_sums, ncclFloat64, ncclSum, S->comm, S->stream),
                   "ncclAllReduce");
      if (n_maxes)
        check_nccl(a.all_reduce(S->send.ptr + n_sums, S->recv.ptr + n_sums, n_maxes, ncclFloat64, ncclMax, S->comm,
                                S->stream),
                   "ncclAllReduce");
      check_nccl(a.group_end(), "ncclGroupEnd");
      KREG_CUDA(cudaMemcpyAsync(v.data(), S->recv.ptr, sizeof(double) * n, cudaMemcpyDeviceToHost, S->stream));
      KREG_CUDA(cudaStreamSynchronize(S->stream));
      std::memcpy(sums, v.data(), sizeof(double) * n_sums);
      std::memcpy(maxes, v.data() + n_sums, sizeof(double) * n_maxes);
    }
    ++S->calls;
    return 0;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return 1;
  }
}

void nccl_attach(kreg_ctx* ctx, const unsigned char id[128], int rank, int world, bool deterministic) {
  const NcclApi& a = nccl();
  if (!a.ok) throw Error(KREG_RUNTIME_ERROR, "libnccl.so.2 not found");
  if (world < 1 || rank < 0 || rank >= world) throw Error(KREG_INVALID_ARGUMENT, "nccl: bad rank / world size");
  KREG_CUDA(cudaSetDevice(ctx->device));
  auto S = std::make_unique<NcclState>();
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  check_nccl(a.comm_init_rank(&S->comm, world, uid, rank), "ncclCommInitRank");
  S->rank = rank;
  S->world = world;
  S->deterministic = deterministic;
  S->stream = ctx->stream;
  nccl_free(ctx->nccl);
  ctx->nccl = S.release();
  ctx->collective.fn = nccl_round;
  ctx->collective.user = ctx->nccl;
}

void nccl_free(NcclState* s) { delete s; }

void nccl_detach(kreg_ctx* ctx) {
  if (ctx->nccl && ctx->collective.user == ctx->nccl) {
    ctx->collective.fn = nullptr;
    ctx->collective.user = nullptr;
  }
  nccl_free(ctx->nccl);
  ctx->nccl = nullptr;
}

long long nccl_calls(const kreg_ctx* ctx) { return ctx->nccl ? ctx->nccl->calls : 0; }

}  // namespace kreg_host
