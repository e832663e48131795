// Native NCCL communicator for the row-partitioned block CG.
//
// Reference: the paper's MPI layer — MPI_Allreduce of the small reduction blocks
// and the halo exchange of the distributed SpMM; the Python
// reference replaces MPI by an in-process reduction.
//
// Without it, every block-CG sweep of a row-partitioned solve calls back into Python
// three times (halo of r, the p'q and ||r||^2 sums) and each callback synchronises the
// host.  With a communicator the library enqueues the halo (grouped ncclSend /
// ncclRecv per neighbour) and the two k-vector ncclAllReduce calls on the context
// stream itself: all sweeps of a distributed CG run without a host round trip, like
// the single-GPU loop.
//
// NCCL is loaded at run time (dlopen of libnccl.so.2 — the one torch already loaded
// when present), so the library has no link-time NCCL dependency and builds and
// loads on hosts without it; the entry points then return GCG_ERR_ARG.

#include <dlfcn.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>

#include <mutex>

#include "common.cuh"

namespace gcg {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*getVersion)(int*) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define LOAD(field, sym) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, sym))
    LOAD(getUniqueId, "ncclGetUniqueId");
    LOAD(commInitRank, "ncclCommInitRank");
    LOAD(commDestroy, "ncclCommDestroy");
    LOAD(allReduce, "ncclAllReduce");
    LOAD(send, "ncclSend");
    LOAD(recv, "ncclRecv");
    LOAD(groupStart, "ncclGroupStart");
    LOAD(groupEnd, "ncclGroupEnd");
    LOAD(getVersion, "ncclGetVersion");
#undef LOAD
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allReduce &&
             api.send && api.recv && api.groupStart && api.groupEnd;
  });
  return api;
}

static int nccl_status(ncclResult_t r) { return r == ncclSuccess ? GCG_OK : GCG_ERR_CUDA; }

// the block-CG hooks (cg.cu): halo of X's ghost rows and the in-place k-vector sum
int nccl_cg_halo(Ctx* c, const gcg_cg_dist* d, int k) {
  NcclApi& api = nccl();
  if (!api.ok || !d->nccl_comm) return GCG_ERR_ARG;
  ncclComm_t comm = reinterpret_cast<ncclComm_t>(d->nccl_comm);
  GCG_TRY(nccl_status(api.groupStart()));
  for (int q = 0; q < d->npeer; ++q) {
    const int64_t s0 = d->peer_send_off[q], s1 = d->peer_send_off[q + 1];
    const int64_t r0 = d->peer_recv_off[q], r1 = d->peer_recv_off[q + 1];
    if (s1 > s0)
      GCG_TRY(nccl_status(api.send(d->send_buf + s0 * k, (size_t)(s1 - s0) * k, ncclDouble,
                                   d->peer_rank[q], comm, c->stream)));
    if (r1 > r0)
      GCG_TRY(nccl_status(api.recv(d->recv_buf + r0 * k, (size_t)(r1 - r0) * k, ncclDouble,
                                   d->peer_rank[q], comm, c->stream)));
  }
  return nccl_status(api.groupEnd());
}

int nccl_cg_allreduce(Ctx* c, const gcg_cg_dist* d, int k) {
  NcclApi& api = nccl();
  if (!api.ok || !d->nccl_comm) return GCG_ERR_ARG;
  return nccl_status(api.allReduce(d->red_buf, d->red_buf, (size_t)k, ncclDouble, ncclSum,
                                   reinterpret_cast<ncclComm_t>(d->nccl_comm), c->stream));
}

}  // namespace gcg

using namespace gcg;

extern "C" {

int gcg_nccl_available(void) {
  NcclApi& api = nccl();
  if (!api.ok) return 0;
  int v = 0;
  if (api.getVersion) api.getVersion(&v);
  return v > 0 ? v : 1;
}

int gcg_nccl_unique_id(uint8_t* out128) {
  NcclApi& api = nccl();
  if (!api.ok || !out128) return GCG_ERR_ARG;
  ncclUniqueId id;
  GCG_TRY(nccl_status(api.getUniqueId(&id)));
  memcpy(out128, id.internal, NCCL_UNIQUE_ID_BYTES);
  return GCG_OK;
}

int gcg_nccl_comm_create(void* ctx, int32_t nranks, int32_t rank, const uint8_t* id128,
                         void** comm_out) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  NcclApi& api = nccl();
  if (!c || !api.ok || !id128 || !comm_out || nranks < 1 || rank < 0 || rank >= nranks)
    return GCG_ERR_ARG;
  ncclUniqueId id;
  memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t comm = nullptr;
  GCG_TRY(cuda_status(cudaSetDevice(c->device)));
  GCG_TRY(nccl_status(api.commInitRank(&comm, nranks, id, rank)));
  *comm_out = comm;
  return GCG_OK;
}

int gcg_nccl_comm_destroy(void* comm) {
  NcclApi& api = nccl();
  if (!api.ok || !comm) return GCG_ERR_ARG;
  return nccl_status(api.commDestroy(reinterpret_cast<ncclComm_t>(comm)));
}

// in-place sum of `count` doubles over the communicator, on the context stream
int gcg_nccl_allreduce_sum(void* ctx, void* comm, double* buf, int64_t count) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  NcclApi& api = nccl();
  if (!c || !api.ok || !comm || !buf || count < 0) return GCG_ERR_ARG;
  return nccl_status(api.allReduce(buf, buf, (size_t)count, ncclDouble, ncclSum,
                                   reinterpret_cast<ncclComm_t>(comm), c->stream));
}

}  // extern "C"
