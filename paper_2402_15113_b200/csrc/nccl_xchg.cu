// nccl_xchg.cu — the library-owned NCCL communicators of a sharded memory
// handle (row E).  The data moves by direct stores into the peers' receive
// windows (shard.cu); NCCL provides only the stream-ordered barrier between
// a phase that writes peers' windows and the phase that reads its own: a
// one-int all-reduce, which completes on a rank only after every rank has
// reached it, i.e. after every rank's preceding kernels (whose remote stores
// end with a system-scope fence) have finished.  Two communicators, so a
// fetch (on the prep stream) and a commit (on the update stream) can each
// barrier without ordering the two streams: every collective of one
// communicator is issued in the same order on every rank.
#include <nccl.h>

#include "internal.cuh"

namespace mspipe {

mspipe_status nccl_comm_init(mspipe_memory* st, const void* unique_id) {
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  ncclComm_t comm = nullptr, comm2 = nullptr;
  ncclResult_t r = ncclCommInitRank(&comm, st->world, id, st->rank);
  if (r != ncclSuccess) return fail(MSPIPE_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  st->nccl_comm = comm;
  r = ncclCommSplit(comm, 0, st->rank, &comm2, nullptr);  // the fetch communicator (collective)
  if (r != ncclSuccess) return fail(MSPIPE_ENCCL, "ncclCommSplit: %s", ncclGetErrorString(r));
  st->nccl_comm_fetch = comm2;
  return MSPIPE_OK;
}

void nccl_comm_destroy(mspipe_memory* st) {
  if (st && st->nccl_comm_fetch) {
    ncclCommDestroy((ncclComm_t)st->nccl_comm_fetch);
    st->nccl_comm_fetch = nullptr;
  }
  if (st && st->nccl_comm) {
    ncclCommDestroy((ncclComm_t)st->nccl_comm);
    st->nccl_comm = nullptr;
  }
}

mspipe_status nccl_barrier(mspipe_memory* st, bool fetch, cudaStream_t s) {
  ncclComm_t comm = (ncclComm_t)(fetch ? st->nccl_comm_fetch : st->nccl_comm);
  ncclResult_t r = ncclAllReduce(st->sh_bar + (fetch ? 1 : 0), st->sh_bar + (fetch ? 1 : 0), 1, ncclInt32, ncclMax,
                                 comm, s);
  if (r != ncclSuccess) return fail(MSPIPE_ENCCL, "barrier all-reduce: %s", ncclGetErrorString(r));
  return MSPIPE_OK;
}

int32_t nccl_unique_id_bytes() { return (int32_t)sizeof(ncclUniqueId); }

mspipe_status nccl_get_unique_id(void* out) {
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(MSPIPE_ENCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  memcpy(out, &id, sizeof(id));
  return MSPIPE_OK;
}

}  // namespace mspipe
