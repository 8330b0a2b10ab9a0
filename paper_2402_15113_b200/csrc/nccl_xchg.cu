// nccl_xchg.cu — the library-owned NCCL communicator of a sharded memory
// handle and the all-to-all that carries fetch requests / replies and
// write-back records over NVLink (row E).  Buffers are fixed-capacity blocks
// of `chunk` bytes per peer, so the exchange needs no host-side counts and is
// capturable into CUDA graphs.
#include <nccl.h>

#include "internal.cuh"

namespace mspipe {

mspipe_status nccl_comm_init(mspipe_memory* st, const void* unique_id) {
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  ncclComm_t comm = nullptr;
  ncclResult_t r = ncclCommInitRank(&comm, st->world, id, st->rank);
  if (r != ncclSuccess) return fail(MSPIPE_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  st->nccl_comm = comm;
  return MSPIPE_OK;
}

void nccl_comm_destroy(mspipe_memory* st) {
  if (st && st->nccl_comm) {
    ncclCommDestroy((ncclComm_t)st->nccl_comm);
    st->nccl_comm = nullptr;
  }
}

mspipe_status nccl_alltoall(mspipe_memory* st, const void* send, void* recv, size_t chunk, cudaStream_t s) {
  ncclComm_t comm = (ncclComm_t)st->nccl_comm;
  ncclResult_t r = ncclGroupStart();
  for (int p = 0; p < st->world && r == ncclSuccess; ++p) {
    r = ncclSend((const char*)send + (size_t)p * chunk, chunk, ncclUint8, p, comm, s);
    if (r == ncclSuccess) r = ncclRecv((char*)recv + (size_t)p * chunk, chunk, ncclUint8, p, comm, s);
  }
  const ncclResult_t r2 = ncclGroupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) return fail(MSPIPE_ENCCL, "all-to-all: %s", ncclGetErrorString(r));
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
