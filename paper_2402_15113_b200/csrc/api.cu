// api.cu — the extern "C" entry points of include/mspipe.h: argument checks,
// handle state, the staleness gate, and dispatch to the kernels.
#include <stdarg.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include "internal.cuh"

namespace mspipe {

__device__ int g_dev_err = 0;

static thread_local char t_last_error[512] = "";

mspipe_status fail(mspipe_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(t_last_error, sizeof(t_last_error), fmt, ap);
  va_end(ap);
  return s;
}

mspipe_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return MSPIPE_OK;
  return fail(MSPIPE_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

int env_int(const char* name, int def) {
  const char* e = getenv(name);
  return (e && *e) ? atoi(e) : def;
}

static mspipe_status after_launch(const char* what) {
  return cuda_status(cudaGetLastError(), what);
}

static bool tcsr_ok(const mspipe_tcsr* g) {
  return g && g->num_nodes >= 0 && g->nnz >= 0 && g->indptr && (g->nnz == 0 || (g->nbr && g->eid && g->ts));
}

}  // namespace mspipe

using namespace mspipe;

extern "C" {

int32_t mspipe_abi_version(void) { return MSPIPE_ABI_VERSION; }

const char* mspipe_last_error(void) { return t_last_error; }

mspipe_status mspipe_check(void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_status(e, "mspipe_check: stream");
  int h = 0;
  e = cudaMemcpyFromSymbol(&h, g_dev_err, sizeof(int));
  if (e != cudaSuccess) return cuda_status(e, "mspipe_check: flag read");
  if (h != 0) {
    int z = 0;
    cudaMemcpyToSymbol(g_dev_err, &z, sizeof(int));
    return fail(MSPIPE_ERANGE, "device error flag 0x%x (1=id out of range, 2=capacity)", h);
  }
  return MSPIPE_OK;
}

mspipe_status mspipe_sample_recent(const mspipe_tcsr* g, const int32_t* roots,
                                   const double* query_ts, int64_t num_roots, int32_t fanout,
                                   int32_t* out_nbr, int32_t* out_eid, double* out_ts,
                                   float* out_dt, int32_t* out_cnt, int32_t* out_sub_ids,
                                   void* stream) {
  if (!tcsr_ok(g)) return fail(MSPIPE_EINVAL, "sample_recent: bad T-CSR");
  if (num_roots < 0 || fanout < 1 || fanout > 64) return fail(MSPIPE_EINVAL, "sample_recent: num_roots=%lld fanout=%d", (long long)num_roots, fanout);
  if (num_roots == 0) return MSPIPE_OK;
  if (!roots || !query_ts || !out_nbr || !out_eid || !out_ts || !out_dt || !out_cnt)
    return fail(MSPIPE_EINVAL, "sample_recent: null output/input");
  launch_sample(to_tcsr(g), roots, query_ts, nullptr, nullptr, nullptr, nullptr, 0, num_roots,
                fanout, out_nbr, out_eid, out_ts, out_dt, out_cnt, out_sub_ids, (cudaStream_t)stream);
  return after_launch("sample_recent");
}

mspipe_status mspipe_sample_batch(const mspipe_tcsr* g, const int32_t* src, const int32_t* dst,
                                  const int32_t* neg, const double* ts, int64_t num_events,
                                  int32_t fanout, int32_t* out_nbr, int32_t* out_eid,
                                  double* out_ts, float* out_dt, int32_t* out_cnt,
                                  int32_t* out_sub_ids, void* stream) {
  if (!tcsr_ok(g)) return fail(MSPIPE_EINVAL, "sample_batch: bad T-CSR");
  if (num_events < 0 || fanout < 1 || fanout > 64) return fail(MSPIPE_EINVAL, "sample_batch: num_events=%lld fanout=%d", (long long)num_events, fanout);
  if (num_events == 0) return MSPIPE_OK;
  if (!src || !dst || !neg || !ts || !out_nbr || !out_eid || !out_ts || !out_dt || !out_cnt)
    return fail(MSPIPE_EINVAL, "sample_batch: null output/input");
  launch_sample(to_tcsr(g), nullptr, nullptr, src, dst, neg, ts, num_events, 3 * num_events, fanout,
                out_nbr, out_eid, out_ts, out_dt, out_cnt, out_sub_ids, (cudaStream_t)stream);
  return after_launch("sample_batch");
}

static mspipe_status nccl_warmup(mspipe_memory* st);

// a library-owned stream of the handle (non-blocking) and a fork / join event
// pair for work the library runs beside the caller's stream; inside a stream
// capture the record / wait pairs become graph edges.  which: 0 = the commit's
// write-back branch, 1 = the prep's mitigation branch (separate streams: one
// shared stream would order the two branches).  Created by
// mspipe_memory_create; one host thread per handle (header), so no locking.
static cudaError_t aux_stream(mspipe_memory* st, cudaStream_t* side, cudaEvent_t* fork, cudaEvent_t* join,
                              int which) {
  if (which < 0 || which > 1 || !st->aux[which]) return cudaErrorInvalidResourceHandle;
  *side = st->aux[which];
  *fork = st->aux_fork[which];
  *join = st->aux_join[which];
  return cudaSuccess;
}

static cudaError_t aux_create(mspipe_memory* st) {
  cudaError_t e = cudaSuccess;
  for (int w = 0; w < 2 && e == cudaSuccess; ++w) {
    e = cudaStreamCreateWithFlags(&st->aux[w], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&st->aux_fork[w], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&st->aux_join[w], cudaEventDisableTiming);
  }
  return e;
}

mspipe_status mspipe_memory_create(mspipe_memory** out, int64_t num_nodes, int32_t mem_dim,
                                   int32_t edge_dim, int32_t staleness_k, float* mem,
                                   double* mem_ts, float* mail, double* mail_ts,
                                   int64_t mail_stride, int32_t rank, int32_t world,
                                   const void* nccl_unique_id) {
  if (!out) return fail(MSPIPE_EINVAL, "memory_create: out is NULL");
  *out = nullptr;
  if (num_nodes < 1 || num_nodes > INT32_MAX || mem_dim < 4 || mem_dim % 4 || edge_dim < 0 || staleness_k < 0)
    return fail(MSPIPE_EINVAL, "memory_create: num_nodes=%lld mem_dim=%d (multiple of 4) edge_dim=%d k=%d",
                (long long)num_nodes, mem_dim, edge_dim, staleness_k);
  int32_t Dm = 2 * mem_dim + edge_dim;
  if (mail_stride < Dm || mail_stride % 4) return fail(MSPIPE_EINVAL, "memory_create: mail_stride=%lld must be >= %d and a multiple of 4", (long long)mail_stride, Dm);
  if (!mem || !mem_ts || !mail || !mail_ts) return fail(MSPIPE_EINVAL, "memory_create: null table");
  if (world < 1 || world > 64 || rank < 0 || rank >= world)
    return fail(MSPIPE_EINVAL, "memory_create: rank=%d world=%d (1..64)", rank, world);
  (void)num_sms();  // cache the SM count now: later calls may run under stream capture
  mspipe_memory* st = new mspipe_memory();
  st->num_nodes = num_nodes;
  st->mem_dim = mem_dim;
  st->edge_dim = edge_dim;
  st->mail_dim = Dm;
  st->k = staleness_k;
  st->mem = mem;
  st->mem_ts = mem_ts;
  st->mail = mail;
  st->mail_ts = mail_ts;
  st->mail_stride = mail_stride;
  st->rank = rank;
  st->world = world;
  st->committed = 0;
  cudaGetDevice(&st->device);
  st->local_rows = (num_nodes - rank + world - 1) / world;
  cudaError_t e = cudaMalloc(&st->scratch, sizeof(int32_t) * (size_t)num_nodes);
  if (e == cudaSuccess) e = cudaMemset(st->scratch, 0xFF, sizeof(int32_t) * (size_t)num_nodes);
  if (e == cudaSuccess) e = cudaMalloc(&st->sample_hint, sizeof(int64_t) * (size_t)num_nodes);
  if (e == cudaSuccess) e = cudaMemset(st->sample_hint, 0, sizeof(int64_t) * (size_t)num_nodes);
  if (e == cudaSuccess && world > 1) {
    st->sh_cap = (num_nodes + world - 1) / world;
    st->sh_capw = st->sh_cap;  // unique nodes per owner never exceed its shard
    shard_layout(st);
    e = cudaMalloc(&st->sh_needed, (size_t)num_nodes);
    if (e == cudaSuccess) e = cudaMemset(st->sh_needed, 0, (size_t)num_nodes);
    if (e == cudaSuccess) e = cudaMalloc(&st->sh_slot_of, sizeof(int32_t) * (size_t)num_nodes);
    if (e == cudaSuccess) e = cudaMalloc(&st->sh_dest, sizeof(int32_t) * (size_t)num_nodes);
    if (e == cudaSuccess) e = cudaMalloc(&st->sh_keytab, sizeof(unsigned long long) * (size_t)st->local_rows);
    if (e == cudaSuccess) e = cudaMemset(st->sh_keytab, 0, sizeof(unsigned long long) * (size_t)st->local_rows);
    if (e == cudaSuccess) e = cudaMalloc(&st->sh_window, (size_t)st->sh_win_bytes);
    if (e == cudaSuccess) e = cudaMemset(st->sh_window, 0, (size_t)st->sh_win_bytes);
    if (e == cudaSuccess) e = cudaMalloc(&st->sh_peers, sizeof(uint8_t*) * (size_t)world);
    if (e == cudaSuccess) e = cudaMalloc(&st->sh_sent, 3 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(st->sh_sent, 0, 3 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMalloc(&st->sh_bar, 2 * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMemset(st->sh_bar, 0, 2 * sizeof(int32_t));
  }
  if (e == cudaSuccess) e = aux_create(st);  // the side streams exist before any stream capture needs them
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    mspipe_memory_destroy(st);
    return cuda_status(e, "memory_create: scratch");
  }
  if (world > 1 && nccl_unique_id) {
    mspipe_status rc = nccl_comm_init(st, nccl_unique_id);
    if (rc == MSPIPE_OK) rc = nccl_warmup(st);
    if (rc != MSPIPE_OK) {
      mspipe_memory_destroy(st);
      return rc;
    }
  }
  *out = st;
  return MSPIPE_OK;
}

// set 1 <- set 0, no previous commit (version 0 in both sets); every copy is
// ordered on `s` (the caller's stream: its earlier writes to set 0, e.g. a
// re-zeroing, are seen) and the host waits for `s` before the bookkeeping
static mspipe_status db_mirror(mspipe_memory* st, cudaStream_t s) {
  const size_t N = (size_t)st->num_nodes;
  cudaError_t e = cudaMemcpyAsync(st->mem1, st->mem, sizeof(float) * N * st->mem_dim, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(st->mem_ts1, st->mem_ts, sizeof(double) * N, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(st->mail1, st->mail, sizeof(float) * N * st->mail_stride, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(st->mail_ts1, st->mail_ts, sizeof(double) * N, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(st->prev_num, 0, 2 * sizeof(int32_t), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(st->stamps, 0, sizeof(int32_t) * (size_t)(st->k + 1) * N, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  st->prev_max[0] = st->prev_max[1] = 0;
  st->caught_up = 0;
  for (int r = 0; r <= st->k; ++r) st->stamp_iter[r] = 0;
  return cuda_status(e, "memory double buffer: mirror");
}

mspipe_status mspipe_memory_double_buffer(mspipe_memory* st, float* mem1, double* mem_ts1, float* mail1,
                                          double* mail_ts1) {
  if (!st) return fail(MSPIPE_EINVAL, "memory_double_buffer: NULL handle");
  if (st->world != 1) return fail(MSPIPE_EUNSUPPORTED, "memory_double_buffer: world > 1");
  if (st->db) return fail(MSPIPE_EINVAL, "memory_double_buffer: already double-buffered");
  if (st->committed != 0) return fail(MSPIPE_EORDER, "memory_double_buffer: committed=%lld (must be 0)", (long long)st->committed);
  if (!mem1 || !mem_ts1 || !mail1 || !mail_ts1) return fail(MSPIPE_EINVAL, "memory_double_buffer: null table");
  cudaError_t e = cudaMalloc(&st->prev_nodes, sizeof(int32_t) * 2 * (size_t)st->num_nodes);
  if (e == cudaSuccess) e = cudaMalloc(&st->prev_num, 2 * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMalloc(&st->stamps, sizeof(int32_t) * (size_t)(st->k + 1) * (size_t)st->num_nodes);
  if (e != cudaSuccess) return cuda_status(e, "memory_double_buffer: alloc");
  st->stamp_iter = new int64_t[st->k + 1]();
  st->mem1 = mem1;
  st->mem_ts1 = mem_ts1;
  st->mail1 = mail1;
  st->mail_ts1 = mail_ts1;
  st->db = 1;
  return db_mirror(st, cudaStreamLegacy);
}

mspipe_status mspipe_memory_set_committed(mspipe_memory* st, int64_t version) {
  if (!st) return fail(MSPIPE_EINVAL, "memory_set_committed: NULL handle");
  if (version < 0) return fail(MSPIPE_EINVAL, "memory_set_committed: version=%lld", (long long)version);
  st->committed = version;
  return MSPIPE_OK;
}

mspipe_status mspipe_memory_tables(const mspipe_memory* st, int64_t version, float** mem, double** mem_ts,
                                   float** mail, double** mail_ts) {
  if (!st) return fail(MSPIPE_EINVAL, "memory_tables: NULL handle");
  if (!(version == st->committed || (st->db && version == st->committed - 1 && version >= 0)))
    return fail(MSPIPE_EINVAL, "memory_tables: version %lld is not held (committed=%lld, double-buffered=%d)",
                (long long)version, (long long)st->committed, st->db);
  const TableSet t = table_set(st, version);
  if (mem) *mem = t.mem;
  if (mem_ts) *mem_ts = t.mem_ts;
  if (mail) *mail = t.mail;
  if (mail_ts) *mail_ts = t.mail_ts;
  return MSPIPE_OK;
}

// where the catch-up of a double-buffered commit runs: 0 = its own kernel
// before the commit, 1 = inside the commit's GEMM kernel, 2 = inside the
// mspipe_memory_prep that precedes the commit (falling back to 1, then 0,
// when the winners of the commit are not stamped yet)
static int catchup_mode() { return env_int("MSPIPE_CATCHUP", 2); }

// the catch-up rows of commit c as a CatchUp (stamps of commit c's winners assumed written)
static CatchUp catchup_args(const mspipe_memory* st, int64_t c) {
  const int64_t N = st->num_nodes;
  const int q = (int)((c - 1) & 1);
  const TableSet o = table_set(st, c - 1), n = table_set(st, c);
  return CatchUp{st->prev_nodes + q * N, st->prev_num + q, o.mem, o.mem_ts, o.mail, o.mail_ts, n.mem, n.mem_ts,
                 n.mail, n.mail_ts, st->stamps + (c % (st->k + 1)) * N, (int32_t)c};
}

// double-buffered commit c, first half (see k_catchup); copy_rows = false when
// a prep already enqueued them: then only this commit's winner list is saved
static cudaError_t db_catchup(mspipe_memory* st, int64_t c, const int32_t* nodes, const int32_t* num, int64_t max_n,
                              cudaStream_t s, bool copy_rows = true) {
  const int p = (int)(c & 1), q = p ^ 1;
  const int64_t N = st->num_nodes;
  const TableSet from = table_set(st, c - 1), to = table_set(st, c);
  launch_catchup(st->prev_nodes + q * N, copy_rows ? st->prev_num + q : nullptr, copy_rows ? st->prev_max[q] : 0,
                 from.mem, from.mem_ts, from.mail,
                 from.mail_ts, to.mem, to.mem_ts, to.mail, to.mail_ts, st->mem_dim, st->mail_stride,
                 max_n > 0 ? nodes : nullptr, max_n > 0 ? num : nullptr, max_n, st->prev_nodes + p * N,
                 st->prev_num + p, s);
  return cudaGetLastError();
}

mspipe_status mspipe_memory_destroy(mspipe_memory* st) {
  if (!st) return MSPIPE_OK;
  nccl_comm_destroy(st);
  for (int p = 0; p < st->world && p < 64; ++p)
    if (st->sh_peer_ipc[p] && st->sh_peer_host[p]) cudaIpcCloseMemHandle(st->sh_peer_host[p]);
  void* bufs[] = {st->scratch, st->sample_hint, st->sh_needed, st->sh_slot_of, st->sh_dest, st->sh_keytab, st->sh_window,
                  st->sh_peers, st->sh_sent, st->sh_bar, st->prev_nodes,
                  st->prev_num, st->stamps};
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (int w = 0; w < 2; ++w) {
    if (st->aux_fork[w]) cudaEventDestroy(st->aux_fork[w]);
    if (st->aux_join[w]) cudaEventDestroy(st->aux_join[w]);
    if (st->aux[w]) cudaStreamDestroy(st->aux[w]);
  }
  delete[] st->stamp_iter;
  delete st;
  return MSPIPE_OK;
}

int64_t mspipe_memory_local_rows(const mspipe_memory* st) { return st ? st->local_rows : -1; }

int64_t mspipe_memory_committed(const mspipe_memory* st) { return st ? st->committed : -1; }

mspipe_status mspipe_memory_reset(mspipe_memory* st, int32_t zero_tables, void* stream) {
  if (!st) return fail(MSPIPE_EINVAL, "memory_reset: NULL handle");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t N = (size_t)st->local_rows;
  cudaError_t e = cudaSuccess;
  if (zero_tables) {  // S_0 = 0 (G17), stream-ordered behind the caller's earlier work
    e = cudaMemsetAsync(st->mem, 0, sizeof(float) * N * st->mem_dim, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(st->mem_ts, 0, sizeof(double) * N, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(st->mail, 0, sizeof(float) * N * st->mail_stride, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(st->mail_ts, 0, sizeof(double) * N, s);
    if (e != cudaSuccess) return cuda_status(e, "memory_reset: zero");
  }
  st->committed = 0;
  if (st->db) {  // version 0 = set 0 (the caller's initial state), mirrored into set 1
    mspipe_status rc = db_mirror(st, s);
    if (rc != MSPIPE_OK) return rc;
  }
  if (st->sh_keytab) {  // keys and the sent-bytes counters restart with the stream
    e = cudaMemsetAsync(st->sh_keytab, 0, sizeof(unsigned long long) * (size_t)st->local_rows, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(st->sh_sent, 0, 3 * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return cuda_status(e, "memory_reset");
  }
  e = cudaStreamSynchronize(s);
  return cuda_status(e, "memory_reset");
}

mspipe_status mspipe_memory_fetch(mspipe_memory* st, int64_t iteration, const int32_t* ids,
                                  int64_t n, float* out_mem, double* out_mem_ts, float* out_mail,
                                  double* out_mail_ts, const mspipe_mitigation* mit,
                                  int64_t* out_version, void* stream) {
  if (!st) return fail(MSPIPE_EINVAL, "memory_fetch: NULL handle");
  if (iteration < 1 || n < 0) return fail(MSPIPE_EINVAL, "memory_fetch: iteration=%lld n=%lld", (long long)iteration, (long long)n);
  // Staleness gate, Eq. (2) / Alg. 1 L8-L11: i-1-k <= committed <= i-1.
  if (st->committed < iteration - 1 - st->k || st->committed > iteration - 1)
    return fail(MSPIPE_ESTALE, "memory_fetch: iteration %lld with committed=%lld violates k=%d",
                (long long)iteration, (long long)st->committed, st->k);
  if (n > 0 && (!ids || !out_mem || !out_mem_ts)) return fail(MSPIPE_EINVAL, "memory_fetch: null ids/outputs");
  if ((out_mail == nullptr) != (out_mail_ts == nullptr)) return fail(MSPIPE_EINVAL, "memory_fetch: out_mail and out_mail_ts go together");
  if (st->world > 1) {
    if (mit) return fail(MSPIPE_EUNSUPPORTED, "memory_fetch: world > 1 runs MSPipe-S through the mspipe_shard_mitigation_* phases");
    if (st->sh_connected != 1)
      return fail(MSPIPE_EUNSUPPORTED, "memory_fetch: %s", st->sh_connected == 2 ? "in-process rank: drive the mspipe_shard_* phases" : "not connected (mspipe_shard_connect)");
    cudaStream_t s = (cudaStream_t)stream;
    mspipe_status rc = mspipe_shard_fetch_plan(st, iteration, ids, n, out_mail != nullptr, stream);
    if (rc == MSPIPE_OK) rc = mspipe_shard_exchange(st, MSPIPE_XCHG_FETCH_IDS, stream);
    if (rc == MSPIPE_OK) rc = mspipe_shard_fetch_serve(st, stream);
    if (rc == MSPIPE_OK) rc = mspipe_shard_exchange(st, MSPIPE_XCHG_FETCH_ROWS, stream);
    if (rc == MSPIPE_OK)
      rc = mspipe_shard_fetch_finish(st, ids, n, out_mem, out_mem_ts, out_mail, out_mail_ts, out_version, stream);
    (void)s;
    return rc;
  }
  if (mit) {
    if (!tcsr_ok(mit->g) || !mit->src || !mit->dst || !mit->ts || !mit->out_h || mit->num_events < 0)
      return fail(MSPIPE_EINVAL, "memory_fetch: bad mitigation arguments");
    if (!(mit->lambda >= 0.f && mit->lambda <= 1.f) || mit->n_sim < 0 || mit->n_sim > 16 || mit->fanout < 1 || mit->fanout > 16)
      return fail(MSPIPE_EINVAL, "memory_fetch: lambda=%g n_sim=%d fanout=%d (fanout<=16, n_sim<=16)", mit->lambda, mit->n_sim, mit->fanout);
  }
  cudaStream_t s = (cudaStream_t)stream;
  const TableSet t = table_set(st, st->committed);  // version v(i) = committed (stream order)
  if (n > 0)
    launch_fetch(ids, n, st->num_nodes, t.mem, t.mem_ts, st->mem_dim, out_mail ? t.mail : nullptr,
                 t.mail_ts, st->mail_stride, out_mem, out_mem_ts, out_mail, out_mail_ts, s);
  if (mit && mit->num_events > 0)
    launch_mitigate(to_tcsr(mit->g), mit->src, mit->dst, mit->ts, mit->num_events, t.mem, t.mem_ts,
                    st->mem_dim, mit->lambda, mit->gamma, mit->n_sim, mit->fanout, mit->out_h,
                    mit->out_omega, mit->out_elig, s);
  if (out_version) *out_version = st->committed;
  return after_launch("memory_fetch");
}

mspipe_status mspipe_gru_create(mspipe_gru** out, int32_t mem_dim, int32_t edge_dim,
                                int32_t time_dim, int32_t precision, int64_t max_events,
                                const float* w_ih, const float* w_hh, const float* b_ih,
                                const float* b_hh, const float* time_w, const float* time_b,
                                void* stream) {
  return mspipe_updater_create(out, mem_dim, edge_dim, time_dim, precision, MSPIPE_CELL_GRU,
                               MSPIPE_MAILBOX_IMMEDIATE, max_events, w_ih, w_hh, b_ih, b_hh, time_w, time_b, stream);
}

mspipe_status mspipe_updater_create(mspipe_gru** out, int32_t mem_dim, int32_t edge_dim, int32_t time_dim,
                                    int32_t precision, int32_t cell, int32_t mailbox, int64_t max_events,
                                    const float* w_ih, const float* w_hh, const float* b_ih, const float* b_hh,
                                    const float* time_w, const float* time_b, void* stream) {
  if (!out) return fail(MSPIPE_EINVAL, "gru_create: out is NULL");
  if ((cell != MSPIPE_CELL_GRU && cell != MSPIPE_CELL_RNN) ||
      (mailbox != MSPIPE_MAILBOX_IMMEDIATE && mailbox != MSPIPE_MAILBOX_DEFERRED))
    return fail(MSPIPE_EINVAL, "updater_create: cell=%d mailbox=%d", cell, mailbox);
  if ((cell != MSPIPE_CELL_GRU || mailbox != MSPIPE_MAILBOX_IMMEDIATE) && precision != MSPIPE_FP32_3XTF32 &&
      !(precision == MSPIPE_BF16 && mailbox == MSPIPE_MAILBOX_IMMEDIATE))
    return fail(MSPIPE_EUNSUPPORTED, "updater_create: variants need a tensor-core precision (deferred: 3xTF32)");
  *out = nullptr;
  if (mem_dim < 4 || mem_dim % 4 || edge_dim < 0 || time_dim < 0 || max_events < 1 || max_events > 16384)
    return fail(MSPIPE_EINVAL, "gru_create: mem_dim=%d edge_dim=%d time_dim=%d max_events=%lld (1..16384)",
                mem_dim, edge_dim, time_dim, (long long)max_events);
  if (!w_ih || !w_hh || !b_ih || !b_hh || (time_dim > 0 && (!time_w || !time_b)))
    return fail(MSPIPE_EINVAL, "gru_create: null weight");
  if (precision != MSPIPE_FP32_SIMT && precision != MSPIPE_FP32_3XTF32 && precision != MSPIPE_BF16)
    return fail(MSPIPE_EUNSUPPORTED, "gru_create: precision %d not in this build", precision);
  mspipe_gru* p = new mspipe_gru();
  GruDesc& d = p->d;
  d.M = mem_dim;
  d.He = edge_dim;
  d.Dt = time_dim;
  d.Dm = 2 * mem_dim + edge_dim;
  d.Dx = d.Dm + time_dim;
  d.K = d.Dx + mem_dim;
  d.bf16 = precision == MSPIPE_BF16 ? 1 : 0;
  d.Kpad = d.bf16 ? (d.K + 63) / 64 * 64 : (d.K + 31) / 32 * 32;
  d.cell = cell;
  d.mailbox = mailbox;
  d.Npad = (mem_dim + 31) / 32 * 128;
  if (precision != MSPIPE_FP32_SIMT && d.Kpad > 2048) {
    delete p;
    return fail(MSPIPE_EUNSUPPORTED, "gru_create: K = 2M + He + Dt + M = %d > 2048 on the tensor-core path", d.K);
  }
  p->precision = precision;
  p->max_events = max_events;
  cudaStream_t s = (cudaStream_t)stream;
  (void)num_sms();
  cudaError_t e = precision == MSPIPE_FP32_SIMT
                      ? cudaMalloc(&p->wpack, sizeof(float) * (size_t)d.Kpad * d.Npad)
                      : cudaMalloc(&p->wtc, sizeof(float) * gru_tc_packed_floats(d));
  if (e == cudaSuccess && precision != MSPIPE_FP32_SIMT)
    e = cudaMalloc(&p->xbuf, sizeof(float) * gru_tc_xbuf_floats(d, max_events));
  if (e == cudaSuccess)
    e = cudaMalloc(&p->bias, sizeof(float) * std::max<size_t>((size_t)d.Npad, gru_tc_bias_floats(d)));
  if (e == cudaSuccess) e = cudaMalloc(&p->time_w, sizeof(float) * (size_t)(time_dim > 0 ? time_dim : 1));
  if (e == cudaSuccess) e = cudaMalloc(&p->time_b, sizeof(float) * (size_t)(time_dim > 0 ? time_dim : 1));
  if (e == cudaSuccess && time_dim > 0) e = cudaMemcpyAsync(p->time_w, time_w, sizeof(float) * time_dim, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess && time_dim > 0) e = cudaMemcpyAsync(p->time_b, time_b, sizeof(float) * time_dim, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) {
    mspipe_gru_destroy(p);
    return cuda_status(e, "gru_create: alloc");
  }
  d.wpack = p->wpack;
  d.bias = p->bias;
  d.time_w = p->time_w;
  d.time_b = p->time_b;
  if (precision == MSPIPE_FP32_SIMT) launch_gru_pack(w_ih, w_hh, b_ih, b_hh, d, p->wpack, p->bias, s);
  else launch_gru_pack_tc(w_ih, w_hh, b_ih, b_hh, d, p->wtc, p->bias, s);
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    mspipe_gru_destroy(p);
    return cuda_status(e, "gru_create: pack");
  }
  *out = p;
  return MSPIPE_OK;
}

mspipe_status mspipe_message_build_deferred(const mspipe_gru* gru, const double* ts, int64_t num_events,
                                            const float* snap_mem, const double* snap_mem_ts,
                                            const float* snap_mail, int64_t mail_stride, int64_t snap_step,
                                            const int32_t* winner, const int32_t* num_unique, double* out_ts,
                                            void* workspace, size_t ws_bytes, void* stream) {
  if (!gru) return fail(MSPIPE_EINVAL, "message_build_deferred: NULL handle");
  if (gru->d.mailbox != MSPIPE_MAILBOX_DEFERRED || gru->precision != MSPIPE_FP32_3XTF32)
    return fail(MSPIPE_EUNSUPPORTED, "message_build_deferred: needs a deferred-mailbox MSPIPE_FP32_3XTF32 handle");
  if (num_events < 0 || num_events > gru->max_events || snap_step < 1 || mail_stride < gru->d.Dm)
    return fail(MSPIPE_EINVAL, "message_build_deferred: num_events=%lld snap_step=%lld mail_stride=%lld",
                (long long)num_events, (long long)snap_step, (long long)mail_stride);
  if (num_events == 0) return MSPIPE_OK;
  if (!ts || !snap_mem || !snap_mem_ts || !snap_mail || !winner || !num_unique || !out_ts || !workspace ||
      ws_bytes < mspipe_gru_workspace_size(gru, num_events))
    return fail(MSPIPE_EINVAL, "message_build_deferred: null argument or workspace too small");
  cudaError_t e = launch_build_deferred(gru->d, (float*)workspace, ts, num_events, snap_mem, snap_mem_ts, snap_mail,
                                        mail_stride, snap_step, winner, num_unique, out_ts, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_status(e, "message_build_deferred: launch");
  return after_launch("message_build_deferred");
}

mspipe_status mspipe_memory_mail_deferred(mspipe_memory* st, int64_t commit_version, const int32_t* src,
                                          const int32_t* dst, const double* ts, const float* edge_feat,
                                          int64_t num_events, const int32_t* nodes, const int32_t* winner,
                                          const int32_t* num_unique, void* stream) {
  if (!st) return fail(MSPIPE_EINVAL, "memory_mail_deferred: NULL handle");
  if (st->world != 1) return fail(MSPIPE_EUNSUPPORTED, "memory_mail_deferred: world > 1");
  if (commit_version != st->committed)
    return fail(MSPIPE_EORDER, "memory_mail_deferred: commit_version=%lld but committed=%lld",
                (long long)commit_version, (long long)st->committed);
  if (num_events < 0) return fail(MSPIPE_EINVAL, "memory_mail_deferred: num_events=%lld", (long long)num_events);
  if (num_events == 0) return MSPIPE_OK;
  if (!src || !dst || !ts || (st->edge_dim > 0 && !edge_feat) || !nodes || !winner || !num_unique)
    return fail(MSPIPE_EINVAL, "memory_mail_deferred: null argument");
  const TableSet t = table_set(st, commit_version);
  launch_mail_deferred(src, dst, ts, edge_feat, st->edge_dim, nodes, winner, num_unique, 2 * num_events, t.mem,
                       st->mem_dim, t.mail, t.mail_ts, st->mail_stride, st->num_nodes, (cudaStream_t)stream);
  return after_launch("memory_mail_deferred");
}

mspipe_status mspipe_gru_destroy(mspipe_gru* p) {
  if (!p) return MSPIPE_OK;
  if (p->wpack) cudaFree(p->wpack);
  if (p->wtc) cudaFree(p->wtc);
  if (p->xbuf) cudaFree(p->xbuf);
  cudaFree(p->bias);
  cudaFree(p->time_w);
  cudaFree(p->time_b);
  delete p;
  return MSPIPE_OK;
}

mspipe_status mspipe_memory_dedup(mspipe_memory* st, const int32_t* src, const int32_t* dst,
                                  int64_t num_events, int32_t* out_nodes, int32_t* out_winner,
                                  int32_t* out_num_unique, void* stream) {
  if (!st) return fail(MSPIPE_EINVAL, "memory_dedup: NULL handle");
  if (num_events < 0 || num_events > 16384)
    return fail(MSPIPE_EINVAL, "memory_dedup: num_events=%lld (0..16384)", (long long)num_events);
  if (!out_num_unique) return fail(MSPIPE_EINVAL, "memory_dedup: null out_num_unique");
  cudaStream_t s = (cudaStream_t)stream;
  if (num_events == 0) return cuda_status(cudaMemsetAsync(out_num_unique, 0, sizeof(int32_t), s), "memory_dedup");
  if (!src || !dst || !out_nodes || !out_winner) return fail(MSPIPE_EINVAL, "memory_dedup: null input/output");
  launch_dedup(src, dst, num_events, st->scratch, st->num_nodes, out_nodes, out_winner, out_num_unique, s);
  return after_launch("memory_dedup");
}


mspipe_status mspipe_memory_update(mspipe_memory* st, const mspipe_gru* gru, const int32_t* src,
                                   const int32_t* dst, const double* ts, int64_t num_events,
                                   const float* edge_feat, const float* snap_mem,
                                   const double* snap_mem_ts, int64_t snap_step,
                                   const float* snap_h, const int32_t* winner,
                                   const int32_t* num_unique, float* out_mem, double* out_ts,
                                   float* out_mail, void* stream) {
  if (!st || !gru) return fail(MSPIPE_EINVAL, "memory_update: NULL handle");
  if (gru->d.M != st->mem_dim || gru->d.He != st->edge_dim)
    return fail(MSPIPE_EINVAL, "memory_update: GRU dims (M=%d He=%d) != memory dims (M=%d He=%d)", gru->d.M, gru->d.He, st->mem_dim, st->edge_dim);
  if (gru->d.mailbox != MSPIPE_MAILBOX_IMMEDIATE)
    return fail(MSPIPE_EUNSUPPORTED, "memory_update: deferred-mailbox handle (use mspipe_message_build_deferred)");
  if (num_events < 0 || num_events > gru->max_events || snap_step < 1)
    return fail(MSPIPE_EINVAL, "memory_update: num_events=%lld (<= max_events %lld of the GRU handle) snap_step=%lld",
                (long long)num_events, (long long)gru->max_events, (long long)snap_step);
  cudaStream_t s = (cudaStream_t)stream;
  if (num_events == 0) return MSPIPE_OK;
  if (!src || !dst || !ts || (st->edge_dim > 0 && !edge_feat) || !snap_mem || !snap_mem_ts || !winner ||
      !num_unique || !out_mem || !out_ts || !out_mail)
    return fail(MSPIPE_EINVAL, "memory_update: null input/output");
  int32_t* out_winner = const_cast<int32_t*>(winner);
  int32_t* out_num_unique = const_cast<int32_t*>(num_unique);
  int32_t* out_nodes = nullptr;
  if (gru->precision != MSPIPE_FP32_SIMT) {
    cudaError_t e = launch_gru_tc(gru->d, gru->wtc, gru->xbuf, ts, num_events, edge_feat, snap_mem, snap_mem_ts, snap_step,
                                  snap_h, out_winner, out_num_unique, out_mem, out_ts, out_mail, st->mail_stride, s);
    if (e != cudaSuccess) return cuda_status(e, "memory_update: tcgen05 GRU launch");
  } else {
    launch_gru_simt(gru->d, src, dst, ts, num_events, edge_feat, snap_mem, snap_mem_ts, snap_step, snap_h,
                    out_nodes, out_winner, out_num_unique, out_mem, out_ts, out_mail, st->mail_stride, s);
  }
  return after_launch("memory_update");
}

mspipe_status mspipe_memory_writeback(mspipe_memory* st, int64_t commit_version,
                                      const int32_t* nodes, const int32_t* num_unique,
                                      int64_t max_n, const float* new_mem, const double* new_ts,
                                      const float* new_mail, void* stream) {
  if (!st) return fail(MSPIPE_EINVAL, "memory_writeback: NULL handle");
  if (st->world > 1) return fail(MSPIPE_EINVAL, "memory_writeback: world > 1 needs mspipe_memory_writeback_keyed");
  if (commit_version != st->committed + 1)
    return fail(MSPIPE_EORDER, "memory_writeback: commit_version=%lld but committed=%lld", (long long)commit_version, (long long)st->committed);
  if (max_n < 0) return fail(MSPIPE_EINVAL, "memory_writeback: max_n=%lld", (long long)max_n);
  if (max_n > 0 && (!nodes || !num_unique || !new_mem || !new_ts || !new_mail))
    return fail(MSPIPE_EINVAL, "memory_writeback: null input");
  if (st->db) {
    cudaError_t e = db_catchup(st, commit_version, nodes, num_unique, max_n, (cudaStream_t)stream,
                               st->caught_up != commit_version);
    if (e != cudaSuccess) return cuda_status(e, "memory_writeback: catch-up");
  }
  const TableSet t = table_set(st, commit_version);
  if (max_n > 0)
    launch_writeback(nodes, num_unique, max_n, new_mem, new_ts, new_mail, st->mem_dim, st->mail_stride,
                     t.mem, t.mem_ts, t.mail, t.mail_ts, st->num_nodes, (cudaStream_t)stream);
  mspipe_status rc = after_launch("memory_writeback");
  if (rc == MSPIPE_OK) {
    st->committed = commit_version;  // i_upd <- i (Alg. 1 L16)
    st->prev_max[commit_version & 1] = max_n;
  }
  return rc;
}


mspipe_status mspipe_memory_prep(mspipe_memory* st, const mspipe_tcsr* g, int64_t iteration, const int32_t* src,
                                 const int32_t* dst, const int32_t* neg, const double* ts, int64_t num_events,
                                 int32_t fanout, int32_t* out_nbr, int32_t* out_eid, double* out_ts, float* out_dt,
                                 int32_t* out_cnt, int32_t* out_sub_ids, int32_t* out_nodes, int32_t* out_winner,
                                 int32_t* out_num_unique, float* out_mem, double* out_mem_ts, float* out_mail,
                                 double* out_mail_ts, const mspipe_mitigation* mit, int64_t* out_version,
                                 void* stream) {
  if (!st) return fail(MSPIPE_EINVAL, "memory_prep: NULL handle");
  if (st->world > 1) return fail(MSPIPE_EUNSUPPORTED, "memory_prep: fused prep reads local tables; world > 1 uses the sharded fetch");
  if (!tcsr_ok(g) || g->num_nodes != st->num_nodes) return fail(MSPIPE_EINVAL, "memory_prep: bad T-CSR");
  if (iteration < 1 || num_events < 0 || num_events > 8192 || fanout < 1 || fanout > 31)
    return fail(MSPIPE_EINVAL, "memory_prep: iteration=%lld num_events=%lld (<= 8192) fanout=%d (<= 31)",
                (long long)iteration, (long long)num_events, fanout);
  if (st->committed < iteration - 1 - st->k || st->committed > iteration - 1)
    return fail(MSPIPE_ESTALE, "memory_prep: iteration %lld with committed=%lld violates k=%d",
                (long long)iteration, (long long)st->committed, st->k);
  if ((out_mail == nullptr) != (out_mail_ts == nullptr)) return fail(MSPIPE_EINVAL, "memory_prep: out_mail and out_mail_ts go together");
  // every argument is validated before any fork or launch (an error return
  // leaves no branch unjoined and nothing enqueued)
  const bool dedup = out_nodes || out_winner || out_num_unique;
  if (dedup && !(out_nodes && out_winner && out_num_unique))
    return fail(MSPIPE_EINVAL, "memory_prep: out_nodes / out_winner / out_num_unique go together");
  if (num_events > 0 &&
      (!src || !dst || !neg || !ts || !out_nbr || !out_eid || !out_ts || !out_dt || !out_cnt || !out_sub_ids ||
       (dedup && (!out_nodes || !out_winner || !out_num_unique)) || !out_mem || !out_mem_ts))
    return fail(MSPIPE_EINVAL, "memory_prep: null input/output");
  if (mit && mit->num_events > 0) {
    if (!tcsr_ok(mit->g) || !mit->src || !mit->dst || !mit->ts || !mit->out_h)
      return fail(MSPIPE_EINVAL, "memory_prep: bad mitigation arguments");
    if (!(mit->lambda >= 0.f && mit->lambda <= 1.f) || mit->n_sim < 0 || mit->n_sim > 16 || mit->fanout < 1 || mit->fanout > 16)
      return fail(MSPIPE_EINVAL, "memory_prep: lambda=%g n_sim=%d fanout=%d", mit->lambda, mit->n_sim, mit->fanout);
  }
  cudaStream_t s = (cudaStream_t)stream;
  const TableSet t = table_set(st, st->committed);
  // A4 reads only the T-CSR and the tables of the version read, not k_prep's
  // outputs: it runs on a forked branch beside k_prep (MSPIPE_MIT_BRANCH=0: after it)
  bool mit_branch = false;
  cudaEvent_t mit_join = nullptr;
  if (mit && mit->num_events > 0 && env_int("MSPIPE_MIT_BRANCH", 1)) {
    cudaStream_t side;
    cudaEvent_t fork;
    cudaError_t e = aux_stream(st, &side, &fork, &mit_join, 1);
    if (e == cudaSuccess) e = cudaEventRecord(fork, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(side, fork, 0);
    if (e != cudaSuccess) return cuda_status(e, "memory_prep: mitigation fork");
    launch_mitigate(to_tcsr(mit->g), mit->src, mit->dst, mit->ts, mit->num_events, t.mem, t.mem_ts, st->mem_dim,
                    mit->lambda, mit->gamma, mit->n_sim, mit->fanout, mit->out_h, mit->out_omega, mit->out_elig, side);
    e = cudaEventRecord(mit_join, side);
    if (e != cudaSuccess) return cuda_status(e, "memory_prep: mitigation branch");
    mit_branch = true;
  }
  if (num_events > 0) {
    // double-buffered: this launch may also carry the catch-up of the next
    // commit c (its winners already stamped, or stamped by this very launch
    // when c == iteration, k = 0: the commit then follows in stream order).
    // Without the dedup block the stamps of c == iteration may still be in
    // flight on another stream: the commit's GEMM then catches up instead.
    const int64_t c = st->committed + 1;
    const bool cu = st->db && catchup_mode() == 2 && st->caught_up != c &&
                    (dedup ? (st->stamp_iter[c % (st->k + 1)] == c || c == iteration)
                           : (c != iteration && st->stamp_iter[c % (st->k + 1)] == c));
    const CatchUp cua = cu ? catchup_args(st, c) : CatchUp{};
    cudaError_t e = launch_prep(to_tcsr(g), src, dst, neg, ts, num_events, fanout, out_nbr, out_eid, out_ts, out_dt,
                                out_cnt, out_sub_ids, st->scratch, out_nodes, out_winner, out_num_unique, t.mem,
                                t.mem_ts, st->mem_dim, t.mail, t.mail_ts, st->mail_stride, out_mem,
                                out_mem_ts, out_mail, out_mail_ts, s,
                                (st->db && dedup) ? st->stamps + (iteration % (st->k + 1)) * st->num_nodes : nullptr,
                                (int32_t)iteration, cu ? &cua : nullptr,
                                env_int("MSPIPE_SAMPLE_HINT", 1) ? st->sample_hint : nullptr);
    if (e != cudaSuccess) return cuda_status(e, "memory_prep: launch");
    if (st->db && dedup) st->stamp_iter[iteration % (st->k + 1)] = iteration;
    if (cu) st->caught_up = c;
  } else if (out_num_unique) {
    cudaError_t e = cudaMemsetAsync(out_num_unique, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return cuda_status(e, "memory_prep");
  }
  if (mit && mit->num_events > 0) {
    if (mit_branch) {  // joined back: the message build after this call reads out_h
      cudaError_t e = cudaStreamWaitEvent(s, mit_join, 0);
      if (e != cudaSuccess) return cuda_status(e, "memory_prep: mitigation join");
    } else {
      launch_mitigate(to_tcsr(mit->g), mit->src, mit->dst, mit->ts, mit->num_events, t.mem, t.mem_ts, st->mem_dim,
                      mit->lambda, mit->gamma, mit->n_sim, mit->fanout, mit->out_h, mit->out_omega, mit->out_elig, s);
    }
  }
  if (out_version) *out_version = st->committed;
  return after_launch("memory_prep");
}

size_t mspipe_gru_workspace_size(const mspipe_gru* gru, int64_t num_events) {
  if (!gru || gru->precision == MSPIPE_FP32_SIMT || num_events < 0) return 0;
  return sizeof(float) * gru_tc_xbuf_floats(gru->d, num_events);
}

mspipe_status mspipe_message_build(const mspipe_gru* gru, const double* ts, int64_t num_events,
                                   const float* edge_feat, const float* snap_mem,
                                   const double* snap_mem_ts, int64_t snap_step,
                                   const float* snap_h, const int32_t* winner,
                                   const int32_t* num_unique, double* out_ts, float* out_mail,
                                   int64_t mail_stride, void* workspace, size_t ws_bytes, void* stream) {
  if (!gru) return fail(MSPIPE_EINVAL, "message_build: NULL handle");
  if (gru->precision == MSPIPE_FP32_SIMT)
    return fail(MSPIPE_EUNSUPPORTED, "message_build: only for precision MSPIPE_FP32_3XTF32 (use mspipe_memory_update)");
  if (gru->d.mailbox != MSPIPE_MAILBOX_IMMEDIATE)
    return fail(MSPIPE_EUNSUPPORTED, "message_build: deferred-mailbox handle (use mspipe_message_build_deferred)");
  if (num_events < 0 || num_events > gru->max_events || snap_step < 1 || mail_stride < gru->d.Dm || mail_stride % 4)
    return fail(MSPIPE_EINVAL, "message_build: num_events=%lld snap_step=%lld mail_stride=%lld", (long long)num_events,
                (long long)snap_step, (long long)mail_stride);
  if (num_events == 0) return MSPIPE_OK;
  if (ws_bytes < mspipe_gru_workspace_size(gru, num_events) || !workspace)
    return fail(MSPIPE_EINVAL, "message_build: workspace of %zu bytes < %zu", ws_bytes, mspipe_gru_workspace_size(gru, num_events));
  if (!ts || (gru->d.He > 0 && !edge_feat) || !snap_mem || !snap_mem_ts || !winner || !num_unique || !out_ts || !out_mail)
    return fail(MSPIPE_EINVAL, "message_build: null input/output");
  cudaError_t e = launch_gru_tc(gru->d, gru->wtc, (float*)workspace, ts, num_events, edge_feat, snap_mem, snap_mem_ts,
                                snap_step, snap_h, winner, num_unique, nullptr, out_ts, out_mail, mail_stride,
                                (cudaStream_t)stream, kGruBuild);
  if (e != cudaSuccess) return cuda_status(e, "message_build: launch");
  return after_launch("message_build");
}


mspipe_status mspipe_gru_apply(const mspipe_gru* gru, int64_t num_events, const float* snap_mem,
                               int64_t snap_step, const float* snap_h, const int32_t* winner,
                               const int32_t* num_unique, float* out_mem, const void* workspace,
                               size_t ws_bytes, void* stream) {
  if (!gru) return fail(MSPIPE_EINVAL, "gru_apply: NULL handle");
  if (gru->precision == MSPIPE_FP32_SIMT)
    return fail(MSPIPE_EUNSUPPORTED, "gru_apply: only for precision MSPIPE_FP32_3XTF32 (use mspipe_memory_update)");
  if (num_events < 0 || num_events > gru->max_events || snap_step < 1)
    return fail(MSPIPE_EINVAL, "gru_apply: num_events=%lld snap_step=%lld", (long long)num_events, (long long)snap_step);
  if (num_events == 0) return MSPIPE_OK;
  if (ws_bytes < mspipe_gru_workspace_size(gru, num_events) || !workspace)
    return fail(MSPIPE_EINVAL, "gru_apply: workspace of %zu bytes too small", ws_bytes);
  if (!snap_mem || !winner || !num_unique || !out_mem) return fail(MSPIPE_EINVAL, "gru_apply: null input/output");
  cudaError_t e = launch_gru_tc(gru->d, gru->wtc, (float*)workspace, nullptr, num_events, nullptr, snap_mem, nullptr,
                                snap_step, snap_h, winner, num_unique, out_mem, nullptr, nullptr, 0,
                                (cudaStream_t)stream, kGruGemm);
  if (e != cudaSuccess) return cuda_status(e, "gru_apply: launch");
  return after_launch("gru_apply");
}

// one-shot timing pair for the next tensor-core GEMM launch of this thread
// (mspipe_util_kernel_events): recorded right before / after the kernel
static thread_local cudaEvent_t g_kev[2] = {nullptr, nullptr};

static mspipe_status apply_commit_impl(const mspipe_gru* gru, mspipe_memory* st, int64_t commit_version,
                                       int64_t num_events, const float* snap_mem, int64_t snap_step,
                                       const float* snap_h, const int32_t* nodes, const int32_t* winner,
                                       const int32_t* num_unique, const double* new_ts, const float* new_mail,
                                       float* out_mem, int32_t* out_nodes, int32_t* out_num,
                                       const void* workspace, size_t ws_bytes, void* stream);

mspipe_status mspipe_gru_apply_commit(const mspipe_gru* gru, mspipe_memory* st,
                                      int64_t commit_version, int64_t num_events,
                                      const float* snap_mem, int64_t snap_step, const float* snap_h,
                                      const int32_t* nodes, const int32_t* winner,
                                      const int32_t* num_unique, const double* new_ts,
                                      const float* new_mail, float* out_mem, const void* workspace,
                                      size_t ws_bytes, void* stream) {
  return apply_commit_impl(gru, st, commit_version, num_events, snap_mem, snap_step, snap_h, nodes, winner,
                           num_unique, new_ts, new_mail, out_mem, nullptr, nullptr, workspace, ws_bytes, stream);
}

mspipe_status mspipe_gru_apply_commit_out(const mspipe_gru* gru, mspipe_memory* st, int64_t commit_version,
                                          int64_t num_events, const float* snap_mem, int64_t snap_step,
                                          const float* snap_h, const int32_t* nodes, const int32_t* winner,
                                          const int32_t* num_unique, const double* new_ts,
                                          const float* new_mail, float* out_mem, int32_t* out_nodes,
                                          int32_t* out_num, const void* workspace, size_t ws_bytes,
                                          void* stream) {
  if (!out_nodes || !out_num) return fail(MSPIPE_EINVAL, "gru_apply_commit_out: null out_nodes / out_num");
  return apply_commit_impl(gru, st, commit_version, num_events, snap_mem, snap_step, snap_h, nodes, winner,
                           num_unique, new_ts, new_mail, out_mem, out_nodes, out_num, workspace, ws_bytes, stream);
}

static mspipe_status apply_commit_impl(const mspipe_gru* gru, mspipe_memory* st, int64_t commit_version,
                                       int64_t num_events, const float* snap_mem, int64_t snap_step,
                                       const float* snap_h, const int32_t* nodes, const int32_t* winner,
                                       const int32_t* num_unique, const double* new_ts, const float* new_mail,
                                       float* out_mem, int32_t* out_nodes, int32_t* out_num,
                                       const void* workspace, size_t ws_bytes, void* stream) {
  if (!gru || !st) return fail(MSPIPE_EINVAL, "gru_apply_commit: NULL handle");
  if (gru->precision == MSPIPE_FP32_SIMT)
    return fail(MSPIPE_EUNSUPPORTED, "gru_apply_commit: only for precision MSPIPE_FP32_3XTF32");
  if (st->world != 1) return fail(MSPIPE_EUNSUPPORTED, "gru_apply_commit: world > 1");
  if (gru->d.M != st->mem_dim || gru->d.He != st->edge_dim) return fail(MSPIPE_EINVAL, "gru_apply_commit: dims");
  if (commit_version != st->committed + 1)
    return fail(MSPIPE_EORDER, "gru_apply_commit: commit_version=%lld but committed=%lld", (long long)commit_version,
                (long long)st->committed);
  if (num_events < 0 || num_events > gru->max_events || snap_step < 1)
    return fail(MSPIPE_EINVAL, "gru_apply_commit: num_events=%lld snap_step=%lld", (long long)num_events,
                (long long)snap_step);
  if (num_events > 0) {
    if (ws_bytes < mspipe_gru_workspace_size(gru, num_events) || !workspace)
      return fail(MSPIPE_EINVAL, "gru_apply_commit: workspace of %zu bytes too small", ws_bytes);
    if (!nodes || !winner || !num_unique || !new_ts || (!new_mail && gru->d.mailbox != MSPIPE_MAILBOX_DEFERRED))
      return fail(MSPIPE_EINVAL, "gru_apply_commit: null input (new_mail may be NULL only for a deferred mailbox)");
    if (!snap_mem && (snap_h || gru->d.mailbox == MSPIPE_MAILBOX_DEFERRED))
      return fail(MSPIPE_EINVAL, "gru_apply_commit: snap_mem may be NULL only with snap_h NULL and an immediate mailbox");
  }
  if (num_events == 0 && out_num) {  // an empty batch's result record: U = 0
    cudaError_t e = cudaMemsetAsync(out_num, 0, sizeof(int32_t), (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_status(e, "gru_apply_commit: out_num");
  }
  const int64_t max_n = 2 * num_events;
  // double-buffered: the GEMM kernel catches up the previous commit's rows
  // itself when mspipe_memory_prep stamped this batch's winners; otherwise a
  // separate k_catchup launch goes first
  const int64_t ring = st->db ? commit_version % (st->k + 1) : 0;
  const bool done = st->db && st->caught_up == commit_version;  // enqueued by a prep
  const bool fused_catchup = st->db && !done && num_events > 0 && catchup_mode() >= 1 &&
                             st->stamp_iter[ring] == commit_version;
  if (st->db && (num_events == 0 || (!done && !fused_catchup))) {
    cudaError_t e = db_catchup(st, commit_version, nodes, num_unique, max_n, (cudaStream_t)stream, !done);
    if (e != cudaSuccess) return cuda_status(e, "gru_apply_commit: catch-up");
  }
  if (num_events > 0) {
    const TableSet t = table_set(st, commit_version);
    GruCommit c{nodes, t.mem, t.mem_ts, t.mail, t.mail_ts, new_ts, new_mail, st->num_nodes, st->mail_stride};
    c.res_nodes = out_nodes;
    c.res_num = out_num;
    if (done || fused_catchup) {  // the kernel saves this commit's winner list
      const int p = (int)(commit_version & 1);
      c.save_nodes = st->prev_nodes + p * st->num_nodes;
      c.save_num = st->prev_num + p;
    }
    if (fused_catchup) c.cu = catchup_args(st, commit_version);
    // split commit: mem_ts / mail / mail_ts of the winners do not depend on the
    // GEMM (the staged mail row and t*), so a k_writeback on a forked branch
    // writes them while the GEMM runs; its epilogue then stores only h'
    // (different table, same rows: no overlap with the catch-up, which skips
    // this commit's winners)
    cudaStream_t s = (cudaStream_t)stream;
    const bool split = new_mail && gru->d.mailbox == MSPIPE_MAILBOX_IMMEDIATE && env_int("MSPIPE_SPLIT_COMMIT", 1);
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // MSPIPE_WB_FIRST=0: the GEMM is enqueued before the write-back branch, so its
    // one-CTA-per-SM grid is dispatched before the branch's blocks fill the SMs
    // large batches: the write-back branch first (GDELT 100.5 vs 95.7 M events/s); small:
    // the GEMM first, its 167-register CTAs leave room for the branch's blocks (wiki 36.9
    // vs 36.0 M; r02zz6).  MSPIPE_WB_FIRST=0/1 forces it.
    const bool wb_first = env_int("MSPIPE_WB_FIRST", max_n > 2048 ? 1 : 0) != 0;
    auto branch = [&]() -> cudaError_t {
      launch_writeback(nodes, num_unique, max_n, nullptr, new_ts, new_mail, 0, st->mail_stride, t.mem, t.mem_ts,
                       t.mail, t.mail_ts, st->num_nodes, side);
      return cudaEventRecord(ev_join, side);
    };
    if (split) {
      cudaError_t e = aux_stream(st, &side, &ev_fork, &ev_join, 0);
      if (e == cudaSuccess) e = cudaEventRecord(ev_fork, s);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(side, ev_fork, 0);
      if (e != cudaSuccess) return cuda_status(e, "gru_apply_commit: fork");
      if (wb_first) {
        e = branch();
        if (e != cudaSuccess) return cuda_status(e, "gru_apply_commit: writeback branch");
      }
      c.skip_meta = 1;
    }
    cudaEvent_t kev0 = g_kev[0], kev1 = g_kev[1];
    g_kev[0] = g_kev[1] = nullptr;
    if (kev0 && cudaEventRecordWithFlags(kev0, s, cudaEventRecordExternal) != cudaSuccess)
      return cuda_status(cudaGetLastError(), "gru_apply_commit: timing event");
    cudaError_t e = launch_gru_tc(gru->d, gru->wtc, (float*)workspace, nullptr, num_events, nullptr, snap_mem, nullptr,
                                  snap_step, snap_h, winner, num_unique, out_mem, nullptr, nullptr, 0,
                                  s, kGruGemm, &c);
    if (e != cudaSuccess) return cuda_status(e, "gru_apply_commit: launch");
    if (kev1 && cudaEventRecordWithFlags(kev1, s, cudaEventRecordExternal) != cudaSuccess)
      return cuda_status(cudaGetLastError(), "gru_apply_commit: timing event");
    if (split && !wb_first) {
      e = branch();
      if (e != cudaSuccess) return cuda_status(e, "gru_apply_commit: writeback branch");
    }
    if (split) {
      e = cudaStreamWaitEvent(s, ev_join, 0);
      if (e != cudaSuccess) return cuda_status(e, "gru_apply_commit: join");
    }
  }
  mspipe_status rc = after_launch("gru_apply_commit");
  if (rc == MSPIPE_OK) {
    st->committed = commit_version;  // i_upd <- i (Alg. 1 L16)
    st->prev_max[commit_version & 1] = max_n;
  }
  return rc;
}


// ---------------------------------------------------------------------------
// row E: sharded memory
// ---------------------------------------------------------------------------
int32_t mspipe_nccl_unique_id(void* out, int32_t out_bytes) {
  if (!out || out_bytes < nccl_unique_id_bytes()) return fail(MSPIPE_EINVAL, "nccl_unique_id: buffer < %d bytes", nccl_unique_id_bytes());
  return nccl_get_unique_id(out);
}

mspipe_status mspipe_memory_writeback_keyed(mspipe_memory* st, int64_t commit_version,
                                            const int32_t* nodes, const int32_t* winner,
                                            const int32_t* num_unique, int64_t max_n, int64_t key_base,
                                            const float* new_mem, const double* new_ts,
                                            const float* new_mail, void* stream) {
  if (!st) return fail(MSPIPE_EINVAL, "memory_writeback_keyed: NULL handle");
  if (st->world == 1) {
    (void)winner;
    (void)key_base;
    return mspipe_memory_writeback(st, commit_version, nodes, num_unique, max_n, new_mem, new_ts, new_mail, stream);
  }
  if (st->sh_connected != 1)
    return fail(MSPIPE_EUNSUPPORTED, "memory_writeback_keyed: %s", st->sh_connected == 2 ? "in-process rank: drive the mspipe_shard_* phases" : "not connected (mspipe_shard_connect)");
  mspipe_status rc = mspipe_shard_commit_pack(st, commit_version, nodes, winner, num_unique, max_n, key_base, new_mem,
                                              new_ts, new_mail, stream);
  if (rc == MSPIPE_OK) rc = mspipe_shard_exchange(st, MSPIPE_XCHG_COMMIT, stream);
  if (rc == MSPIPE_OK) rc = mspipe_shard_commit_merge(st, commit_version, stream);
  return rc;
}

static mspipe_status shard_ok(const mspipe_memory* st, const char* what) {
  if (!st) return fail(MSPIPE_EINVAL, "%s: NULL handle", what);
  if (st->world < 2) return fail(MSPIPE_EINVAL, "%s: handle has world == 1", what);
  if (!st->sh_connected) return fail(MSPIPE_EUNSUPPORTED, "%s: peers not connected (mspipe_shard_connect[_local])", what);
  return MSPIPE_OK;
}

mspipe_status mspipe_shard_fetch_plan(mspipe_memory* st, int64_t iteration, const int32_t* ids, int64_t n,
                                      int32_t with_mail, void* stream) {
  mspipe_status rc = shard_ok(st, "shard_fetch_plan");
  if (rc != MSPIPE_OK) return rc;
  if (iteration < 1 || n < 0 || (n > 0 && !ids)) return fail(MSPIPE_EINVAL, "shard_fetch_plan: iteration=%lld n=%lld", (long long)iteration, (long long)n);
  if (st->committed < iteration - 1 - st->k || st->committed > iteration - 1)
    return fail(MSPIPE_ESTALE, "shard_fetch_plan: iteration %lld with committed=%lld violates k=%d",
                (long long)iteration, (long long)st->committed, st->k);
  st->sh_with_mail = with_mail ? 1 : 0;
  st->sh_fetch_iter = iteration;
  shard_fetch_plan(st, ids, n, (cudaStream_t)stream);
  return after_launch("shard_fetch_plan");
}

mspipe_status mspipe_shard_fetch_serve(mspipe_memory* st, void* stream) {
  mspipe_status rc = shard_ok(st, "shard_fetch_serve");
  if (rc != MSPIPE_OK) return rc;
  shard_fetch_serve(st, st->sh_with_mail != 0, (cudaStream_t)stream);
  return after_launch("shard_fetch_serve");
}

mspipe_status mspipe_shard_fetch_finish(mspipe_memory* st, const int32_t* ids, int64_t n, float* out_mem,
                                        double* out_mem_ts, float* out_mail, double* out_mail_ts,
                                        int64_t* out_version, void* stream) {
  mspipe_status rc = shard_ok(st, "shard_fetch_finish");
  if (rc != MSPIPE_OK) return rc;
  if (n > 0 && ((out_mail != nullptr) != (st->sh_with_mail != 0) || (out_mail == nullptr) != (out_mail_ts == nullptr)))
    return fail(MSPIPE_EINVAL, "shard_fetch_finish: mail outputs must match the plan's with_mail");
  if (n > 0 && (!ids || !out_mem || !out_mem_ts)) return fail(MSPIPE_EINVAL, "shard_fetch_finish: null ids/outputs");
  if (n > 0) shard_fetch_finish(st, ids, n, out_mem, out_mem_ts, out_mail, out_mail_ts, (cudaStream_t)stream);
  if (out_version) *out_version = st->committed;
  return after_launch("shard_fetch_finish");
}

mspipe_status mspipe_shard_mitigation_candidates(mspipe_memory* st, const mspipe_mitigation* mit,
                                                const double* root_mem_ts, int64_t root_step, int32_t* out_ids,
                                                void* stream) {
  mspipe_status rc = shard_ok(st, "shard_mitigation_candidates");
  if (rc != MSPIPE_OK) return rc;
  if (!mit || !tcsr_ok(mit->g) || mit->num_events < 0 || mit->fanout < 1 || mit->fanout > 16 || root_step < 1 ||
      (mit->num_events > 0 && (!mit->src || !mit->dst || !mit->ts || !root_mem_ts || !out_ids)))
    return fail(MSPIPE_EINVAL, "shard_mitigation_candidates: bad arguments");
  if (mit->num_events == 0) return MSPIPE_OK;
  shard_mit_candidates(to_tcsr(mit->g), mit->src, mit->dst, mit->ts, mit->num_events, root_mem_ts, root_step,
                       mit->gamma, mit->fanout, out_ids, (cudaStream_t)stream);
  return after_launch("shard_mitigation_candidates");
}

mspipe_status mspipe_shard_fetch_finish_table(mspipe_memory* st, const int32_t* ids, int64_t n, float* table_mem,
                                              double* table_mem_ts, void* stream) {
  mspipe_status rc = shard_ok(st, "shard_fetch_finish_table");
  if (rc != MSPIPE_OK) return rc;
  if (n < 0 || (n > 0 && (!ids || !table_mem || !table_mem_ts)))
    return fail(MSPIPE_EINVAL, "shard_fetch_finish_table: null ids/outputs");
  if (n > 0) shard_fetch_finish_table(st, ids, n, table_mem, table_mem_ts, (cudaStream_t)stream);
  return after_launch("shard_fetch_finish_table");
}

mspipe_status mspipe_shard_mitigate(mspipe_memory* st, const mspipe_mitigation* mit, const float* table_mem,
                                    const double* table_mem_ts, void* stream) {
  mspipe_status rc = shard_ok(st, "shard_mitigate");
  if (rc != MSPIPE_OK) return rc;
  if (!mit || !tcsr_ok(mit->g) || mit->num_events < 0 || !(mit->lambda >= 0.f && mit->lambda <= 1.f) ||
      mit->n_sim < 0 || mit->n_sim > 16 || mit->fanout < 1 || mit->fanout > 16 ||
      (mit->num_events > 0 && (!mit->src || !mit->dst || !mit->ts || !mit->out_h || !table_mem || !table_mem_ts)))
    return fail(MSPIPE_EINVAL, "shard_mitigate: bad arguments");
  if (mit->num_events == 0) return MSPIPE_OK;
  launch_mitigate(to_tcsr(mit->g), mit->src, mit->dst, mit->ts, mit->num_events, table_mem, table_mem_ts,
                  st->mem_dim, mit->lambda, mit->gamma, mit->n_sim, mit->fanout, mit->out_h, mit->out_omega,
                  mit->out_elig, (cudaStream_t)stream);
  return after_launch("shard_mitigate");
}

mspipe_status mspipe_shard_commit_pack(mspipe_memory* st, int64_t commit_version, const int32_t* nodes,
                                       const int32_t* winner, const int32_t* num_unique, int64_t max_n,
                                       int64_t key_base, const float* new_mem, const double* new_ts,
                                       const float* new_mail, void* stream) {
  mspipe_status rc = shard_ok(st, "shard_commit_pack");
  if (rc != MSPIPE_OK) return rc;
  if (commit_version != st->committed + 1)
    return fail(MSPIPE_EORDER, "shard_commit_pack: commit_version=%lld but committed=%lld", (long long)commit_version, (long long)st->committed);
  if (max_n < 0 || max_n > st->num_nodes || key_base < 0)
    return fail(MSPIPE_EINVAL, "shard_commit_pack: max_n=%lld key_base=%lld", (long long)max_n, (long long)key_base);
  if (max_n > 0 && (!nodes || !winner || !num_unique || !new_mem || !new_ts || !new_mail))
    return fail(MSPIPE_EINVAL, "shard_commit_pack: null input");
  shard_commit_pack(st, commit_version, nodes, winner, num_unique, max_n, key_base, new_mem, new_ts, new_mail,
                    (cudaStream_t)stream);
  return after_launch("shard_commit_pack");
}

mspipe_status mspipe_shard_commit_merge(mspipe_memory* st, int64_t commit_version, void* stream) {
  mspipe_status rc = shard_ok(st, "shard_commit_merge");
  if (rc != MSPIPE_OK) return rc;
  if (commit_version != st->committed + 1)
    return fail(MSPIPE_EORDER, "shard_commit_merge: commit_version=%lld but committed=%lld", (long long)commit_version, (long long)st->committed);
  shard_commit_merge(st, commit_version, (cudaStream_t)stream);
  rc = after_launch("shard_commit_merge");
  if (rc == MSPIPE_OK) st->committed = commit_version;
  return rc;
}

// The NCCL communicators connect their peers now (one eager barrier each): a
// lazy connection setup inside a CUDA-graph capture would allocate and break it.
static mspipe_status nccl_warmup(mspipe_memory* st) {
  cudaStream_t s = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (e != cudaSuccess) return cuda_status(e, "memory_create: NCCL warm-up stream");
  mspipe_status rc = nccl_barrier(st, false, s);
  if (rc == MSPIPE_OK) rc = nccl_barrier(st, true, s);
  e = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (rc == MSPIPE_OK && e != cudaSuccess) rc = cuda_status(e, "memory_create: NCCL warm-up");
  return rc;
}

mspipe_status mspipe_shard_window_handle(const mspipe_memory* st, void* out, int32_t out_bytes) {
  if (!st || st->world < 2 || !out || out_bytes < (int32_t)sizeof(cudaIpcMemHandle_t))
    return fail(MSPIPE_EINVAL, "shard_window_handle: needs a world > 1 handle and a %d-byte buffer",
                (int)sizeof(cudaIpcMemHandle_t));
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, st->sh_window);
  if (e != cudaSuccess) return cuda_status(e, "shard_window_handle");
  memcpy(out, &h, sizeof(h));
  return MSPIPE_OK;
}

static mspipe_status upload_peers(mspipe_memory* st) {
  cudaError_t e = cudaMemcpy(st->sh_peers, st->sh_peer_host, sizeof(uint8_t*) * (size_t)st->world,
                             cudaMemcpyHostToDevice);
  return cuda_status(e, "shard_connect: peer table");
}

mspipe_status mspipe_shard_connect(mspipe_memory* st, const void* handles, int32_t handle_bytes) {
  if (!st || st->world < 2 || !handles || handle_bytes != (int32_t)sizeof(cudaIpcMemHandle_t))
    return fail(MSPIPE_EINVAL, "shard_connect: needs a world > 1 handle and world x %d handle bytes",
                (int)sizeof(cudaIpcMemHandle_t));
  if (!st->nccl_comm) return fail(MSPIPE_EUNSUPPORTED, "shard_connect: no NCCL communicator (create with an id)");
  if (st->sh_connected) return fail(MSPIPE_EINVAL, "shard_connect: already connected");
  for (int32_t p = 0; p < st->world; ++p) {
    if (p == st->rank) {
      st->sh_peer_host[p] = st->sh_window;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, (const char*)handles + (size_t)p * sizeof(h), sizeof(h));
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_status(e, "shard_connect: cudaIpcOpenMemHandle");
    st->sh_peer_host[p] = ptr;
    st->sh_peer_ipc[p] = 1;
  }
  mspipe_status rc = upload_peers(st);
  if (rc == MSPIPE_OK) st->sh_connected = 1;
  return rc;
}

mspipe_status mspipe_shard_connect_local(mspipe_memory* const* ranks, int32_t world) {
  if (!ranks || world < 2 || world > 64) return fail(MSPIPE_EINVAL, "shard_connect_local: world=%d", world);
  for (int32_t r = 0; r < world; ++r)
    if (!ranks[r] || ranks[r]->world != world || ranks[r]->rank != r || ranks[r]->sh_connected ||
        ranks[r]->num_nodes != ranks[0]->num_nodes || ranks[r]->device != ranks[0]->device)
      return fail(MSPIPE_EINVAL, "shard_connect_local: ranks[%d] is not an unconnected rank %d of a world of %d",
                  r, r, world);
  for (int32_t r = 0; r < world; ++r) {
    for (int32_t p = 0; p < world; ++p) ranks[r]->sh_peer_host[p] = ranks[p]->sh_window;
    mspipe_status rc = upload_peers(ranks[r]);
    if (rc != MSPIPE_OK) return rc;
    ranks[r]->sh_connected = 2;
  }
  return MSPIPE_OK;
}

mspipe_status mspipe_shard_sent_bytes(const mspipe_memory* st, int64_t* out) {
  if (!st || st->world < 2 || !out) return fail(MSPIPE_EINVAL, "shard_sent_bytes: needs a world > 1 handle");
  unsigned long long h[3];
  cudaError_t e = cudaMemcpy(h, st->sh_sent, sizeof(h), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_status(e, "shard_sent_bytes");
  for (int i = 0; i < 3; ++i) out[i] = (int64_t)h[i];
  return MSPIPE_OK;
}

mspipe_status mspipe_shard_exchange(mspipe_memory* st, int32_t kind, void* stream) {
  mspipe_status rc = shard_ok(st, "shard_exchange");
  if (rc != MSPIPE_OK) return rc;
  if (kind < 0 || kind > 2) return fail(MSPIPE_EINVAL, "shard_exchange: kind %d", kind);
  if (st->sh_connected == 2) return MSPIPE_OK;  // in-process ranks: the stream orders the phases
  return nccl_barrier(st, kind != MSPIPE_XCHG_COMMIT, (cudaStream_t)stream);
}

mspipe_status mspipe_shard_loopback(mspipe_memory* const* ranks, int32_t world, int32_t kind, void* stream) {
  (void)stream;
  if (!ranks || world < 2 || kind < 0 || kind > 2) return fail(MSPIPE_EINVAL, "shard_loopback: world=%d kind=%d", world, kind);
  for (int32_t r = 0; r < world; ++r)
    if (!ranks[r] || ranks[r]->world != world || ranks[r]->rank != r || ranks[r]->sh_connected != 2)
      return fail(MSPIPE_EINVAL, "shard_loopback: ranks[%d] is not an in-process rank %d of a world of %d", r, r, world);
  return MSPIPE_OK;  // the data is already in the windows: one stream orders the phases of all ranks
}

mspipe_status mspipe_util_kernel_events(void* begin, void* end) {
  if ((begin == nullptr) != (end == nullptr)) return fail(MSPIPE_EINVAL, "util_kernel_events: both or neither");
  g_kev[0] = (cudaEvent_t)begin;
  g_kev[1] = (cudaEvent_t)end;
  return MSPIPE_OK;
}

mspipe_status mspipe_util_event_record(void* event, void* stream) {
  if (!event) return fail(MSPIPE_EINVAL, "util_event_record: NULL event");
  return cuda_status(cudaEventRecordWithFlags((cudaEvent_t)event, (cudaStream_t)stream, cudaEventRecordExternal),
                     "util_event_record");
}

mspipe_status mspipe_feature_fetch(const int32_t* sub_ids, const int32_t* sampled_eids, int64_t num_roots,
                                   int32_t fanout, const float* node_feat, int64_t num_nodes, int32_t node_stride,
                                   const float* edge_feat, int64_t num_edges, int32_t edge_stride,
                                   float* out_node_feat, float* out_edge_feat, void* stream) {
  if (num_roots < 0 || fanout < 1 || (node_feat && (node_stride < 1 || !out_node_feat || num_nodes < 1)) ||
      (edge_feat && (edge_stride < 1 || !out_edge_feat || num_edges < 1)))
    return fail(MSPIPE_EINVAL, "feature_fetch: num_roots=%lld fanout=%d node_stride=%d edge_stride=%d",
                (long long)num_roots, fanout, node_stride, edge_stride);
  if (num_roots > 0 && ((node_feat && !sub_ids) || (edge_feat && !sampled_eids)))
    return fail(MSPIPE_EINVAL, "feature_fetch: null sub_ids / sampled_eids");
  if ((node_feat && ((uintptr_t)node_feat | (uintptr_t)out_node_feat) % 16 && node_stride % 4 == 0) ||
      (edge_feat && ((uintptr_t)edge_feat | (uintptr_t)out_edge_feat) % 16 && edge_stride % 4 == 0))
    return fail(MSPIPE_EINVAL, "feature_fetch: tables with a stride that is a multiple of 4 must be 16-byte aligned");
  cudaError_t e = launch_feature_fetch(sub_ids, sampled_eids, num_roots, fanout, node_feat, num_nodes, node_stride,
                                       edge_feat, num_edges, edge_stride, out_node_feat, out_edge_feat,
                                       (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_status(e, "feature_fetch: launch");
  return after_launch("feature_fetch");
}

mspipe_status mspipe_stale_histogram(const mspipe_tcsr* g, const int32_t* src, const int32_t* dst,
                                     int64_t num_events, int64_t batch, int32_t max_d, int64_t* out_hist,
                                     void* stream) {
  if (!tcsr_ok(g) || num_events < 0 || batch < 1 || max_d < 1 || max_d > 4096 || !out_hist ||
      (num_events > 0 && (!src || !dst)))
    return fail(MSPIPE_EINVAL, "stale_histogram: num_events=%lld batch=%lld max_d=%d (1..4096)", (long long)num_events,
                (long long)batch, max_d);
  cudaError_t e = launch_stale_hist(to_tcsr(g), src, dst, num_events, batch, max_d, (unsigned long long*)out_hist,
                                    (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_status(e, "stale_histogram: launch");
  return after_launch("stale_histogram");
}

mspipe_status mspipe_staleness_error(const int32_t* winner, const int32_t* num_unique, int64_t num_events,
                                     const float* rows_a, int64_t stride_a, const float* rows_b, int64_t stride_b,
                                     int32_t mem_dim, double* out, void* stream) {
  if (num_events < 0 || stride_a < 1 || stride_b < 1 || mem_dim < 1)
    return fail(MSPIPE_EINVAL, "staleness_error: num_events=%lld strides %lld/%lld mem_dim=%d",
                (long long)num_events, (long long)stride_a, (long long)stride_b, mem_dim);
  if (!winner || !num_unique || !rows_a || !rows_b || !out) return fail(MSPIPE_EINVAL, "staleness_error: null pointer");
  cudaError_t e = launch_staleness_error(winner, num_unique, num_events, rows_a, stride_a, rows_b, stride_b, mem_dim,
                                         out, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_status(e, "staleness_error: launch");
  return after_launch("staleness_error");
}

mspipe_status mspipe_util_record_to_device(void* dst, const void* host_src, int64_t bytes, void* stream) {
  if (!dst || !host_src || bytes < 0) return fail(MSPIPE_EINVAL, "util_record_to_device: NULL or bytes=%lld", (long long)bytes);
  if (bytes == 0) return MSPIPE_OK;
  return cuda_status(cudaMemcpyAsync(dst, host_src, (size_t)bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream),
                     "util_record_to_device");
}

mspipe_status mspipe_util_rows_to_host(const int32_t* num, int32_t* host_num, const void* a, void* host_a,
                                       int64_t a_row_bytes, const void* b, void* host_b, int64_t b_row_bytes,
                                       int64_t max_rows, void* stream) {
  if (!num || !host_num || max_rows < 0 || a_row_bytes < 0 || b_row_bytes < 0 || a_row_bytes % 4 ||
      b_row_bytes % 4 || (a_row_bytes && (!a || !host_a)) || (b_row_bytes && (!b || !host_b)) ||
      ((uintptr_t)a | (uintptr_t)host_a | (uintptr_t)b | (uintptr_t)host_b) % 16)
    return fail(MSPIPE_EINVAL, "util_rows_to_host: row bytes must be multiples of 4, pointers 16-byte aligned");
  launch_rows_to_host(num, host_num, a, host_a, a_row_bytes, b, host_b, b_row_bytes, max_rows, (cudaStream_t)stream);
  return after_launch("util_rows_to_host");
}

mspipe_status mspipe_util_graph_begin(void* stream) {
  return cuda_status(cudaStreamBeginCapture((cudaStream_t)stream, cudaStreamCaptureModeThreadLocal),
                     "util_graph_begin");
}

mspipe_status mspipe_util_graph_end(void* stream, void** out_exec) {
  if (!out_exec) return fail(MSPIPE_EINVAL, "util_graph_end: out_exec is NULL");
  *out_exec = nullptr;
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture((cudaStream_t)stream, &g);
  if (e != cudaSuccess) {
    if (g) cudaGraphDestroy(g);
    return cuda_status(e, "util_graph_end: end capture");
  }
  cudaGraphExec_t x = nullptr;
  // MSPIPE_GRAPH_PRIO=1: kernel nodes keep the priority of the stream they were
  // captured on (the prep's side stream vs the commit's), an A/B knob
  e = cudaGraphInstantiate(&x, g, env_int("MSPIPE_GRAPH_PRIO", 0) ? cudaGraphInstantiateFlagUseNodePriority : 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_status(e, "util_graph_end: instantiate");
  *out_exec = (void*)x;
  return MSPIPE_OK;
}

mspipe_status mspipe_util_graph_launch(void* exec, void* stream) {
  if (!exec) return fail(MSPIPE_EINVAL, "util_graph_launch: NULL exec");
  return cuda_status(cudaGraphLaunch((cudaGraphExec_t)exec, (cudaStream_t)stream), "util_graph_launch");
}

mspipe_status mspipe_util_graph_destroy(void* exec) {
  if (!exec) return MSPIPE_OK;
  return cuda_status(cudaGraphExecDestroy((cudaGraphExec_t)exec), "util_graph_destroy");
}

}  // extern "C"
