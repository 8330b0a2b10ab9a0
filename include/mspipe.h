/*
 * mspipe.h — C ABI of the B200 (sm_100a) node-memory stage of MSPipe
 * (arXiv 2402.15113).  Implemented by paper_2402_15113_b200/libmspipe.so.
 *
 * "P:Lnnn" cites /root/reference/PAPER.md line nnn, "S:Lnnn" SPEC.md, "Gnn"
 * a reading of the paper listed in DESIGN.md §3.
 *
 * The per-batch stage (one "iteration" i, 1-based) is, in stream order:
 *   mspipe_sample_batch / mspipe_sample_recent   A1  recent-𝒩 sampler
 *   mspipe_memory_dedup                          A2  most-recent-message winners
 *   mspipe_memory_fetch                          A3  snapshot fetch (+A4 mitigation)
 *   mspipe_memory_update                         A5+A6 message, time encoding, GRU
 *   mspipe_memory_writeback                      A7  last-writer-wins commit
 *
 * Conventions (all entry points):
 *  - Array pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors) on
 *    the current CUDA device unless marked [host].  The caller owns every
 *    array; the library never frees caller memory.
 *  - Every compute call is asynchronous on `stream` (a cudaStream_t passed as
 *    void*; NULL = legacy default stream) and never synchronises the host.
 *    Only *_create / *_destroy allocate or free (their own handle state).
 *  - Host-checkable precondition failures return a negative status at once
 *    and set mspipe_last_error().  Errors found on the device (an id outside
 *    [0, num_nodes), ...) set a sticky device flag reported by
 *    mspipe_check().  Nothing throws or aborts across the ABI.
 *  - Node ids and event ids are int32; timestamps are float64 ("ticks");
 *    memory and mail values are float32.  Row-major layouts throughout.
 *  - Determinism: every output is a pure function of the inputs and of the
 *    stream order of the calls (no dependence on atomic arrival order).
 *  - One host thread per handle at a time.
 */
#ifndef MSPIPE_H_
#define MSPIPE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSPIPE_ABI_VERSION 2

#if defined(__GNUC__)
#define MSPIPE_API __attribute__((visibility("default")))
#else
#define MSPIPE_API
#endif

typedef int32_t mspipe_status;
enum {
  MSPIPE_OK = 0,
  MSPIPE_EINVAL = -1,      /* null pointer, negative size, bad dims / fanout / lambda */
  MSPIPE_ERANGE = -2,      /* an id outside [0, num_nodes) (device-detected; via mspipe_check) */
  MSPIPE_ESTALE = -3,      /* fetch would violate i-1-k <= committed <= i-1 */
  MSPIPE_EORDER = -4,      /* commit_version != committed + 1 */
  MSPIPE_EUNSUPPORTED = -5,/* valid request this build does not implement (reported, never faked) */
  MSPIPE_ECUDA = -6,       /* a CUDA runtime error; text in mspipe_last_error() */
  MSPIPE_ENCCL = -7        /* an NCCL error (world > 1) */
};

/* Device-flag bits reported by mspipe_check (OR-ed). */
enum { MSPIPE_DEVERR_RANGE = 1, MSPIPE_DEVERR_CAPACITY = 2 };

MSPIPE_API int32_t mspipe_abi_version(void);                  /* [host] == MSPIPE_ABI_VERSION */
MSPIPE_API const char* mspipe_last_error(void);               /* [host] thread-local text of the last non-OK status */
/* Synchronises `stream`, then returns MSPIPE_ERANGE if any kernel of this
 * library raised the device flag since the last check (clearing it), else OK
 * (or ECUDA on a pending CUDA error). */
MSPIPE_API mspipe_status mspipe_check(void* stream);

/* ---------------------------------------------------------------------------
 * Temporal CSR ("T-CSR"): per node, its incident events in stream order, so
 * ts is non-decreasing inside a row and ties keep eid order.  A self-loop
 * contributes one entry.  Read-only, caller-owned, device memory.
 *   indptr [num_nodes+1] int64, nbr/eid [nnz] int32 (other endpoint, event id),
 *   ts [nnz] float64.
 * ------------------------------------------------------------------------- */
typedef struct {
  int64_t num_nodes, nnz;
  const int64_t* indptr;
  const int32_t* nbr;
  const int32_t* eid;
  const double* ts;
} mspipe_tcsr;

/* A1 — recent-𝒩 temporal neighbour sampler.  "We sampled the 10 most recent
 * 1-hop neighbors", run on the GPU per local batch;
 * S:L98-L106.  For root r with query time t_q it returns the
 * min(fanout, #incident events with ts < t_q) most recent events, newest
 * first (G15: strict <, ties by larger eid first).
 *   roots [num_roots] int32, query_ts [num_roots] float64.
 *   out_nbr/out_eid [num_roots, fanout] int32 (-1 pad), out_ts [.., fanout]
 *   float64 (0 pad), out_dt [.., fanout] float32 = (float)(t_q - ts) (0 pad),
 *   out_cnt [num_roots] int32.  out_sub_ids (nullable) [num_roots, fanout+1]
 *   int32: the subgraph node list, column 0 = the root, then the neighbours
 *   (-1 pad) — the MFG layout of 3B(𝒩+1) nodes per batch.
 * Roots outside [0, num_nodes) yield an empty row and raise MSPIPE_DEVERR_RANGE. */
MSPIPE_API mspipe_status mspipe_sample_recent(const mspipe_tcsr* g, const int32_t* roots,
                                   const double* query_ts, int64_t num_roots, int32_t fanout,
                                   int32_t* out_nbr, int32_t* out_eid, double* out_ts,
                                   float* out_dt, int32_t* out_cnt, int32_t* out_sub_ids,
                                   void* stream);

/* A1 in batch form: the 3B roots of one batch are [src_0..src_{B-1},
 * dst_0.., neg_0..] ("three nodes per sample ... source, destination and
 * neg_sample"), each queried at its event's time ts_a.  Same outputs
 * as mspipe_sample_recent with num_roots = 3 * num_events. */
MSPIPE_API mspipe_status mspipe_sample_batch(const mspipe_tcsr* g, const int32_t* src, const int32_t* dst,
                                  const int32_t* neg, const double* ts, int64_t num_events,
                                  int32_t fanout, int32_t* out_nbr, int32_t* out_eid,
                                  double* out_ts, float* out_dt, int32_t* out_cnt,
                                  int32_t* out_sub_ids, void* stream);

/* ---------------------------------------------------------------------------
 * Node-memory state.  Tables are caller-owned device arrays:
 *   mem [num_nodes, mem_dim] f32, mem_ts [num_nodes] f64,
 *   mail [num_nodes, mail_stride] f32 (the first Dm = 2*mem_dim + edge_dim
 *   columns are used, padding columns are copied verbatim), mail_ts [num_nodes] f64.
 * mem_dim % 4 == 0 and mail_stride % 4 == 0 (16-byte row vectors).
 * staleness_k is the build staleness k (= paper k - 1, G8): a fetch for
 * iteration i is legal iff  i-1-k <= committed <= i-1  (Eq. 2, P:L196-L204;
 * Alg. 1 gate "while i - i_upd > k_i: wait").
 * world > 1: see "Row E" below (the tables are this rank's shard).
 * create allocates O(num_nodes) scratch (and, for world > 1, the fixed-capacity
 * exchange buffers and the NCCL communicator) on the current device; destroy
 * frees them.
 * ------------------------------------------------------------------------- */
typedef struct mspipe_memory mspipe_memory;

MSPIPE_API mspipe_status mspipe_memory_create(mspipe_memory** out, int64_t num_nodes, int32_t mem_dim,
                                   int32_t edge_dim, int32_t staleness_k, float* mem,
                                   double* mem_ts, float* mail, double* mail_ts,
                                   int64_t mail_stride, int32_t rank, int32_t world,
                                   const void* nccl_unique_id /* [host] 128 B, NULL iff world==1 */);
MSPIPE_API mspipe_status mspipe_memory_destroy(mspipe_memory* st);
MSPIPE_API int64_t mspipe_memory_committed(const mspipe_memory* st); /* [host] last enqueued commit version */
/* [host] restart an epoch: committed := 0; zero_tables != 0 re-zeroes this
 * rank's tables (S_0 = 0, G17; else the caller has written the initial state);
 * when double-buffered, set 0 is then mirrored into set 1.  Every device write
 * is enqueued on `stream` (so it is ordered after the caller's earlier work on
 * that stream) and the call returns after `stream` has drained.  Errors:
 * EINVAL (NULL handle), ECUDA. */
MSPIPE_API mspipe_status mspipe_memory_reset(mspipe_memory* st, int32_t zero_tables, void* stream);

/* Double-buffered state (world == 1).  With staleness k >= 1 the fetch of
 * batch t+k reads version t-1 while commit t writes version t (Eq. 2,
 * P:L196-L204); with one table set the commit must wait for that fetch.  With
 * two sets, version c lives in set c & 1 (set 0 = the tables given to
 * mspipe_memory_create, set 1 = the tables given here, same shapes, caller-
 * owned, device); commit c first copies the rows of commit c-1 from set
 * (c-1)&1 into set c&1, then writes its own rows there.  A fetch or prep reads
 * the set of version `committed` at the time it is enqueued, so the fetch of
 * version c-1 and commit c touch different tables and may run concurrently.
 * Caller's obligation (stream order): a fetch/prep enqueued while committed = c
 * completes before commit c+2 is enqueued (one commit per pipeline step and a
 * join per step satisfy it).  Call once, with committed == 0 (else
 * MSPIPE_EORDER); set 0 is mirrored into set 1 (synchronously).  world > 1:
 * MSPIPE_EUNSUPPORTED.  Extra device memory besides set 1: (k+3)·N·4 + 8 bytes
 * (previous-commit winner lists, and the winner stamps mspipe_memory_prep
 * writes so that mspipe_gru_apply_commit can do the catch-up inside its GEMM
 * kernel instead of a separate launch). */
MSPIPE_API mspipe_status mspipe_memory_double_buffer(mspipe_memory* st, float* mem1, double* mem_ts1,
                                          float* mail1, double* mail_ts1);
/* [host] bookkeeping after replaying captured work (CUDA graphs): the
 * handle's `committed` counter advances when a commit is ENQUEUED, so a
 * capture leaves it at the last captured version and mspipe_memory_reset
 * rewinds it; after replaying the captured commits up to `version` from a
 * reset, call this so that the counter (and, double-buffered, the table set
 * holding the state) match the device again.  No device work. */
MSPIPE_API mspipe_status mspipe_memory_set_committed(mspipe_memory* st, int64_t version);
/* [host] the tables holding `version` (version == committed, or committed - 1
 * when double-buffered; else MSPIPE_EINVAL).  Any output pointer may be NULL. */
MSPIPE_API mspipe_status mspipe_memory_tables(const mspipe_memory* st, int64_t version, float** mem,
                                   double** mem_ts, float** mail, double** mail_ts);

/* A4 — similarity-based staleness mitigation (MSPipe-S), applied "in the
 * memory fetching stage".  Targets are the 2B update endpoints
 * of the batch in root layout [src_0..src_{B-1}, dst_0..dst_{B-1}], target a
 * queried at t* = ts[a mod B].  For target w (snapshot state S):
 *   eligible iff t* - S.mem_ts[w] > gamma (G11);
 *   N1 = distinct ids of sample(w, t*) minus w; every distinct u of
 *   sample(x, t*) minus w, x in N1, scores c(u) += 1 ("count their common
 *   neighbors", G9); active iff S.mem_ts[u] > S.mem_ts[w] and
 *   t* - S.mem_ts[u] < gamma; Omega = first n_sim active u by
 *   (c desc, S.mem_ts[u] desc, u asc) (G10);
 *   out_h[w] = lambda*S.mem[w] + (1-lambda)*mean_{u in Omega} S.mem[u], or
 *   S.mem[w] when not eligible or Omega is empty.
 * out_h [2B, mem_dim] f32 (the GRU hidden input, G13); out_omega nullable
 * [2B, n_sim] int32 (-1 pad); out_elig nullable [2B] uint8.
 * 1 <= fanout <= 32, 0 <= n_sim <= 16, lambda in [0, 1]. */
typedef struct {
  float lambda;
  double gamma;
  int32_t n_sim;
  int32_t fanout;
  const mspipe_tcsr* g;
  const int32_t* src;
  const int32_t* dst;
  const double* ts;
  int64_t num_events;
  float* out_h;
  int32_t* out_omega;
  uint8_t* out_elig;
} mspipe_mitigation;

/* A3 — fetch under the staleness bound.  Copies rows of the state as of the
 * stream point of the call (which, by the ordering contract above, is the
 * state after commits 1..committed) for `ids` into dense outputs:
 *   out_mem [n, mem_dim], out_mem_ts [n]; out_mail [n, mail_stride] and
 *   out_mail_ts [n] are optional (NULL = not fetched).  id -1 gives a zero
 *   row and ts 0 (padding of the sampler's subgraph list).
 * Then runs the optional mitigation on the same state.  *out_version [host]
 * receives v(i) = committed.  Returns MSPIPE_ESTALE (and enqueues nothing) if
 * the staleness gate fails. */
MSPIPE_API mspipe_status mspipe_memory_fetch(mspipe_memory* st, int64_t iteration, const int32_t* ids,
                                  int64_t n, float* out_mem, double* out_mem_ts, float* out_mail,
                                  double* out_mail_ts, const mspipe_mitigation* mit,
                                  int64_t* out_version, void* stream);

/* GRU memory updater parameters, torch.nn.GRUCell layout, gates (r, z, n)
 * (G5): w_ih [3M, Dx], w_hh [3M, M], b_ih [3M], b_hh [3M], time encoder
 * enc_q = cos(fmaf(time_w[q], dt, time_b[q])) (G2), q < time_dim.
 * Dx = 2M + edge_dim + time_dim.  create packs the weights once into the
 * kernel layout and allocates the operand workspace for batches of up to
 * max_events events (device memory owned by the handle).
 * precision: MSPIPE_FP32_3XTF32 = tcgen05 tensor cores, fp32 parity via the
 * 3xTF32 split (default); MSPIPE_FP32_SIMT = CUDA-core fp32 (baseline);
 * MSPIPE_BF16 = tcgen05 kind::f16 with bf16 operands (message and weights
 * rounded to bf16, fp32 accumulation and state; the north star's bf16
 * tolerance 2e-2).  The tensor-core precisions share every entry point. */
enum { MSPIPE_FP32_SIMT = 0, MSPIPE_FP32_3XTF32 = 1, MSPIPE_BF16 = 2 };
typedef struct mspipe_gru mspipe_gru;
MSPIPE_API mspipe_status mspipe_gru_create(mspipe_gru** out, int32_t mem_dim, int32_t edge_dim,
                                int32_t time_dim, int32_t precision, int64_t max_events,
                                const float* w_ih, const float* w_hh, const float* b_ih,
                                const float* b_hh, const float* time_w, const float* time_b,
                                void* stream);
MSPIPE_API mspipe_status mspipe_gru_destroy(mspipe_gru* p);

/* Row F3 — memory-updater variants the paper trains (TGN, JODIE,
 * APAN "modified from TGL"; readings F3-1..F3-3 in DESIGN.md).
 *   cell MSPIPE_CELL_GRU: as mspipe_gru_create (TGN, APAN);
 *   cell MSPIPE_CELL_RNN: torch.nn.RNNCell (tanh), h' = tanh(W_ih x + b_ih +
 *     W_hh h + b_hh), w_ih [M, Dx], w_hh [M, M], b_ih [M], b_hh [M] (JODIE's
 *     updater);
 *   mailbox MSPIPE_MAILBOX_IMMEDIATE: the message is built from the current
 *     event (G14; all the entry points above);
 *   mailbox MSPIPE_MAILBOX_DEFERRED (TGL's TGN): the update consumes the
 *     node's STORED mail, x = [S.mail[w] (Dm) | cos(w dt + p)], dt = t* -
 *     S.mem_ts[w]; the new mail [h'_w | h'_o | e] is built from the updated
 *     memories after the commit.  Path: mspipe_memory_prep (fetching mail
 *     rows) -> mspipe_message_build_deferred -> mspipe_gru_apply_commit with
 *     new_mail = NULL -> mspipe_memory_mail_deferred.
 * Variants need precision MSPIPE_FP32_3XTF32 (else MSPIPE_EUNSUPPORTED);
 * mspipe_memory_update / mspipe_message_build refuse a deferred handle. */
enum { MSPIPE_CELL_GRU = 0, MSPIPE_CELL_RNN = 1 };
enum { MSPIPE_MAILBOX_IMMEDIATE = 0, MSPIPE_MAILBOX_DEFERRED = 1 };
MSPIPE_API mspipe_status mspipe_updater_create(mspipe_gru** out, int32_t mem_dim, int32_t edge_dim,
                                    int32_t time_dim, int32_t precision, int32_t cell,
                                    int32_t mailbox, int64_t max_events, const float* w_ih,
                                    const float* w_hh, const float* b_ih, const float* b_hh,
                                    const float* time_w, const float* time_b, void* stream);
/* A5 of a deferred-mailbox handle: the GEMM operand images of the U winners
 * from the snapshot rows the prep fetched (snap_mem / snap_mem_ts / snap_mail
 * [.., mail_stride], row of winner pair p = root row (p odd ? B + p/2 : p/2)
 * times snap_step), out_ts [<=2B] = the winners' event times. */
MSPIPE_API mspipe_status mspipe_message_build_deferred(const mspipe_gru* gru, const double* ts,
                                            int64_t num_events, const float* snap_mem,
                                            const double* snap_mem_ts, const float* snap_mail,
                                            int64_t mail_stride, int64_t snap_step,
                                            const int32_t* winner, const int32_t* num_unique,
                                            double* out_ts, void* workspace, size_t ws_bytes,
                                            void* stream);
/* After commit `commit_version` (== committed, else MSPIPE_EORDER) of a
 * deferred-mailbox batch: mail[w] = [mem[w] | mem[o] | e_ev], mail_ts[w] =
 * t_ev for every winner w (event ev, other endpoint o) — reading the memories
 * that commit wrote.  Stream-ordered after the commit and before the next
 * fetch of that version. */
MSPIPE_API mspipe_status mspipe_memory_mail_deferred(mspipe_memory* st, int64_t commit_version,
                                          const int32_t* src, const int32_t* dst, const double* ts,
                                          const float* edge_feat, int64_t num_events,
                                          const int32_t* nodes, const int32_t* winner,
                                          const int32_t* num_unique, void* stream);

/* A2 — pair expansion and most-recent-message aggregation of one batch.
 *   Event a gives p = 2a (node src_a, other dst_a) and p = 2a+1 (node dst_a,
 *   other src_a); win(w) = max{p : node_p = w} (the message "generated by the
 *   graph event related to v", last event wins; G6);
 *   negatives are never written (G7).  U winners in win order:
 *   out_nodes [<=2B] int32, out_winner [<=2B] int32 (pair index),
 *   *out_num_unique (device int32) = U.  Integer only, bit-exact,
 *   independent of the memory state, so it may run ahead with the sampler.
 *   num_events <= 16384. */
MSPIPE_API mspipe_status mspipe_memory_dedup(mspipe_memory* st, const int32_t* src, const int32_t* dst,
                                  int64_t num_events, int32_t* out_nodes, int32_t* out_winner,
                                  int32_t* out_num_unique, void* stream);

/* A5 + A6 — message build and GRU update of the U winners of one batch of
 * num_events events (winner / num_unique from mspipe_memory_dedup; global
 * eids are the caller's business; edge_feat holds this batch's rows
 * [num_events, edge_dim]).
 *   Snapshot rows in root layout: row r in [0, 2B) is [src_0..src_{B-1},
 *   dst_0..dst_{B-1}][r] and lives at snap_mem + r*snap_step*mem_dim,
 *   snap_mem_ts + r*snap_step (snap_step = fanout+1 when the rows come from a
 *   subgraph fetch of mspipe_sample_*'s out_sub_ids, 1 for a dense fetch).
 *   snap_h (nullable) [2B, mem_dim]: mitigated hidden input per row.
 *   For winner w with pair p (event a, other o, t* = ts_a):
 *     dt = (float)(t* - S.mem_ts[w]) (Δt, G4);
 *     x = [S.mem[w] ‖ S.mem[o] ‖ edge_feat[a] ‖ cos(fmaf(ω, dt, φ))] (G1-G3);
 *     h' = GRUCell(x, h) with h = snap_h or S.mem[w].
 *   out_mem [<=2B, mem_dim] = h', out_ts [<=2B] = t*, out_mail
 *   [<=2B, mail_stride] = x[0:Dm] (G14), all in winner order. */
MSPIPE_API mspipe_status mspipe_memory_update(mspipe_memory* st, const mspipe_gru* gru, const int32_t* src,
                                   const int32_t* dst, const double* ts, int64_t num_events,
                                   const float* edge_feat, const float* snap_mem,
                                   const double* snap_mem_ts, int64_t snap_step,
                                   const float* snap_h, const int32_t* winner,
                                   const int32_t* num_unique, float* out_mem, double* out_ts,
                                   float* out_mail, void* stream);

/* A7 — last-writer-wins write-back, committing version `commit_version`
 * (must equal committed + 1, else MSPIPE_EORDER): for u < *num_unique,
 *   mem[nodes[u]] = new_mem[u], mem_ts[nodes[u]] = new_ts[u],
 *   mail[nodes[u]] = new_mail[u] (mail_stride row), mail_ts[nodes[u]] = new_ts[u]
 * ("written back to the node memory storage"; i_upd <- i,
 * P:L855).  nodes must be unique (as produced by mspipe_memory_update);
 * max_n bounds *num_unique (grid sizing). */
MSPIPE_API mspipe_status mspipe_memory_writeback(mspipe_memory* st, int64_t commit_version,
                                      const int32_t* nodes, const int32_t* num_unique,
                                      int64_t max_n, const float* new_mem, const double* new_ts,
                                      const float* new_mail, void* stream);

/* ---------------------------------------------------------------------------
 * Fused forms of the same steps (same results, fewer launches).
 * ------------------------------------------------------------------------- */

/* A1 + A2 + A3 (+ A4) of batch `iteration` in one launch (plus one for the
 * mitigation when `mit` is given): exactly mspipe_sample_batch, then
 * mspipe_memory_dedup, then mspipe_memory_fetch(ids = out_sub_ids,
 * n = 3B(𝒩+1)) with the same arguments and outputs as those calls.  The same
 * staleness gate applies.  fanout <= 31; num_events <= 8192.
 * out_nodes, out_winner and out_num_unique all NULL: no dedup (A1 + A3 only;
 * the winners then come from mspipe_memory_dedup). */
MSPIPE_API mspipe_status mspipe_memory_prep(mspipe_memory* st, const mspipe_tcsr* g, int64_t iteration,
                                 const int32_t* src, const int32_t* dst, const int32_t* neg,
                                 const double* ts, int64_t num_events, int32_t fanout,
                                 int32_t* out_nbr, int32_t* out_eid, double* out_ts, float* out_dt,
                                 int32_t* out_cnt, int32_t* out_sub_ids, int32_t* out_nodes,
                                 int32_t* out_winner, int32_t* out_num_unique, float* out_mem,
                                 double* out_mem_ts, float* out_mail, double* out_mail_ts,
                                 const mspipe_mitigation* mit, int64_t* out_version, void* stream);

/* mspipe_memory_update split in its two halves (precision MSPIPE_FP32_3XTF32
 * only), so the message build of a later batch can run ahead of the GRU of the
 * current one.  `workspace` (device, caller-owned, >= mspipe_gru_workspace_size
 * bytes) carries the tensor-core A-operand images from the build to the apply
 * of the SAME batch.
 *   mspipe_message_build (A5): out_ts [<=2B], out_mail [<=2B, mail_stride]
 *     exactly as mspipe_memory_update;
 *   mspipe_gru_apply (A6): out_mem [<=2B, mem_dim] exactly as
 *     mspipe_memory_update. */
MSPIPE_API size_t mspipe_gru_workspace_size(const mspipe_gru* gru, int64_t num_events);
MSPIPE_API mspipe_status mspipe_message_build(const mspipe_gru* gru, const double* ts, int64_t num_events,
                                   const float* edge_feat, const float* snap_mem,
                                   const double* snap_mem_ts, int64_t snap_step,
                                   const float* snap_h, const int32_t* winner,
                                   const int32_t* num_unique, double* out_ts, float* out_mail,
                                   int64_t mail_stride, void* workspace, size_t ws_bytes, void* stream);
MSPIPE_API mspipe_status mspipe_gru_apply(const mspipe_gru* gru, int64_t num_events, const float* snap_mem,
                               int64_t snap_step, const float* snap_h, const int32_t* winner,
                               const int32_t* num_unique, float* out_mem, const void* workspace,
                               size_t ws_bytes, void* stream);

/* A6 + A7 in one launch: mspipe_gru_apply, then mspipe_memory_writeback of
 * (nodes, num_unique, h', new_ts, new_mail) as version commit_version, the
 * write-back done by the GEMM epilogue (world == 1).  new_ts / new_mail are
 * message_build's out_ts / out_mail; out_mem (nullable) still receives h' in
 * winner order.  snap_mem may be NULL (immediate mailbox, snap_h NULL): the
 * GRU's hidden input h = S.mem[w] is then read from new_mail[u][0:mem_dim]
 * (the mail row starts with S.mem[w], G14).  Same ordering contract as mspipe_memory_writeback (the
 * caller orders it after the fetch of iteration commit_version + k). */
MSPIPE_API mspipe_status mspipe_gru_apply_commit(const mspipe_gru* gru, mspipe_memory* st,
                                      int64_t commit_version, int64_t num_events,
                                      const float* snap_mem, int64_t snap_step, const float* snap_h,
                                      const int32_t* nodes, const int32_t* winner,
                                      const int32_t* num_unique, const double* new_ts,
                                      const float* new_mail, float* out_mem, const void* workspace,
                                      size_t ws_bytes, void* stream);

/* mspipe_gru_apply_commit that also fills a result record for a host read-back:
 * out_nodes [<=2B] = the U winner node ids (nodes[0..U)) and *out_num = U,
 * written by the GEMM kernel itself (no extra copy after the commit).  Both
 * device pointers, required (MSPIPE_EINVAL if NULL); an empty batch writes
 * *out_num = 0.  Otherwise exactly mspipe_gru_apply_commit. */
MSPIPE_API mspipe_status mspipe_gru_apply_commit_out(const mspipe_gru* gru, mspipe_memory* st,
                                          int64_t commit_version, int64_t num_events,
                                          const float* snap_mem, int64_t snap_step, const float* snap_h,
                                          const int32_t* nodes, const int32_t* winner,
                                          const int32_t* num_unique, const double* new_ts,
                                          const float* new_mail, float* out_mem, int32_t* out_nodes,
                                          int32_t* out_num, const void* workspace, size_t ws_bytes,
                                          void* stream);

/* ---------------------------------------------------------------------------
 * Row E: node memory sharded by node id (world > 1).  owner(v) = v mod world,
 * local row = v / world: the tables passed to mspipe_memory_create hold this
 * rank's rows only (ceil((num_nodes - rank) / world) rows).  Every rank runs
 * the same iterations on its own local batch of each global batch;
 * the T-CSR is replicated (sampling and dedup stay local).
 *
 * Transport: every rank owns a receive window; the sending phase stores its
 * data straight into the peer's window (NVLink peer memory), only the real
 * entries (request ids, reply rows, commit records) plus per-sender counts,
 * and a barrier separates it from the phase that reads the window.  Windows
 * are double-buffered by iteration parity.  Bytes stored per kind are
 * counted on the device (mspipe_shard_sent_bytes).
 *
 * With an nccl_unique_id at create, the ranks are processes (one per GPU):
 * after create, every rank exports its window (mspipe_shard_window_handle,
 * a 64-byte CUDA IPC handle), the handles are all-gathered (e.g. through
 * torch.distributed) and every rank calls mspipe_shard_connect with all of
 * them.  mspipe_memory_fetch and mspipe_memory_writeback_keyed are then
 * collective (every rank calls them with the same iteration / version, in
 * the same stream order); their barriers are one-int NCCL all-reduces on
 * `stream`, fetches and commits on two communicators (so a fetch on one
 * stream and a commit on another never order each other).  Without an id
 * (NULL) the handles are in-process ranks on one device, connected by
 * mspipe_shard_connect_local: the caller drives the phases below for all
 * ranks on one stream (the stream orders them; mspipe_shard_exchange and
 * mspipe_shard_loopback are then no-ops), e.g. G virtual ranks on one GPU for
 * testing.  The phases fail with MSPIPE_EUNSUPPORTED before a connect.
 *
 * MSPipe-S with world > 1 (A4): the 2-hop
 * candidates' mem_ts and the Ω rows belong to other ranks.  After the
 * subgraph fetch of iteration i (which brought each target's own row and
 * mem_ts as its root row), mspipe_shard_mitigation_candidates lists, for
 * every target t, w and, if t is eligible (Δ = t* − S.mem_ts[w] > γ, G11),
 * the ids of sample(x, t*) \ {w} for x in sample(w, t*) \ {w} into out_ids
 * [2B, 1 + fanout²] (pads −1; the T-CSR is replicated); a second fetch of
 * that list (plan -> exchange -> serve -> exchange ->
 * mspipe_shard_fetch_finish_table) writes those rows into a node-indexed
 * table [num_nodes, mem_dim] / [num_nodes] of version v(i); mspipe_shard_mitigate
 * then computes eligibility, Ω and the blend exactly as the single-GPU fetch
 * does (same outputs as mspipe_mitigation), reading only table rows the list
 * requested.  memory_fetch with mitigation at world > 1: MSPIPE_EUNSUPPORTED
 * (use these phases).
 *
 * Phases of a fetch: plan (stores the request ids into the owners' windows)
 * -> exchange(FETCH_IDS) -> serve (owner stores the reply rows into the
 * requesters' windows) -> exchange(FETCH_ROWS) -> finish.  Phases of a
 * commit: pack (stores the records into the owners' windows) ->
 * exchange(COMMIT) -> merge.  The LWW key of a record is key_base + winner
 * pair index, key_base = 2 x (global index of this rank's first event in the
 * iteration), i.e. the global pair index of the single-GPU batch G·B; the
 * owner keeps, per node, the record with the largest key (64-bit atomicMax,
 * then a keyed copy), so the result does not depend on arrival order.
 * ------------------------------------------------------------------------- */
enum { MSPIPE_XCHG_FETCH_IDS = 0, MSPIPE_XCHG_FETCH_ROWS = 1, MSPIPE_XCHG_COMMIT = 2 };

MSPIPE_API int64_t mspipe_memory_local_rows(const mspipe_memory* st); /* [host] rows of this rank's tables */
/* [host] rank 0 creates the NCCL unique id (128 bytes) and broadcasts it
 * (e.g. through torch.distributed) before every rank's mspipe_memory_create. */
MSPIPE_API int32_t mspipe_nccl_unique_id(void* out, int32_t out_bytes);
MSPIPE_API mspipe_status mspipe_memory_writeback_keyed(mspipe_memory* st, int64_t commit_version,
                                            const int32_t* nodes, const int32_t* winner,
                                            const int32_t* num_unique, int64_t max_n, int64_t key_base,
                                            const float* new_mem, const double* new_ts,
                                            const float* new_mail, void* stream);
MSPIPE_API mspipe_status mspipe_shard_fetch_plan(mspipe_memory* st, int64_t iteration, const int32_t* ids,
                                      int64_t n, int32_t with_mail, void* stream);
MSPIPE_API mspipe_status mspipe_shard_fetch_serve(mspipe_memory* st, void* stream);
MSPIPE_API mspipe_status mspipe_shard_fetch_finish(mspipe_memory* st, const int32_t* ids, int64_t n,
                                        float* out_mem, double* out_mem_ts, float* out_mail,
                                        double* out_mail_ts, int64_t* out_version, void* stream);
MSPIPE_API mspipe_status mspipe_shard_mitigation_candidates(mspipe_memory* st, const mspipe_mitigation* mit,
                                                 const double* root_mem_ts, int64_t root_step,
                                                 int32_t* out_ids, void* stream);
MSPIPE_API mspipe_status mspipe_shard_fetch_finish_table(mspipe_memory* st, const int32_t* ids, int64_t n,
                                              float* table_mem, double* table_mem_ts, void* stream);
MSPIPE_API mspipe_status mspipe_shard_mitigate(mspipe_memory* st, const mspipe_mitigation* mit,
                                    const float* table_mem, const double* table_mem_ts, void* stream);
MSPIPE_API mspipe_status mspipe_shard_commit_pack(mspipe_memory* st, int64_t commit_version,
                                       const int32_t* nodes, const int32_t* winner,
                                       const int32_t* num_unique, int64_t max_n, int64_t key_base,
                                       const float* new_mem, const double* new_ts,
                                       const float* new_mail, void* stream);
MSPIPE_API mspipe_status mspipe_shard_commit_merge(mspipe_memory* st, int64_t commit_version, void* stream);
/* the barrier of a phase (NCCL all-reduce of one int; no-op for in-process ranks) */
MSPIPE_API mspipe_status mspipe_shard_exchange(mspipe_memory* st, int32_t kind, void* stream);
/* [host] this rank's receive window as a CUDA IPC handle (out >= 64 bytes) */
MSPIPE_API mspipe_status mspipe_shard_window_handle(const mspipe_memory* st, void* out, int32_t out_bytes);
/* [host] open every peer's window: handles = world x handle_bytes (64) host
 * bytes, rank order, own entry ignored.  Needs a handle created with an NCCL
 * id; once.  MSPIPE_ECUDA if a window cannot be opened (no peer access). */
MSPIPE_API mspipe_status mspipe_shard_connect(mspipe_memory* st, const void* handles, int32_t handle_bytes);
/* [host] connect `world` in-process ranks (same device, created without an id) */
MSPIPE_API mspipe_status mspipe_shard_connect_local(mspipe_memory* const* ranks, int32_t world);
/* [host] bytes this rank has stored into windows since create / the last
 * reset: out[0] fetch request ids (+ counts), out[1] reply rows, out[2] commit
 * records (+ counts).  Synchronises the device. */
MSPIPE_API mspipe_status mspipe_shard_sent_bytes(const mspipe_memory* st, int64_t* out);
MSPIPE_API mspipe_status mspipe_shard_loopback(mspipe_memory* const* ranks, int32_t world, int32_t kind,
                                    void* stream);

/* ------------------------------------------------------------------------
 * F2 — feature fetch ("Fetch feature", stage 2 of the pipeline, P:L189,
 * P:L176-L180) for the sampled subgraphs.  Device pointers.
 *   sub_ids      [R, fanout+1] subgraph node ids (mspipe_sample_* out_sub_ids;
 *                -1 = pad), read when node_feat != NULL;
 *   sampled_eids [R, fanout] eids of the sampled links (out_eid; -1 = pad),
 *                read when edge_feat != NULL;
 *   node_feat    [num_nodes, node_stride] (NULL: no node features; GDELT
 *                |d_v| = 413, Table `tab:datasets` P:L395), edge_feat
 *                [num_edges, edge_stride] (NULL: none), f32 row-major;
 *   out_node_feat[r, s, :] = node_feat[sub_ids[r, s], :] (zeros for pads),
 *   out_edge_feat[r, s, :] = edge_feat[sampled_eids[r, s], :] (zeros for pads).
 * Strides are in floats; a stride that is a multiple of 4 needs 16-byte
 * aligned tables (vector copies).  Ids >= num_nodes / num_edges give zero
 * rows and raise MSPIPE_DEVERR_RANGE.  Errors: MSPIPE_EINVAL. */
MSPIPE_API mspipe_status mspipe_feature_fetch(const int32_t* sub_ids, const int32_t* sampled_eids,
                                   int64_t num_roots, int32_t fanout, const float* node_feat,
                                   int64_t num_nodes, int32_t node_stride, const float* edge_feat,
                                   int64_t num_edges, int32_t edge_stride, float* out_node_feat,
                                   float* out_edge_feat, void* stream);

/* ------------------------------------------------------------------------
 * F1 — minimal-staleness planner (MSPipe §3.2; Alg. 1)
 * ------------------------------------------------------------------------
 * Host functions (no GPU work).  Stages j = 1..5 of an iteration: sample,
 * fetch feature, fetch memory, train, update memory; tau[j-1] = profiled
 * duration of stage j (any time unit, >= 0).  Iterations i = 1..num_iters.
 * Paper staleness k_i >= 1 (k = 1: no staleness): iteration i fetches
 * memory updated through iteration i - k_i.
 *
 * mspipe_plan_timeline: Eq. 3-4.  out_b / out_e [num_iters][5]
 *   (row i-1, column j-1) = b_i^(j), e_i^(j).  k NULL: Eq. 3 as printed; else
 *   k[i-1] = k_i >= 1 adds the Alg. 1 gate b_i^(3) >= e_{i-k_i}^(5) (C1;
 *   i - k_i < 1: no gate).  Errors: MSPIPE_EINVAL (tau < 0, k_i < 1, NULL).
 * mspipe_plan_min_staleness: the optimisation of P:L300-L307, iteration by
 *   iteration: least k_i in [1, min(i, k_max)) with e_{i-k_i}^(5) <= b_i^(4) -
 *   tau^(3), b_i^(4) from the schedule with iteration i's gate relaxed (C2);
 *   the chosen k_i is then applied as the gate (C1).  Iterations i <= k_max
 *   with no such k are warm-up: k_i = i (no gate).  Later ones with
 *   none are infeasible: k_i = k_max - 1 and *out_infeasible_iter = the first
 *   such i (0 if none; the binding constraint is C2).  out_k [num_iters].
 * mspipe_stale_histogram: the C3 statistic (Fig. `fig:overlap`) on the
 *   GPU.  For every batch i (events [(i-1)B, iB)) and every distinct src/dst
 *   node v of the batch, d = i - (batch of v's previous event), or 0 if v has
 *   none; out_hist [max_d + 2] (device, int64, overwritten) counts d = 0,
 *   1..max_d, and > max_d in its last bin.  Under staleness k the stale share
 *   is sum_{1 <= d <= k-1} hist[d] / sum hist (reading F6); k_max is chosen
 *   so that it stays <= 50 % (C3).  g must be the T-CSR of the same stream
 *   (rows in stream order).  Errors: MSPIPE_EINVAL (bad T-CSR, batch < 1,
 *   max_d outside 1..4096). */
MSPIPE_API mspipe_status mspipe_plan_timeline(const double* tau, int64_t num_iters, const int32_t* k,
                                   double* out_b, double* out_e);
MSPIPE_API mspipe_status mspipe_plan_min_staleness(const double* tau, int64_t num_iters, int32_t k_max,
                                        int32_t* out_k, int64_t* out_infeasible_iter);
MSPIPE_API mspipe_status mspipe_stale_histogram(const mspipe_tcsr* g, const int32_t* src, const int32_t* dst,
                                     int64_t num_events, int64_t batch, int32_t max_d, int64_t* out_hist,
                                     void* stream);
/* [host] stale shares from a histogram of mspipe_stale_histogram (copied to
 * the host): out[q] = sum_{1 <= d <= k_q - 1} hist[d] / sum hist for the paper
 * staleness k_q = k_values[q] >= 1 (k = 1: 0, no staleness; reading
 * F6), 0 for an empty histogram.  nbins = max_d + 2.  Errors: MSPIPE_EINVAL
 * (NULL, nbins < 2, k_q < 1). */
MSPIPE_API mspipe_status mspipe_plan_stale_fractions(const int64_t* hist, int32_t nbins, const int32_t* k_values,
                                          int32_t nk, double* out);
/* Staleness error (MSPipe §5.5, Fig. `fig:staleness_error`;
 * Theorem 1's ε_s): *out (device f64) = ‖x − s‖_F over the U = *num_unique
 * update targets of one batch of num_events events, x = rows_a (what the
 * updater consumed: the stale snapshot rows S_{v(i)} or MSPipe-S's mitigated
 * rows) and s = rows_b (the precise memory S_{i−1} of a k = 0 run of the same
 * stream, reading F7).  winner [U] are the dedup winners (pair p = 2a + role);
 * both row arrays are in root layout: the row of pair p is at
 * rows + ((p & 1)·num_events + (p >> 1))·stride·mem_dim floats (stride = 𝒩+1 for
 * a prep's subgraph rows, 1 for a [2B, M] array).  f64 accumulation in a fixed
 * order: deterministic.  Errors: MSPIPE_EINVAL (NULL, bad sizes). */
MSPIPE_API mspipe_status mspipe_staleness_error(const int32_t* winner, const int32_t* num_unique,
                                     int64_t num_events, const float* rows_a, int64_t stride_a,
                                     const float* rows_b, int64_t stride_b, int32_t mem_dim, double* out,
                                     void* stream);

/* Utility (timing): record `event` (a cudaEvent_t) on `stream` with
 * cudaEventRecordExternal, so that under stream capture it becomes an
 * event-record node of the graph and can still be used for elapsed-time
 * measurement of the captured kernels. */
MSPIPE_API mspipe_status mspipe_util_event_record(void* event, void* stream);
/* [host] timing: the next mspipe_gru_apply_commit(_out) of this thread records
 * cudaEvent_t `begin` / `end` (timing events, also as graph nodes) on its
 * stream right before and right after its GEMM kernel (not the write-back
 * branch); one-shot.  Both or neither (MSPIPE_EINVAL). */
MSPIPE_API mspipe_status mspipe_util_kernel_events(void* begin, void* end);

/* Utility (step graphs): the stage of one step is captured once and replayed
 * (the "CUDA graphs instead of a tracing compiler" of DESIGN.md §2).
 *   mspipe_util_graph_begin(stream)            starts a thread-local capture on `stream`
 *                                               (streams forked from it by event waits join it)
 *   mspipe_util_graph_end(stream, &exec)       ends it and instantiates; *exec owned by the
 *                                               caller, freed with mspipe_util_graph_destroy
 *   mspipe_util_graph_launch(exec, stream)     one replay on `stream`; no other work is added
 *                                               (no RNG-offset fills, unlike torch.cuda.CUDAGraph)
 * Errors: MSPIPE_EINVAL for NULL exec, MSPIPE_ECUDA with the runtime's message
 * (a capture that fails to end is discarded). */
MSPIPE_API mspipe_status mspipe_util_graph_begin(void* stream);
/* Utility (e2e inputs): one asynchronous host -> device copy of a batch's
 * packed input record (`bytes` from pinned host memory at host_src to the
 * device buffer dst) on `stream`; capturable (a memcpy node of the step
 * graph).  Errors: MSPIPE_EINVAL (NULL, bytes < 0), MSPIPE_ECUDA. */
MSPIPE_API mspipe_status mspipe_util_record_to_device(void* dst, const void* host_src, int64_t bytes, void* stream);
/* Utility (e2e read-back): copy the first *num (device) rows of two device
 * arrays a [.., a_row_bytes] and b [.., b_row_bytes] into host_a / host_b —
 * mapped pinned host memory (cudaHostAlloc; mapped under UVA) written by the
 * kernel over PCIe — and *num into *host_num.  Whole 16-byte words are
 * copied (up to 12 bytes past the last row; the host buffers must hold
 * max_rows rows); row bytes multiples of 4, pointers 16-byte aligned (else
 * MSPIPE_EINVAL); max_rows sizes the grid. */
MSPIPE_API mspipe_status mspipe_util_rows_to_host(const int32_t* num, int32_t* host_num, const void* a,
                                       void* host_a, int64_t a_row_bytes, const void* b, void* host_b,
                                       int64_t b_row_bytes, int64_t max_rows, void* stream);
MSPIPE_API mspipe_status mspipe_util_graph_end(void* stream, void** out_exec);
MSPIPE_API mspipe_status mspipe_util_graph_launch(void* exec, void* stream);
MSPIPE_API mspipe_status mspipe_util_graph_destroy(void* exec);

/* Row F3 — the APAN updater ("modified from TGL"; "RNN as the
 * memory update function while incorporating an attention mechanism ...
 * asynchronous propagation"; readings F3-4..F3-8 in DESIGN.md).  The GRU
 * handle is a deferred-mailbox GRUCell MSPIPE_FP32_3XTF32 one (x = [message
 * (Dm) | cos(ω Δt + ϕ)], so the weights have the TGN shapes).
 *   Mailbox tables (caller-owned device memory, zeroed by the caller for an
 *   epoch start): mb [num_nodes, slots, Dm] f32, mb_ts [num_nodes, slots]
 *   f64, mb_pos / mb_cnt [num_nodes] int32 (next ring slot, filled slots).
 *   w_q [M, M], w_k [M, Dm] (host or device f32; copied at create).
 * mspipe_message_build_apan (A5 of APAN, after mspipe_memory_prep of the
 *   batch): for winner w, q = W_q S.mem[w], k_s = W_k mb[w, s] over its
 *   filled slots, α = softmax(q·k / √M), x = [Σ α mb[w, s] ‖ cos(ω Δt + ϕ)],
 *   Δt = t* - S.mem_ts[w], h = S.mem[w] (snap rows in root layout, as
 *   mspipe_message_build_deferred), into the GEMM operand `workspace`;
 *   out_ts [<=2B] = t*.  The mailbox is read from the tables: the caller
 *   orders the call after the previous delivery (k = 0 in the stage).
 * Then mspipe_gru_apply_commit(new_mail = NULL) commits h' and mem_ts.
 * mspipe_apan_deliver (after that commit, version commit_version): mail of
 *   winner w = [mem[w] | mem[o] | e_ev] from the committed tables, time
 *   t_ev, delivered to w and to the sampled neighbours of w's root row (nbr
 *   / cnt: the prep's sampler outputs [3B, fanout], [3B]); per node the mail
 *   with the largest key p (fanout + 1) + s wins (s = 0: itself, 1 + j:
 *   neighbour j) and fills the node's next ring slot.  world == 1 only. */
/* mspipe_apan_refresh_keys: the handle caches k = W_k mail for every ring
 *   slot (written with the mail at delivery); after the caller writes the
 *   mailbox tables directly (anything but an all-zero reset), it recomputes
 *   the cache from them. */
typedef struct mspipe_apan mspipe_apan;
MSPIPE_API mspipe_status mspipe_apan_create(mspipe_apan** out, int64_t num_nodes, int32_t mem_dim, int32_t edge_dim,
                                            int32_t slots, int64_t max_events, const float* w_q, const float* w_k,
                                            float* mb, double* mb_ts, int32_t* mb_pos, int32_t* mb_cnt, void* stream);
MSPIPE_API mspipe_status mspipe_apan_destroy(mspipe_apan* a);
MSPIPE_API mspipe_status mspipe_apan_refresh_keys(mspipe_apan* a, void* stream);
MSPIPE_API mspipe_status mspipe_message_build_apan(mspipe_apan* a, const mspipe_gru* gru, const double* ts,
                                                   int64_t num_events, const float* snap_mem,
                                                   const double* snap_mem_ts, int64_t snap_step,
                                                   const int32_t* nodes, const int32_t* winner,
                                                   const int32_t* num_unique, double* out_ts, void* workspace,
                                                   size_t ws_bytes, void* stream);
MSPIPE_API mspipe_status mspipe_apan_deliver(mspipe_apan* a, mspipe_memory* st, int64_t commit_version,
                                             const int32_t* src, const int32_t* dst, const double* ts,
                                             const float* edge_feat, int64_t num_events, const int32_t* nodes,
                                             const int32_t* winner, const int32_t* num_unique, const int32_t* nbr,
                                             const int32_t* cnt, int32_t fanout, void* stream);

/* ------------------------------------------------------------------------
 * F4 — the MTGNN training stage of one iteration ("the memory updater
 * computes the updated memory, the MTGNN layer computes the embeddings, and
 * the loss and backward steps are performed (including all-reduce)", P:L763;
 * Eq. 2: h^(i)_v = emb(s~^(i)_v, s~^(i)_u | u ∈ N(v)), "emb (e.g.,
 * a single layer GAT)").  Readings T1-T7 in DESIGN.md §3:
 *   s~(v) = h'_v (this batch's GRU output) if v is a winner, else the
 *   fetched snapshot row (T1); q = W_q s~(r), k_u / v_u = W_k / W_v [s~(u) ‖
 *   φ(Δt_u)], α = softmax(q·k_u/√H) over the cnt valid neighbours, h_r = W_o
 *   [Σ α_u v_u ‖ s~(r)] + b_o (T3); logit(a, b) = w_2·tanh(W_1 [h_a ‖ h_b] +
 *   b_1) + b_2 (T4); loss = mean BCE over (src_j, dst_j) = 1 and (src_j,
 *   neg_j) = 0 (T5); gradients of every learnable tensor, through h' into the
 *   GRU weights (T2); SGD (T6).  The DP all-reduce of `grads` (T7) is the
 *   caller's (one flat buffer: one collective).
 *
 * mspipe_train_layout: the flat parameter layout, returns the float count;
 *   offsets[13] (nullable) of [w_q (H,M), w_k (H,M+Dt), w_v (H,M+Dt),
 *   w_o (H,H+M), b_o (H), w_1 (H,2H), b_1 (H), w_2 (H), b_2 (1), w_ih (3M,Dx),
 *   w_hh (3M,M), b_ih (3M), b_hh (3M)], row-major, each 16-byte aligned.
 * mspipe_train_create: params / grads are caller-owned device buffers of
 *   that many floats (params initialised by the caller; the GRU section is
 *   the master copy: the updater's tensor-core images are repacked from it at
 *   create and after every SGD step).  gru: a GRUCell, immediate-mailbox,
 *   MSPIPE_FP32_3XTF32 handle (else MSPIPE_EUNSUPPORTED).  Allocates the
 *   step's workspace for max_events events (<= the gru's max_events) and a
 *   cuBLAS handle; fanout <= 31.
 * mspipe_gru_save_gates: the GEMM epilogue of `gru` also stores every
 *   winner's gate pre-activations [r | z | n_x | n_h] (biases included) into
 *   gates [<=2B, 4M] (device; NULL stops it).  Needed by mspipe_train_step.
 * mspipe_train_step: batch i after its prep and commit — sub_ids [3B, F+1],
 *   sub_dt [3B, F], sub_cnt [3B] (the sampler outputs of the 3B roots),
 *   snap_mem [3B(F+1), M] (the fetched subgraph rows), nodes / num_unique
 *   (winners), new_mem [<=2B, M] (h' in winner order), workspace (the batch's
 *   GEMM operand images), gates (saved by its GEMM).  Writes *out_loss
 *   (device f64), out_logits (nullable, [2B]: positives then negatives) and
 *   the full gradient into grads (overwritten).  Deterministic.  An empty
 *   batch (num_events == 0) enqueues nothing.  Errors: MSPIPE_EINVAL.
 * mspipe_train_sgd: params -= lr * grads, then repacks the GRU images. */
typedef struct mspipe_train mspipe_train;
MSPIPE_API int64_t mspipe_train_layout(int32_t mem_dim, int32_t edge_dim, int32_t time_dim, int32_t emb_dim,
                                       int64_t* offsets);
MSPIPE_API mspipe_status mspipe_train_create(mspipe_train** out, const mspipe_gru* gru, int64_t num_nodes,
                                             int32_t emb_dim, int32_t fanout, int64_t max_events, float* params,
                                             float* grads, void* stream);
MSPIPE_API mspipe_status mspipe_train_destroy(mspipe_train* t);
MSPIPE_API mspipe_status mspipe_gru_save_gates(mspipe_gru* gru, float* gates);
MSPIPE_API mspipe_status mspipe_train_step(mspipe_train* t, const mspipe_gru* gru, int64_t num_events,
                                           const int32_t* sub_ids, const float* sub_dt, const int32_t* sub_cnt,
                                           const float* snap_mem, const int32_t* nodes, const int32_t* num_unique,
                                           const float* new_mem, const void* workspace, size_t ws_bytes,
                                           const float* gates, double* out_loss, float* out_logits, void* stream);
MSPIPE_API mspipe_status mspipe_train_sgd(mspipe_train* t, mspipe_gru* gru, float lr, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MSPIPE_H_ */
