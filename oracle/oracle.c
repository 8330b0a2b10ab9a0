/*
 * oracle.c — plain CPU oracle of MSPipe's node-memory stage.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant generator with the CUDA path
 * (paper_2402_15113_b200/), and neither side includes or links the other.
 *
 * Paper: MSPipe (arXiv 2402.15113), /root/reference/PAPER.md.  "P:Lnnn" is a
 * PAPER.md line; "S:Lnnn" a SPEC.md line; "Gnn" a reading listed in DESIGN.md.
 *
 * Numerics: f32 inputs/state, f64 accumulation, one rounding to f32 per
 * stored value.  Build with -O2 -fno-fast-math -ffp-contract=off; OpenMP only
 * over independent rows inside one batch (batches stay sequential).
 *
 * Parity pins (tests/test_oracle_*.py): brute-force sampler definition,
 * hand-worked example, bias-only closed form, torch.nn.GRUCell (f64),
 * time-block closed form, mitigation identities and exhaustive ranking,
 * |mem| <= 1, k = 0 == sequential loop, nearest-rank quantile == numpy
 * 'inverted_cdf'.  Nothing here is "parity unpinned" except long free-running
 * float trajectories.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_EINVAL (-1)
#define ORC_ENOMEM (-2)

void orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int orc_get_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------------
 * A1 — recent-𝒩 temporal neighbour sampler.
 * "We sampled the 10 most recent 1-hop neighbors".
 * Reading G15: strict ts < t_q, newest first, ties by larger eid first
 * (stream order), a self-loop contributes one entry whose neighbour is the
 * node itself.  Output per entry: (other endpoint, eid, ts, dt=f32(t_q-ts)).
 * ---------------------------------------------------------------------- */

/* Definition, written out: scan the whole event log backwards. O(E) per root. */
int orc_sample_brute(int64_t E, const int32_t* src, const int32_t* dst, const double* ts,
                     int64_t nroots, const int32_t* roots, const double* qts, int32_t fanout,
                     int32_t* out_nbr, int32_t* out_eid, double* out_ts, float* out_dt,
                     int32_t* out_cnt) {
  if (fanout < 1 || E < 0 || nroots < 0) return ORC_EINVAL;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t r = 0; r < nroots; ++r) {
    int32_t v = roots[r];
    double tq = qts[r];
    int32_t cnt = 0;
    for (int64_t j = E - 1; j >= 0 && cnt < fanout; --j) {
      if (!(ts[j] < tq)) continue;
      if (src[j] != v && dst[j] != v) continue;
      int32_t other = (src[j] == v) ? dst[j] : src[j];
      out_nbr[r * fanout + cnt] = other;
      out_eid[r * fanout + cnt] = (int32_t)j;
      out_ts[r * fanout + cnt] = ts[j];
      out_dt[r * fanout + cnt] = (float)(tq - ts[j]);
      ++cnt;
    }
    out_cnt[r] = cnt;
    for (int32_t c = cnt; c < fanout; ++c) {
      out_nbr[r * fanout + c] = -1;
      out_eid[r * fanout + c] = -1;
      out_ts[r * fanout + c] = 0.0;
      out_dt[r * fanout + c] = 0.0f;
    }
  }
  return ORC_OK;
}

/* Per-node incident-event lists in stream order (the oracle's own adjacency;
 * built here by counting, independent of the CUDA path's T-CSR). */
typedef struct {
  int64_t num_nodes, num_events;
  int64_t* ptr;      /* [N+1] */
  int32_t* eid;      /* [nnz] incident events, ascending eid */
  const int32_t* src;
  const int32_t* dst;
  const double* ts;
} orc_graph;

orc_graph* orc_graph_create(int64_t N, int64_t E, const int32_t* src, const int32_t* dst,
                            const double* ts) {
  orc_graph* g = (orc_graph*)calloc(1, sizeof(orc_graph));
  if (!g) return NULL;
  g->num_nodes = N;
  g->num_events = E;
  g->src = src;
  g->dst = dst;
  g->ts = ts;
  g->ptr = (int64_t*)calloc((size_t)N + 1, sizeof(int64_t));
  for (int64_t j = 0; j < E; ++j) {
    g->ptr[src[j] + 1] += 1;
    if (dst[j] != src[j]) g->ptr[dst[j] + 1] += 1; /* self-loop once */
  }
  for (int64_t v = 0; v < N; ++v) g->ptr[v + 1] += g->ptr[v];
  g->eid = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->ptr[N] > 0 ? g->ptr[N] : 1));
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N > 0 ? N : 1));
  for (int64_t v = 0; v < N; ++v) fill[v] = g->ptr[v];
  for (int64_t j = 0; j < E; ++j) {
    g->eid[fill[src[j]]++] = (int32_t)j;
    if (dst[j] != src[j]) g->eid[fill[dst[j]]++] = (int32_t)j;
  }
  free(fill);
  return g;
}

void orc_graph_free(orc_graph* g) {
  if (!g) return;
  free(g->ptr);
  free(g->eid);
  free(g);
}

/* Number of incident events of v with ts < tq: plain lower-bound bisection on
 * the (non-decreasing) ts of v's list. */
static int64_t orc_count_before(const orc_graph* g, int32_t v, double tq) {
  int64_t lo = g->ptr[v], hi = g->ptr[v + 1];
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (g->ts[g->eid[mid]] < tq) lo = mid + 1;
    else hi = mid;
  }
  return lo; /* absolute index: entries [ptr[v], lo) have ts < tq */
}

/* Same result as orc_sample_brute (pinned by tests), O(log deg + 𝒩) per root. */
int orc_sample(const orc_graph* g, int64_t nroots, const int32_t* roots, const double* qts,
               int32_t fanout, int32_t* out_nbr, int32_t* out_eid, double* out_ts,
               float* out_dt, int32_t* out_cnt) {
  if (fanout < 1 || nroots < 0) return ORC_EINVAL;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < nroots; ++r) {
    int32_t v = roots[r];
    double tq = qts[r];
    int32_t cnt = 0;
    if (v >= 0 && v < g->num_nodes) {
      int64_t end = orc_count_before(g, v, tq);
      for (int64_t q = end - 1; q >= g->ptr[v] && cnt < fanout; --q) {
        int32_t j = g->eid[q];
        out_nbr[r * fanout + cnt] = (g->src[j] == v) ? g->dst[j] : g->src[j];
        out_eid[r * fanout + cnt] = j;
        out_ts[r * fanout + cnt] = g->ts[j];
        out_dt[r * fanout + cnt] = (float)(tq - g->ts[j]);
        ++cnt;
      }
    }
    out_cnt[r] = cnt;
    for (int32_t c = cnt; c < fanout; ++c) {
      out_nbr[r * fanout + c] = -1;
      out_eid[r * fanout + c] = -1;
      out_ts[r * fanout + c] = 0.0;
      out_dt[r * fanout + c] = 0.0f;
    }
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------
 * A2 — pair expansion + most-recent-message aggregation.
 * Event a of the batch yields pairs p=2a (node=src, other=dst) and p=2a+1
 * (node=dst, other=src); "m_v generated by the graph event related to v"
 * (P:L153); last event wins; src and dst both updated
 * (S:L364); negatives are never written (G7).  win(w) = max{p : node_p = w};
 * U is listed by win ascending (G6).  Returns U.
 * ---------------------------------------------------------------------- */
int64_t orc_dedup(int64_t N, int64_t B, const int32_t* src, const int32_t* dst,
                  int32_t* out_nodes, int32_t* out_winner) {
  int64_t* last = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N > 0 ? N : 1));
  if (!last) return ORC_ENOMEM;
  for (int64_t v = 0; v < N; ++v) last[v] = -1;
  for (int64_t p = 0; p < 2 * B; ++p) {
    int32_t node = (p & 1) ? dst[p >> 1] : src[p >> 1];
    last[node] = p;
  }
  int64_t U = 0;
  for (int64_t p = 0; p < 2 * B; ++p) {
    int32_t node = (p & 1) ? dst[p >> 1] : src[p >> 1];
    if (last[node] == p) {
      out_nodes[U] = node;
      out_winner[U] = (int32_t)p;
      ++U;
    }
  }
  free(last);
  return U;
}

/* ------------------------------------------------------------------------
 * A4 — similarity-based staleness mitigation (MSPipe-S).
 * For target w at time t* with snapshot state (mem, mem_ts):
 *   eligible iff Δ = t* - mem_ts[w] > γ ("not been updated for time Δt,
 *   longer than a threshold γ"; G11);
 *   N1 = distinct ids of sample(w, t*) \ {w};  for x in N1, every distinct
 *   u in sample(x, t*) \ {w} gets c(u) += 1 ("count their common
 *   neighbors"; G9);
 *   active: mem_ts[u] > mem_ts[w] and t* - mem_ts[u] < γ (G11);
 *   Ω = first n_sim active u by (c desc, mem_ts[u] desc, u asc) (G10);
 *   ŝ = λ s_w + (1-λ) mean_{u∈Ω} s_u, else ŝ = s_w.
 * Computed in f64 from f32 values, rounded once (O5).
 * ---------------------------------------------------------------------- */
typedef struct {
  int32_t id;
  int32_t c;
  double mts;
} orc_cand;

static int orc_cand_cmp(const void* a, const void* b) {
  const orc_cand* x = (const orc_cand*)a;
  const orc_cand* y = (const orc_cand*)b;
  if (x->c != y->c) return x->c > y->c ? -1 : 1;
  if (x->mts != y->mts) return x->mts > y->mts ? -1 : 1;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return 0;
}

/* distinct ids of sample(v, tq) except `excl`, in newest-first order; returns count */
static int orc_distinct_recent(const orc_graph* g, int32_t v, double tq, int32_t fanout,
                               int32_t excl, int32_t* out) {
  int n = 0;
  int64_t end = orc_count_before(g, v, tq);
  int32_t taken = 0;
  for (int64_t q = end - 1; q >= g->ptr[v] && taken < fanout; --q, ++taken) {
    int32_t j = g->eid[q];
    int32_t o = (g->src[j] == v) ? g->dst[j] : g->src[j];
    if (o == excl) continue;
    int dup = 0;
    for (int i = 0; i < n; ++i) dup |= (out[i] == o);
    if (!dup) out[n++] = o;
  }
  return n;
}

/* One target.  Writes h[M] (f32) and omega[n_sim] (-1 padded); returns 1 if
 * eligible else 0. */
static int orc_mitigate_one(const orc_graph* g, int32_t w, double tstar, const float* mem,
                            const double* mem_ts, int32_t M, float lambda, double gamma,
                            int32_t n_sim, int32_t fanout, float* h, int32_t* omega) {
  for (int32_t s = 0; s < n_sim; ++s) omega[s] = -1;
  const float* sw = mem + (int64_t)w * M;
  double delta = tstar - mem_ts[w];
  if (!(delta > gamma)) {
    for (int32_t m = 0; m < M; ++m) h[m] = sw[m];
    return 0;
  }
  int32_t n1[64];
  int32_t nn1 = orc_distinct_recent(g, w, tstar, fanout, w, n1);
  orc_cand cand[4096];
  int32_t nc = 0;
  int32_t tmp[64];
  for (int32_t i = 0; i < nn1; ++i) {
    int32_t nt = orc_distinct_recent(g, n1[i], tstar, fanout, w, tmp);
    for (int32_t t = 0; t < nt; ++t) {
      int32_t u = tmp[t];
      int32_t found = -1;
      for (int32_t c = 0; c < nc; ++c)
        if (cand[c].id == u) { found = c; break; }
      if (found >= 0) cand[found].c += 1;
      else { cand[nc].id = u; cand[nc].c = 1; cand[nc].mts = mem_ts[u]; ++nc; }
    }
  }
  /* keep active candidates */
  int32_t na = 0;
  for (int32_t c = 0; c < nc; ++c) {
    double mu = mem_ts[cand[c].id];
    if (mu > mem_ts[w] && (tstar - mu) < gamma) cand[na++] = cand[c];
  }
  qsort(cand, (size_t)na, sizeof(orc_cand), orc_cand_cmp);
  int32_t k = na < n_sim ? na : n_sim;
  if (k == 0) {
    for (int32_t m = 0; m < M; ++m) h[m] = sw[m];
    return 1;
  }
  for (int32_t s = 0; s < k; ++s) omega[s] = cand[s].id;
  double lam = (double)lambda;
  for (int32_t m = 0; m < M; ++m) {
    double acc = 0.0;
    for (int32_t s = 0; s < k; ++s) acc += (double)mem[(int64_t)cand[s].id * M + m];
    double mean = acc / (double)k;
    h[m] = (float)(lam * (double)sw[m] + (1.0 - lam) * mean);
  }
  return 1;
}

int orc_mitigate(const orc_graph* g, int64_t n, const int32_t* ids, const double* tstar,
                 const float* mem, const double* mem_ts, int32_t M, float lambda, double gamma,
                 int32_t n_sim, int32_t fanout, float* out_h, int32_t* out_omega,
                 uint8_t* out_elig) {
  if (n_sim < 0 || n_sim > 64 || fanout < 1 || fanout > 64 || !(lambda >= 0.f && lambda <= 1.f))
    return ORC_EINVAL;
#pragma omp parallel for schedule(dynamic, 8)
  for (int64_t i = 0; i < n; ++i) {
    int32_t om[64];
    int e = orc_mitigate_one(g, ids[i], tstar[i], mem, mem_ts, M, lambda, gamma, n_sim, fanout,
                             out_h + i * M, om);
    if (out_omega)
      for (int32_t s = 0; s < n_sim; ++s) out_omega[i * n_sim + s] = om[s];
    if (out_elig) out_elig[i] = (uint8_t)e;
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------
 * A5 + A6 — message build, time encoding and GRU memory update for ONE
 * winner.  Eq. (1)/(2): m_v = msg(s_v, s_u, y_uv(t), Δt); s_v <- mem(s_v, m_v)
 * (P:L148-L153).  Readings: identity-concat message + GRUCell
 * (G1, G5), enc_q = cos(ω_q Δt + φ_q) with d_t = 100 (G2, G3), Δt read from
 * the snapshot's mem_ts (G4), mitigated ŝ only as the GRU hidden input (G13).
 *   x  = [s_w ‖ s_o ‖ e ‖ enc],  Dx = 2M + He + d_t
 *   r  = σ(W_ir x + b_ir + W_hr h + b_hr)
 *   z  = σ(W_iz x + b_iz + W_hz h + b_hz)
 *   n  = tanh(W_in x + b_in + r ⊙ (W_hn h + b_hn))
 *   h' = (1 - z) ⊙ n + z ⊙ h                      (torch.nn.GRUCell)
 * ---------------------------------------------------------------------- */
typedef struct {
  int32_t M, He, Dt;
  const float *w_ih, *w_hh, *b_ih, *b_hh, *time_w, *time_b;
  int32_t cell; /* 0: GRUCell (TGN, APAN); 1: RNNCell tanh (JODIE's updater, row F3) */
} orc_gru;

/* Row F3 updater variants (readings F3-1..F3-3 in DESIGN.md):
 * variant bit 0 = deferred mailbox (TGL's TGN: the update consumes the node's
 * STORED mail, and the new mail is built from post-update memories), bit 1 =
 * RNN cell  h' = tanh(W_ih x + b_ih + W_hh h + b_hh)  (torch.nn.RNNCell, tanh;
 * W_ih [M, Dx], W_hh [M, M]). */
#define ORC_VAR_DEFERRED 1
#define ORC_VAR_RNN 2

static void orc_gru_row(const orc_gru* P, const float* x /*[Dx]*/, const float* h /*[M]*/,
                        float* out /*[M]*/) {
  const int32_t M = P->M;
  const int32_t Dx = 2 * M + P->He + P->Dt;
  if (P->cell == 1) {
    for (int32_t j = 0; j < M; ++j) {
      double a = (double)P->b_ih[j] + (double)P->b_hh[j];
      for (int32_t k = 0; k < Dx; ++k) a += (double)P->w_ih[(int64_t)j * Dx + k] * (double)x[k];
      for (int32_t k = 0; k < M; ++k) a += (double)P->w_hh[(int64_t)j * M + k] * (double)h[k];
      out[j] = (float)tanh(a);
    }
    return;
  }
  for (int32_t j = 0; j < M; ++j) {
    double gi[3], gh[3];
    for (int g = 0; g < 3; ++g) {
      const float* wi = P->w_ih + (int64_t)(g * M + j) * Dx;
      const float* wh = P->w_hh + (int64_t)(g * M + j) * M;
      double a = (double)P->b_ih[g * M + j];
      for (int32_t k = 0; k < Dx; ++k) a += (double)wi[k] * (double)x[k];
      double b = (double)P->b_hh[g * M + j];
      for (int32_t k = 0; k < M; ++k) b += (double)wh[k] * (double)h[k];
      gi[g] = a;
      gh[g] = b;
    }
    double r = 1.0 / (1.0 + exp(-(gi[0] + gh[0])));
    double z = 1.0 / (1.0 + exp(-(gi[1] + gh[1])));
    double n = tanh(gi[2] + r * gh[2]);
    out[j] = (float)((1.0 - z) * n + z * (double)h[j]);
  }
}

/* Build x for winner pair p of a batch whose events start at eid0. */
static void orc_build_x(const orc_gru* P, int64_t p, const int32_t* src, const int32_t* dst,
                        const double* ts, const float* ef /* batch rows */, const float* mem,
                        const double* mem_ts, float* x) {
  const int32_t M = P->M, He = P->He;
  int64_t a = p >> 1;
  int32_t w = (p & 1) ? dst[a] : src[a];
  int32_t o = (p & 1) ? src[a] : dst[a];
  float dt = (float)(ts[a] - mem_ts[w]);
  for (int32_t m = 0; m < M; ++m) x[m] = mem[(int64_t)w * M + m];
  for (int32_t m = 0; m < M; ++m) x[M + m] = mem[(int64_t)o * M + m];
  for (int32_t c = 0; c < He; ++c) x[2 * M + c] = ef[a * He + c];
  for (int32_t q = 0; q < P->Dt; ++q)
    x[2 * M + He + q] = (float)cos((double)fmaf(P->time_w[q], dt, P->time_b[q]));
}

/* Row F3, deferred mailbox, A5: x = [S.mail[w] (Dm) | cos(omega dt + phi)],
 * dt = t* - S.mem_ts[w] as in G4 (reading F3-1). */
static void orc_build_x_deferred(const orc_gru* P, int64_t p, const int32_t* src, const int32_t* dst,
                                 const double* ts, const float* mail, const double* mem_ts, float* x) {
  const int32_t M = P->M, He = P->He, Dm = 2 * M + He;
  int64_t a = p >> 1;
  int32_t w = (p & 1) ? dst[a] : src[a];
  float dt = (float)(ts[a] - mem_ts[w]);
  for (int32_t c = 0; c < Dm; ++c) x[c] = mail[(int64_t)w * Dm + c];
  for (int32_t q = 0; q < P->Dt; ++q)
    x[Dm + q] = (float)cos((double)fmaf(P->time_w[q], dt, P->time_b[q]));
}

/* Teacher-forced memory update for one batch of B events against snapshot
 * tables (mem [N,M], mem_ts [N], mail [N, Dm] — read only in the deferred
 * variant).  If `mit_on`, the GRU hidden input of each winner is the mitigated
 * ŝ (needs g).  Outputs in winner order; returns U.  out_mail: immediate = the
 * message x[0:Dm] (G14); deferred = [h'_w | h'_o | e] from this batch's
 * updated memories of both endpoints (reading F3-2). */
int64_t orc_memory_update(int64_t N, int64_t B, const int32_t* src, const int32_t* dst,
                          const double* ts, const float* ef, int32_t M, int32_t He, int32_t Dt,
                          const float* w_ih, const float* w_hh, const float* b_ih,
                          const float* b_hh, const float* time_w, const float* time_b,
                          const float* mem, const double* mem_ts, int32_t mit_on,
                          const orc_graph* g, float lambda, double gamma, int32_t n_sim,
                          int32_t fanout, int32_t* out_nodes, int32_t* out_winner,
                          float* out_mem, double* out_ts, float* out_mail, float* out_h,
                          int32_t* out_omega, uint8_t* out_elig, const float* mail, int32_t variant) {
  orc_gru P = {M, He, Dt, w_ih, w_hh, b_ih, b_hh, time_w, time_b, (variant & ORC_VAR_RNN) ? 1 : 0};
  const int deferred = (variant & ORC_VAR_DEFERRED) != 0;
  if (deferred && !mail) return ORC_EINVAL;
  int64_t U = orc_dedup(N, B, src, dst, out_nodes, out_winner);
  if (U < 0) return U;
  const int32_t Dm = 2 * M + He, Dx = Dm + Dt;
  int rc = ORC_OK;
#pragma omp parallel for schedule(static)
  for (int64_t u = 0; u < U; ++u) {
    float* x = (float*)malloc(sizeof(float) * (size_t)Dx);
    float* h = (float*)malloc(sizeof(float) * (size_t)M);
    int32_t om[64];
    int64_t p = out_winner[u];
    int32_t w = out_nodes[u];
    double tstar = ts[p >> 1];
    if (deferred) orc_build_x_deferred(&P, p, src, dst, ts, mail, mem_ts, x);
    else orc_build_x(&P, p, src, dst, ts, ef, mem, mem_ts, x);
    int e = 0;
    if (mit_on) {
      e = orc_mitigate_one(g, w, tstar, mem, mem_ts, M, lambda, gamma, n_sim, fanout, h, om);
    } else {
      for (int32_t m = 0; m < M; ++m) h[m] = mem[(int64_t)w * M + m];
      for (int32_t s = 0; s < n_sim && s < 64; ++s) om[s] = -1;
    }
    orc_gru_row(&P, x, h, out_mem + u * M);
    out_ts[u] = tstar;
    if (out_mail && !deferred)
      for (int32_t c = 0; c < Dm; ++c) out_mail[u * Dm + c] = x[c];
    if (out_h)
      for (int32_t m = 0; m < M; ++m) out_h[u * M + m] = h[m];
    if (out_omega)
      for (int32_t s = 0; s < n_sim; ++s) out_omega[u * n_sim + s] = om[s];
    if (out_elig) out_elig[u] = (uint8_t)e;
    free(x);
    free(h);
  }
  if (deferred && out_mail) {
    /* new mail of winner w (event a, other endpoint o): [h'_w | h'_o | e_a]; o
     * is an endpoint of a batch event, so it has a winner row of its own */
    int32_t* row_of = (int32_t*)malloc(sizeof(int32_t) * (size_t)(N > 0 ? N : 1));
    for (int64_t v = 0; v < N; ++v) row_of[v] = -1;
    for (int64_t u = 0; u < U; ++u) row_of[out_nodes[u]] = (int32_t)u;
    for (int64_t u = 0; u < U; ++u) {
      int64_t p = out_winner[u], a = p >> 1;
      int32_t o = (p & 1) ? src[a] : dst[a];
      int32_t uo = row_of[o];
      for (int32_t m = 0; m < M; ++m) out_mail[u * Dm + m] = out_mem[u * M + m];
      for (int32_t m = 0; m < M; ++m) out_mail[u * Dm + M + m] = out_mem[(int64_t)uo * M + m];
      for (int32_t c = 0; c < He; ++c) out_mail[u * Dm + 2 * M + c] = ef[a * He + c];
    }
    free(row_of);
  }
  return rc == ORC_OK ? U : rc;
}

/* ------------------------------------------------------------------------
 * A3 — staleness schedule (Eq. 2; Alg. 1 gate P:L844-L847).
 * Build k = paper k - 1 (G8; "k=1 represents the baseline").
 * exact:   v(i) = max(0, i-1-k)
 * grouped: v(i) = (k+1) * floor((i-1)/(k+1))
 * Both satisfy i-1-k <= v(i) <= i-1.
 * ---------------------------------------------------------------------- */
int64_t orc_snapshot_version(int64_t i, int32_t k, int32_t schedule) {
  if (schedule == 1) return (int64_t)(k + 1) * ((i - 1) / (k + 1));
  int64_t v = i - 1 - k;
  return v > 0 ? v : 0;
}

/* ------------------------------------------------------------------------
 * Full stream (C.2 O1-O8): for i = 1..: S <- state after commits 1..v(i);
 * dedup; (mitigation); message; GRU; commit version i (A7: mem, mem_ts,
 * mail, mail_ts of each winner; "updated memory vectors ... written back",
 * P:L154).  State tables are in/out (initial state in,
 * final state out).  Keeps k+1 full state copies (one per version still
 * readable).  Returns number of batches run.
 * ---------------------------------------------------------------------- */
/* Test hook (no arithmetic): copies of the A3s output (subgraph ids and the
 * snapshot rows S_{v(i)} gathered for them) of the listed batches, so tests
 * can compare the GPU's subgraph fetch with the oracle's, batch by batch.
 * batches: ascending 1-based iterations; outputs [n, 3B(fanout+1)(, M)]. */
typedef struct {
  int64_t n;
  const int64_t* batches;
  int32_t* sub_ids;
  float* mem;
  double* mem_ts;
} orc_dump;

int64_t orc_run_stream_ex(int64_t N, int64_t E, const int32_t* src, const int32_t* dst,
                          const double* ts, const float* ef, int32_t M, int32_t He, int32_t Dt,
                          const float* w_ih, const float* w_hh, const float* b_ih,
                          const float* b_hh, const float* time_w, const float* time_b, int64_t B,
                          int32_t k, int32_t schedule, int32_t mit_on, float lambda, double gamma,
                          int32_t n_sim, int32_t fanout, float* mem, double* mem_ts, float* mail,
                          double* mail_ts, int64_t max_batches, int64_t* out_versions,
                          const int32_t* neg, int32_t subgraph, const int32_t* plan_k, int32_t variant,
                          const orc_dump* dump);

int64_t orc_run_stream(int64_t N, int64_t E, const int32_t* src, const int32_t* dst,
                       const double* ts, const float* ef, int32_t M, int32_t He, int32_t Dt,
                       const float* w_ih, const float* w_hh, const float* b_ih,
                       const float* b_hh, const float* time_w, const float* time_b, int64_t B,
                       int32_t k, int32_t schedule, int32_t mit_on, float lambda, double gamma,
                       int32_t n_sim, int32_t fanout, float* mem, double* mem_ts, float* mail,
                       double* mail_ts, int64_t max_batches, int64_t* out_versions,
                       const int32_t* neg, int32_t subgraph, const int32_t* plan_k, int32_t variant) {
  return orc_run_stream_ex(N, E, src, dst, ts, ef, M, He, Dt, w_ih, w_hh, b_ih, b_hh, time_w, time_b, B, k,
                           schedule, mit_on, lambda, gamma, n_sim, fanout, mem, mem_ts, mail, mail_ts,
                           max_batches, out_versions, neg, subgraph, plan_k, variant, NULL);
}

int64_t orc_run_stream_ex(int64_t N, int64_t E, const int32_t* src, const int32_t* dst,
                          const double* ts, const float* ef, int32_t M, int32_t He, int32_t Dt,
                          const float* w_ih, const float* w_hh, const float* b_ih,
                          const float* b_hh, const float* time_w, const float* time_b, int64_t B,
                          int32_t k, int32_t schedule, int32_t mit_on, float lambda, double gamma,
                          int32_t n_sim, int32_t fanout, float* mem, double* mem_ts, float* mail,
                          double* mail_ts, int64_t max_batches, int64_t* out_versions,
                          const int32_t* neg, int32_t subgraph, const int32_t* plan_k, int32_t variant,
                          const orc_dump* dump) {
  if (B < 1 || k < 0 || M < 1) return ORC_EINVAL;
  if (subgraph && !neg) return ORC_EINVAL;
  if (dump && dump->n > 0 && !subgraph) return ORC_EINVAL;
  int64_t d_next = 0; /* next entry of dump->batches */
  const int32_t Dm = 2 * M + He;
  int64_t nb = (E + B - 1) / B;
  if (max_batches >= 0 && max_batches < nb) nb = max_batches;
  orc_graph* g = (mit_on || subgraph) ? orc_graph_create(N, E, src, dst, ts) : NULL;
  /* optional A1 + A3s: sample the 3B roots [src, dst, neg] at their event
   * times and copy the snapshot rows of the 3B(𝒩+1) subgraph nodes (P:L818,
   * P:L1153) — not needed for the state, done so the timed CPU baseline runs
   * every step of the per-batch path. */
  int64_t R3 = 3 * B;
  int32_t* sroots = NULL; double* sq = NULL; int32_t *snbr = NULL, *seid = NULL, *scnt = NULL;
  double* sts = NULL; float* sdt = NULL; float* smem = NULL; double* smts = NULL;
  if (subgraph) {
    sroots = (int32_t*)malloc(sizeof(int32_t) * R3);
    sq = (double*)malloc(sizeof(double) * R3);
    snbr = (int32_t*)malloc(sizeof(int32_t) * R3 * fanout);
    seid = (int32_t*)malloc(sizeof(int32_t) * R3 * fanout);
    sts = (double*)malloc(sizeof(double) * R3 * fanout);
    sdt = (float*)malloc(sizeof(float) * R3 * fanout);
    scnt = (int32_t*)malloc(sizeof(int32_t) * R3);
    smem = (float*)malloc(sizeof(float) * R3 * (fanout + 1) * M);
    smts = (double*)malloc(sizeof(double) * R3 * (fanout + 1));
  }
  int32_t R = k + 1;
  int plan_bad = 0;
  size_t szm = sizeof(float) * (size_t)N * M, szt = sizeof(double) * (size_t)N;
  float** rmem = (float**)malloc(sizeof(float*) * R);
  double** rts = (double**)malloc(sizeof(double*) * R);
  for (int32_t s = 0; s < R; ++s) {
    rmem[s] = (float*)malloc(szm ? szm : 1);
    rts[s] = (double*)malloc(szt ? szt : 1);
  }
  memcpy(rmem[0], mem, szm);
  memcpy(rts[0], mem_ts, szt);
  /* deferred mailbox: the update reads the snapshot mail too, so keep its versions */
  const int deferred = (variant & ORC_VAR_DEFERRED) != 0;
  size_t sza = sizeof(float) * (size_t)N * Dm;
  float** rmail = (float**)malloc(sizeof(float*) * R);
  for (int32_t s = 0; s < R; ++s) rmail[s] = deferred ? (float*)malloc(sza ? sza : 1) : NULL;
  if (deferred) memcpy(rmail[0], mail, sza);
  int32_t* nodes = (int32_t*)malloc(sizeof(int32_t) * 2 * B);
  int32_t* winner = (int32_t*)malloc(sizeof(int32_t) * 2 * B);
  float* nmem = (float*)malloc(sizeof(float) * 2 * B * M);
  double* nts = (double*)malloc(sizeof(double) * 2 * B);
  float* nmail = (float*)malloc(sizeof(float) * 2 * B * Dm);
  for (int64_t i = 1; i <= nb; ++i) {
    /* plan (row F1): paper staleness k_i, v(i) = max(0, i - k_i) (Alg. 1 gate,
     * P:L845-L848); the ring of k+1 copies must hold it */
    int64_t v = orc_snapshot_version(i, k, schedule);
    if (plan_k) {
      v = i - plan_k[i - 1] > 0 ? i - plan_k[i - 1] : 0;
      if (plan_k[i - 1] < 1 || i - v > k + 1) {
        plan_bad = 1;
        nb = i - 1;
        break;
      }
    }
    if (out_versions) out_versions[i - 1] = v;
    int64_t j0 = (i - 1) * B;
    int64_t nb_ev = (j0 + B <= E) ? B : E - j0;
    if (subgraph) {
      const float* Sm = rmem[v % R];
      const double* St = rts[v % R];
      for (int64_t a = 0; a < nb_ev; ++a) {
        sroots[a] = src[j0 + a];
        sroots[nb_ev + a] = dst[j0 + a];
        sroots[2 * nb_ev + a] = neg[j0 + a];
        sq[a] = sq[nb_ev + a] = sq[2 * nb_ev + a] = ts[j0 + a];
      }
      orc_sample(g, 3 * nb_ev, sroots, sq, fanout, snbr, seid, sts, sdt, scnt);
#pragma omp parallel for schedule(static)
      for (int64_t r = 0; r < 3 * nb_ev; ++r) {
        for (int32_t c = 0; c <= fanout; ++c) {
          int32_t id = (c == 0) ? sroots[r] : snbr[r * fanout + c - 1];
          float* dstrow = smem + (r * (fanout + 1) + c) * M;
          if (id >= 0) {
            memcpy(dstrow, Sm + (int64_t)id * M, sizeof(float) * M);
            smts[r * (fanout + 1) + c] = St[id];
          } else {
            memset(dstrow, 0, sizeof(float) * M);
            smts[r * (fanout + 1) + c] = 0.0;
          }
        }
      }
      if (dump && d_next < dump->n && dump->batches[d_next] == i) {
        const int64_t slots = R3 * (fanout + 1), used = 3 * nb_ev * (fanout + 1);
        int32_t* di = dump->sub_ids + d_next * slots;
        for (int64_t r = 0; r < 3 * nb_ev; ++r)
          for (int32_t c = 0; c <= fanout; ++c)
            di[r * (fanout + 1) + c] = (c == 0) ? sroots[r] : snbr[r * fanout + c - 1];
        memcpy(dump->mem + d_next * slots * M, smem, sizeof(float) * used * M);
        memcpy(dump->mem_ts + d_next * slots, smts, sizeof(double) * used);
        ++d_next;
      }
    }
    int64_t U = orc_memory_update(N, nb_ev, src + j0, dst + j0, ts + j0, ef + j0 * He, M, He,
                                  Dt, w_ih, w_hh, b_ih, b_hh, time_w, time_b, rmem[v % R],
                                  rts[v % R], mit_on, g, lambda, gamma, n_sim, fanout, nodes,
                                  winner, nmem, nts, nmail, NULL, NULL, NULL, rmail[v % R], variant);
    for (int64_t u = 0; u < U; ++u) {
      int32_t w = nodes[u];
      memcpy(mem + (int64_t)w * M, nmem + u * M, sizeof(float) * M);
      mem_ts[w] = nts[u];
      memcpy(mail + (int64_t)w * Dm, nmail + u * Dm, sizeof(float) * Dm);
      mail_ts[w] = nts[u];
    }
    memcpy(rmem[i % R], mem, szm);
    memcpy(rts[i % R], mem_ts, szt);
    if (deferred) memcpy(rmail[i % R], mail, sza);
  }
  for (int32_t s = 0; s < R; ++s) {
    free(rmem[s]);
    free(rts[s]);
    free(rmail[s]);
  }
  free(rmail);
  free(rmem);
  free(rts);
  free(nodes);
  free(winner);
  free(nmem);
  free(nts);
  free(nmail);
  if (subgraph) {
    free(sroots); free(sq); free(snbr); free(seid); free(sts); free(sdt); free(scnt); free(smem); free(smts);
  }
  orc_graph_free(g);
  return plan_bad ? ORC_EINVAL : nb;
}

/* ------------------------------------------------------------------------
 * Row F1 analytics: staleness error series (MSPipe §5.5, Fig.
 * `fig:staleness_error`; Theorem 1's ε_s; SPEC staleness_error).
 * Two runs of the same stream in lockstep:
 *   the stale run  (build staleness k, schedule, MSPipe-S if mit_on) and
 *   the reference  (k = 0: "a synchronous (k=0) oracle run with identical
 *                   seeds and data order").
 * For iteration i, over the update targets w of batch i (the dedup winners,
 * identical in both runs): x_w = the GRU hidden input of the stale run (the
 * stale snapshot row S̃_{v(i)}[w], or the mitigated ŝ_w) and s_w = the
 * reference's S_{i-1}[w];  out_err[i-1] = sqrt(Σ_w Σ_c (x_w,c − s_w,c)^2),
 * summed in f64 in (winner, column) order (reading F7).  Returns nb.
 * ---------------------------------------------------------------------- */
int64_t orc_staleness_error_series(int64_t N, int64_t E, const int32_t* src, const int32_t* dst,
                                   const double* ts, const float* ef, int32_t M, int32_t He, int32_t Dt,
                                   const float* w_ih, const float* w_hh, const float* b_ih,
                                   const float* b_hh, const float* time_w, const float* time_b, int64_t B,
                                   int32_t k, int32_t schedule, int32_t mit_on, float lambda, double gamma,
                                   int32_t n_sim, int32_t fanout, int64_t max_batches, double* out_err) {
  if (B < 1 || k < 0 || M < 1 || !out_err) return ORC_EINVAL;
  const int32_t Dm = 2 * M + He;
  int64_t nb = (E + B - 1) / B;
  if (max_batches >= 0 && max_batches < nb) nb = max_batches;
  orc_graph* g = mit_on ? orc_graph_create(N, E, src, dst, ts) : NULL;
  const int32_t R = k + 1;
  size_t szm = sizeof(float) * (size_t)N * M, szt = sizeof(double) * (size_t)N;
  /* stale run: the live state plus a ring of the k+1 versions still readable */
  float* mem = (float*)calloc((size_t)N * M + 1, sizeof(float));
  double* mem_ts = (double*)calloc((size_t)N + 1, sizeof(double));
  float** rmem = (float**)malloc(sizeof(float*) * R);
  double** rts = (double**)malloc(sizeof(double*) * R);
  for (int32_t r = 0; r < R; ++r) {
    rmem[r] = (float*)calloc((size_t)N * M + 1, sizeof(float));
    rts[r] = (double*)calloc((size_t)N + 1, sizeof(double));
  }
  /* reference run (k = 0): its live state is S_{i-1} at iteration i */
  float* rf_mem = (float*)calloc((size_t)N * M + 1, sizeof(float));
  double* rf_ts = (double*)calloc((size_t)N + 1, sizeof(double));
  int32_t* nodes = (int32_t*)malloc(sizeof(int32_t) * 2 * B);
  int32_t* winner = (int32_t*)malloc(sizeof(int32_t) * 2 * B);
  float* nmem = (float*)malloc(sizeof(float) * 2 * B * M);
  double* nts = (double*)malloc(sizeof(double) * 2 * B);
  float* nmail = (float*)malloc(sizeof(float) * 2 * B * Dm);
  float* nh = (float*)malloc(sizeof(float) * 2 * B * M);
  int64_t rc = nb;
  for (int64_t i = 1; i <= nb; ++i) {
    int64_t v = orc_snapshot_version(i, k, schedule);
    int64_t j0 = (i - 1) * B;
    int64_t n = (j0 + B <= E) ? B : E - j0;
    /* stale run: update from S_{v(i)}, x = its GRU hidden input */
    int64_t U = orc_memory_update(N, n, src + j0, dst + j0, ts + j0, ef + j0 * He, M, He, Dt, w_ih, w_hh,
                                  b_ih, b_hh, time_w, time_b, rmem[v % R], rts[v % R], mit_on, g, lambda,
                                  gamma, n_sim, fanout, nodes, winner, nmem, nts, nmail, nh, NULL, NULL, NULL, 0);
    if (U < 0) {
      rc = U;
      break;
    }
    double acc = 0.0;
    for (int64_t u = 0; u < U; ++u)
      for (int32_t c = 0; c < M; ++c) {
        double d = (double)nh[u * M + c] - (double)rf_mem[(int64_t)nodes[u] * M + c];
        acc += d * d;
      }
    out_err[i - 1] = sqrt(acc);
    for (int64_t u = 0; u < U; ++u) {
      memcpy(mem + (int64_t)nodes[u] * M, nmem + u * M, sizeof(float) * M);
      mem_ts[nodes[u]] = nts[u];
    }
    memcpy(rmem[i % R], mem, szm);
    memcpy(rts[i % R], mem_ts, szt);
    /* reference run: update from its own S_{i-1}, then commit */
    U = orc_memory_update(N, n, src + j0, dst + j0, ts + j0, ef + j0 * He, M, He, Dt, w_ih, w_hh, b_ih, b_hh,
                          time_w, time_b, rf_mem, rf_ts, 0, NULL, 1.0f, 0.0, n_sim, fanout, nodes, winner, nmem,
                          nts, nmail, NULL, NULL, NULL, NULL, 0);
    for (int64_t u = 0; u < U; ++u) {
      memcpy(rf_mem + (int64_t)nodes[u] * M, nmem + u * M, sizeof(float) * M);
      rf_ts[nodes[u]] = nts[u];
    }
  }
  for (int32_t r = 0; r < R; ++r) {
    free(rmem[r]);
    free(rts[r]);
  }
  free(rmem); free(rts); free(mem); free(mem_ts); free(rf_mem); free(rf_ts);
  free(nodes); free(winner); free(nmem); free(nts); free(nmail); free(nh);
  orc_graph_free(g);
  return rc;
}

/* ------------------------------------------------------------------------
 * γ helper (A-8): Δt population = for each event j and each endpoint v
 * (self-loop once), ts_j - ts of v's previous event; first appearances are
 * excluded (G16).  Quantile is nearest-rank.
 * ---------------------------------------------------------------------- */
int64_t orc_delta_t_population(int64_t N, int64_t E, const int32_t* src, const int32_t* dst,
                               const double* ts, double* out) {
  double* last = (double*)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
  uint8_t* seen = (uint8_t*)calloc((size_t)(N > 0 ? N : 1), 1);
  int64_t n = 0;
  for (int64_t j = 0; j < E; ++j) {
    int32_t e2[2] = {src[j], dst[j]};
    int ne = (src[j] == dst[j]) ? 1 : 2;
    for (int t = 0; t < ne; ++t) {
      int32_t v = e2[t];
      if (seen[v]) out[n++] = ts[j] - last[v];
      seen[v] = 1;
      last[v] = ts[j];
    }
  }
  free(last);
  free(seen);
  return n;
}

static int orc_dcmp(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* nearest rank: the ceil(p*n)-th smallest value (1-based), p in (0,1]. */
double orc_quantile_nearest_rank(int64_t n, const double* values, double p) {
  if (n <= 0) return NAN;
  double* s = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(s, values, sizeof(double) * (size_t)n);
  qsort(s, (size_t)n, sizeof(double), orc_dcmp);
  int64_t r = (int64_t)ceil(p * (double)n);
  if (r < 1) r = 1;
  if (r > n) r = n;
  double q = s[r - 1];
  free(s);
  return q;
}
