// internal.cuh — shared declarations of libmspipe (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "mspipe.h"

namespace mspipe {

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// Sticky device error flag (one per device, lives in this module).
extern __device__ int g_dev_err;

__device__ __forceinline__ void raise_dev(int bits) { atomicOr(&g_dev_err, bits); }

mspipe_status fail(mspipe_status s, const char* fmt, ...);
mspipe_status cuda_status(cudaError_t e, const char* what);

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// ---- L2 warm-up of a range a later bulk copy will read ------------------
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

// Time encoding cos(x), x = fmaf(omega, dt, phi) (G2, G22).  With raw Δt the
// argument reaches 10^6..10^7, where cosf takes its slow (Payne-Hanek, local
// memory) reduction path; reduce x mod 2π in double instead (two-term 2π,
// error ~ |k| 2^-105 + 2^-53|x|, < 1e-9 here) and evaluate cosf on |r| <= π.
__device__ __forceinline__ float time_cos(float x) {
  const double xd = (double)x;
  const double k = rint(xd * 0.15915494309189535);  // 1 / (2π)
  double r = fma(-k, 6.283185307179586232, xd);
  r = fma(-k, 2.4492935982947064e-16, r);
  return cosf((float)r);
}

// integer knob from the environment (experiments only; defaults are the tuned values)
int env_int(const char* name, int def);
// cudaLaunchKernelEx with an optional (cx,1,1) cluster.
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     unsigned cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  unsigned n = 0;
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

struct Tcsr {
  int64_t num_nodes, nnz;
  const int64_t* indptr;
  const int32_t* nbr;
  const int32_t* eid;
  const double* ts;
  int32_t stream;  // 1: the sampler's probes of nbr / eid / ts load evict-first (MSPIPE_TCSR_LDCS, A/B)
};

// T-CSR entry loads of the sampler: read-only path, or cache-streaming (evict-first)
__device__ __forceinline__ double tcsr_ts(const Tcsr& g, int64_t i) { return g.stream ? __ldcs(g.ts + i) : __ldg(g.ts + i); }
__device__ __forceinline__ int32_t tcsr_nbr(const Tcsr& g, int64_t i) {
  return g.stream ? __ldcs(g.nbr + i) : __ldg(g.nbr + i);
}
__device__ __forceinline__ int32_t tcsr_eid(const Tcsr& g, int64_t i) {
  return g.stream ? __ldcs(g.eid + i) : __ldg(g.eid + i);
}

// A1 core, executed by a whole warp for one root v at query time tq: returns
// `end`, the first row position with ts >= tq (the entries [beg, end) are the
// incident events with ts < tq, G15), and *beg = row start.  33-ary search:
// 32 lanes probe 32 interior positions of [lo, hi) per round and a ballot
// (ts is sorted, so the true lanes are a prefix) shrinks the range 33x; a row
// of L entries costs ceil(log33(L/32)) + 1 dependent rounds instead of log2(L).
// An id outside [0, N) gives an empty row and raises MSPIPE_DEVERR_RANGE.
// binary search: first position in row(v) whose ts >= t (A4's per-thread search)
__device__ __forceinline__ int64_t lower_bound_ts(const Tcsr& g, int32_t v, double t,
                                                  int64_t* beg_out) {
  const int64_t beg = __ldg(g.indptr + v);
  int64_t lo = beg, hi = __ldg(g.indptr + v + 1);
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (tcsr_ts(g, mid) < t) lo = mid + 1;
    else hi = mid;
  }
  *beg_out = beg;
  return lo;
}

// ((lane + 1) * span) / 33 without a 64-bit division (~70 instructions on the
// integer pipe, once per lane per probe round): for products below 2^32 the
// quotient is umulhi(x, ceil(2^37 / 33)) >> 5, exact for every x < 2^32
// (ceil(2^37/33) * 33 - 2^37 = 4 <= 2^(37-32)); rows of >= 2^27 entries keep
// the division.
__device__ __forceinline__ int64_t probe_offset33(int lane, int64_t span) {
  if (span < (int64_t(1) << 27)) {
    const uint32_t x = (uint32_t)(lane + 1) * (uint32_t)span;
    return (int64_t)(__umulhi(x, 0xF83E0F84u) >> 5);
  }
  return ((int64_t)(lane + 1) * span) / 33;
}

__device__ __forceinline__ int64_t warp_recent_end(const Tcsr& g, int32_t v, double tq, int lane,
                                                   int64_t* beg_out) {
  if (v < 0 || v >= g.num_nodes) {
    if (lane == 0) raise_dev(MSPIPE_DEVERR_RANGE);
    *beg_out = 0;
    return 0;
  }
  const int64_t beg = __ldg(g.indptr + v);
  int64_t lo = beg, hi = __ldg(g.indptr + v + 1);
  while (hi - lo > 32) {
    const int64_t span = hi - lo;
    const int64_t p = lo + probe_offset33(lane, span);  // strictly inside [lo, hi)
    const bool below = tcsr_ts(g, p) < tq;
    const int c = __popc(__ballot_sync(0xffffffffu, below));
    const int64_t plast = __shfl_sync(0xffffffffu, p, c > 0 ? c - 1 : 0);
    const int64_t pfirst = __shfl_sync(0xffffffffu, p, c < 32 ? c : 31);
    if (c > 0) lo = plast + 1;
    if (c < 32) hi = pfirst;
  }
  const int64_t q = lo + lane;
  const bool below = q < hi && tcsr_ts(g, q) < tq;
  *beg_out = beg;
  return lo + __popc(__ballot_sync(0xffffffffu, below));
}

// warp_recent_end plus the sample itself: lane s < F receives entry end-1-s
// (nbr, eid, ts) or nbr = eid = -1 past the row start.  The last window's ts,
// nbr and eid are loaded in ONE round and handed out by shuffles, so a row of
// at most 32 entries (most rows) costs one dependent round less than
// warp_recent_end followed by the loads; entries below the last window (a long
// row whose F most recent straddle it) are loaded directly.
__device__ __forceinline__ int64_t warp_recent_sample(const Tcsr& g, int32_t v, double tq, int lane, int F,
                                                      int64_t* beg_out, int32_t* nbr_out, int32_t* eid_out,
                                                      double* ts_out) {
  *nbr_out = -1;
  *eid_out = -1;
  *ts_out = 0.0;
  if (v < 0 || v >= g.num_nodes) {
    if (lane == 0) raise_dev(MSPIPE_DEVERR_RANGE);
    *beg_out = 0;
    return 0;
  }
  const int64_t beg = __ldg(g.indptr + v);
  int64_t lo = beg, hi = __ldg(g.indptr + v + 1);
  while (hi - lo > 32) {
    const int64_t span = hi - lo;
    const int64_t p = lo + probe_offset33(lane, span);
    const bool below = tcsr_ts(g, p) < tq;
    const int c = __popc(__ballot_sync(0xffffffffu, below));
    const int64_t plast = __shfl_sync(0xffffffffu, p, c > 0 ? c - 1 : 0);
    const int64_t pfirst = __shfl_sync(0xffffffffu, p, c < 32 ? c : 31);
    if (c > 0) lo = plast + 1;
    if (c < 32) hi = pfirst;
  }
  const int64_t q = lo + lane;
  const bool in = q < hi;
  const double tq_q = in ? tcsr_ts(g, q) : 0.0;
  const int32_t nb_q = in ? tcsr_nbr(g, q) : -1;
  const int32_t ei_q = in ? tcsr_eid(g, q) : -1;
  const int64_t end = lo + __popc(__ballot_sync(0xffffffffu, in && tq_q < tq));
  const int64_t e = end - 1 - lane;  // this lane's output slot s = lane
  const int src_lane = (int)(e - lo);
  const int32_t nb_s = __shfl_sync(0xffffffffu, nb_q, src_lane & 31);
  const int32_t ei_s = __shfl_sync(0xffffffffu, ei_q, src_lane & 31);
  const double ts_s = __shfl_sync(0xffffffffu, tq_q, src_lane & 31);
  if (lane < F && e >= beg) {
    if (e >= lo) {
      *nbr_out = nb_s;
      *eid_out = ei_s;
      *ts_out = ts_s;
    } else {
      *nbr_out = tcsr_nbr(g, e);
      *eid_out = tcsr_eid(g, e);
      *ts_out = tcsr_ts(g, e);
    }
  }
  *beg_out = beg;
  return end;
}

// warp_recent_sample with a per-node hint (k_prep; hint[v] = the answer of
// node v's previous query, stored back by every warp; any value is a valid
// start, so results never depend on it).  The stage's queries move forward in
// time and a node's answer moves only when it had events since, so most
// queries land on or just after the hint.  Round 1 loads, per lane, one entry
// of the window [w0, w0 + 32), w0 = max(beg, h - F) — the F entries below the
// hint and 32 - F after it, with their nbr / eid — and one galloping probe at
// h + 2^l - 1 (lanes 0..15) or h - 2^(l-16) (lanes 16..31).  If the answer
// falls inside the window (a hit: the common case), the window also holds
// the F most recent entries and the query costs ONE dependent round instead
// of the gallop + search + window + tail rounds; otherwise the window and the
// probes bracket the answer for the 33-ary search, which stops once one
// final window [lo - F, lo - F + 32) covers both the count and the outputs.
__device__ __forceinline__ int64_t warp_recent_sample_hinted(const Tcsr& g, int32_t v, double tq, int lane, int F,
                                                             int64_t* beg_out, int32_t* nbr_out, int32_t* eid_out,
                                                             double* ts_out, int64_t* hint) {
  *nbr_out = -1;
  *eid_out = -1;
  *ts_out = 0.0;
  if (v < 0 || v >= g.num_nodes) {
    if (lane == 0) raise_dev(MSPIPE_DEVERR_RANGE);
    *beg_out = 0;
    return 0;
  }
  const int64_t beg = __ldg(g.indptr + v), rend = __ldg(g.indptr + v + 1);
  int64_t h = __ldcg(hint + v);
  h = h < beg ? beg : (h > rend ? rend : h);
  int64_t w0 = h - F < beg ? beg : h - F;
  // round 1: window entry + galloping probe, all independent loads
  int64_t q = w0 + lane;
  bool qin = q < rend;
  double ts_q = qin ? tcsr_ts(g, q) : 0.0;
  int32_t nb_q = qin ? tcsr_nbr(g, q) : -1;
  int32_t ei_q = qin ? tcsr_eid(g, q) : -1;
  const int64_t p = lane < 16 ? h + ((int64_t(1) << lane) - 1) : h - (int64_t(1) << (lane - 16));
  const bool pin = p >= beg && p < rend;
  const bool pbelow = pin && tcsr_ts(g, p) < tq;
  int c = __popc(__ballot_sync(0xffffffffu, qin && ts_q < tq));  // below-t_q entries: a prefix of the window
  const int nin = (int)min64(32, rend - w0);
  int64_t end;
  if (c < nin && (c > 0 || w0 == beg)) {
    end = w0 + c;  // hit: entry w0 + c is the first at or after t_q, everything before it is below
  } else if (c == nin && w0 + 32 >= rend) {
    end = rend;    // the rest of the row is below t_q
  } else {
    // miss: bracket with the window (c == 0: the answer is below w0; c == 32: above the window) and the probes
    int64_t lo = c == 0 ? beg : w0 + 32, hi = c == 0 ? w0 : rend;
    int64_t lo_c = pbelow ? p + 1 : lo, hi_c = (pin && !pbelow) ? p : hi;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int64_t a = __shfl_xor_sync(0xffffffffu, lo_c, o), b = __shfl_xor_sync(0xffffffffu, hi_c, o);
      lo_c = a > lo_c ? a : lo_c;
      hi_c = b < hi_c ? b : hi_c;
    }
    lo = lo_c > lo ? lo_c : lo;
    hi = hi_c < hi ? hi_c : hi;
    while (hi - lo > 32 - F) {
      const int64_t span = hi - lo;
      const int64_t pp = lo + probe_offset33(lane, span);
      const bool below = tcsr_ts(g, pp) < tq;
      const int cc = __popc(__ballot_sync(0xffffffffu, below));
      const int64_t plast = __shfl_sync(0xffffffffu, pp, cc > 0 ? cc - 1 : 0);
      const int64_t pfirst = __shfl_sync(0xffffffffu, pp, cc < 32 ? cc : 31);
      if (cc > 0) lo = plast + 1;
      if (cc < 32) hi = pfirst;
    }
    // final window: the count over [lo, hi) and the F entries below the answer
    w0 = lo - F < beg ? beg : lo - F;
    q = w0 + lane;
    qin = q < rend;
    ts_q = qin ? tcsr_ts(g, q) : 0.0;
    nb_q = qin ? tcsr_nbr(g, q) : -1;
    ei_q = qin ? tcsr_eid(g, q) : -1;
    end = lo + __popc(__ballot_sync(0xffffffffu, q >= lo && q < hi && ts_q < tq));
  }
  const int64_t e = end - 1 - lane;  // this lane's output slot s = lane
  const int src_lane = (int)(e - w0);
  const int32_t nb_s = __shfl_sync(0xffffffffu, nb_q, src_lane & 31);
  const int32_t ei_s = __shfl_sync(0xffffffffu, ei_q, src_lane & 31);
  const double ts_s = __shfl_sync(0xffffffffu, ts_q, src_lane & 31);
  if (lane < F && e >= beg) {
    if (e >= w0) {
      *nbr_out = nb_s;
      *eid_out = ei_s;
      *ts_out = ts_s;
    } else {  // a hit below a hint that ran ahead (e.g. after an epoch reset)
      *nbr_out = tcsr_nbr(g, e);
      *eid_out = tcsr_eid(g, e);
      *ts_out = tcsr_ts(g, e);
    }
  }
  if (lane == 0) hint[v] = end;
  *beg_out = beg;
  return end;
}

// The sampler's probes of a T-CSR much larger than L2 (GDELT: 382M entries, 6 GB)
// load evict-first: the probed sectors are rarely reused and pushed the state
// tables and GEMM operands out of L2 (r02zl: 97.2 vs 96.0 M events/s); a small
// T-CSR keeps the read-only path (wiki: neutral).  MSPIPE_TCSR_LDCS=0/1 forces it.
inline Tcsr to_tcsr(const mspipe_tcsr* g) {
  const int forced = env_int("MSPIPE_TCSR_LDCS", -1);
  const int stream = forced >= 0 ? forced : (g->nnz * 16 > (int64_t)(256ll << 20) ? 1 : 0);
  return Tcsr{g->num_nodes, g->nnz, g->indptr, g->nbr, g->eid, g->ts, stream};
}

// ---- kernels' host-side launchers (one .cu each) -------------------------
// sampler.cu
void launch_sample(const Tcsr& g, const int32_t* roots, const double* qts, const int32_t* src,
                   const int32_t* dst, const int32_t* neg, const double* ev_ts, int64_t num_events,
                   int64_t num_roots, int32_t fanout, int32_t* out_nbr, int32_t* out_eid,
                   double* out_ts, float* out_dt, int32_t* out_cnt, int32_t* out_sub,
                   cudaStream_t s);
// memory.cu
void launch_fetch(const int32_t* ids, int64_t n, int64_t num_nodes, const float* mem,
                  const double* mem_ts, int32_t mem_dim, const float* mail, const double* mail_ts,
                  int64_t mail_stride, float* out_mem, double* out_mem_ts, float* out_mail,
                  double* out_mail_ts, cudaStream_t s);
void launch_mitigate(const Tcsr& g, const int32_t* src, const int32_t* dst, const double* ts,
                     int64_t num_events, const float* mem, const double* mem_ts, int32_t mem_dim,
                     float lambda, double gamma, int32_t n_sim, int32_t fanout, float* out_h,
                     int32_t* out_omega, uint8_t* out_elig, cudaStream_t s);
void launch_dedup(const int32_t* src, const int32_t* dst, int64_t num_events, int32_t* scratch,
                  int64_t num_nodes, int32_t* out_nodes, int32_t* out_winner, int32_t* out_num,
                  cudaStream_t s, int32_t* stamp = nullptr, int32_t stamp_iter = 0);
void launch_writeback(const int32_t* nodes, const int32_t* num, int64_t max_n,
                      const float* new_mem, const double* new_ts, const float* new_mail,
                      int32_t mem_dim, int64_t mail_stride, float* mem, double* mem_ts,
                      float* mail, double* mail_ts, int64_t num_nodes, cudaStream_t s);
void launch_rows_to_host(const int32_t* num, int32_t* host_num, const void* a, void* host_a, int64_t a_row_bytes,
                         const void* b, void* host_b, int64_t b_row_bytes, int64_t max_rows, cudaStream_t s);
void launch_catchup(const int32_t* prev_nodes, const int32_t* prev_num, int64_t prev_max, const float* src_mem,
                    const double* src_mem_ts, const float* src_mail, const double* src_mail_ts, float* dst_mem,
                    double* dst_mem_ts, float* dst_mail, double* dst_mail_ts, int32_t mem_dim, int64_t mail_stride,
                    const int32_t* cur_nodes, const int32_t* cur_num, int64_t cur_max, int32_t* save_nodes,
                    int32_t* save_num, cudaStream_t s);
// gru_simt.cu
struct GruDesc {
  int32_t M, He, Dt, Dm, Dx, K, Kpad, Npad;
  const float* wpack;   // [Kpad, Npad]
  const float* bias;    // [Npad]
  const float* time_w;  // [Dt]
  const float* time_b;  // [Dt]
  int32_t bf16;         // 1: bf16 tensor-core operands (MSPIPE_BF16), Kpad a multiple of 64
  int32_t cell;         // MSPIPE_CELL_GRU | MSPIPE_CELL_RNN (row F3)
  int32_t mailbox;      // MSPIPE_MAILBOX_IMMEDIATE | MSPIPE_MAILBOX_DEFERRED (row F3)
  float* gates;         // optional sink (row F4, mspipe_gru_save_gates): gate pre-activations [rows, 4M]
};
void launch_gru_pack(const float* w_ih, const float* w_hh, const float* b_ih, const float* b_hh,
                     const GruDesc& d, float* wpack, float* bias, cudaStream_t s);
void launch_gru_simt(const GruDesc& d, const int32_t* src, const int32_t* dst, const double* ts,
                     int64_t num_events, const float* edge_feat, const float* snap_mem,
                     const double* snap_mem_ts, int64_t snap_step, const float* snap_h,
                     const int32_t* nodes, const int32_t* winner, const int32_t* num_unique,
                     float* out_mem, double* out_ts, float* out_mail, int64_t mail_stride,
                     cudaStream_t s);

// gru_tc.cu
size_t gru_tc_packed_floats(const GruDesc& d);
size_t gru_tc_bias_floats(const GruDesc& d);  // J tiles x 4 gates x kJ
size_t gru_tc_xbuf_floats(const GruDesc& d, int64_t max_events);
void launch_gru_pack_tc(const float* w_ih, const float* w_hh, const float* b_ih, const float* b_hh,
                        const GruDesc& d, float* wtc, float* bias, cudaStream_t s);
enum { kGruBuild = 1, kGruGemm = 2 };
// double-buffered state: copy the rows of the previous commit (prev_nodes,
// from set `old_*`) into the next commit's set (`new_*`), skipping the nodes
// with stamp[v] == iter (that commit's own winners, which it writes itself)
struct CatchUp {
  const int32_t* prev_nodes;
  const int32_t* prev_num;
  const float* old_mem;
  const double* old_mem_ts;
  const float* old_mail;
  const double* old_mail_ts;
  float* new_mem;
  double* new_mem_ts;
  float* new_mail;
  double* new_mail_ts;
  const int32_t* stamp;
  int32_t iter;
};

// fused A5 inside the prep kernel (mspipe_memory_prep_build)
// one warp copies row v of every table (4 x 16 B loads in flight per lane)
__device__ __forceinline__ void catchup_row(const CatchUp& c, int32_t v, int32_t Qm, int32_t Qa, int lane) {
  const float4* om = reinterpret_cast<const float4*>(c.old_mem) + (int64_t)v * Qm;
  const float4* oa = reinterpret_cast<const float4*>(c.old_mail) + (int64_t)v * Qa;
  float4* nm = reinterpret_cast<float4*>(c.new_mem) + (int64_t)v * Qm;
  float4* na = reinterpret_cast<float4*>(c.new_mail) + (int64_t)v * Qa;
  const int total = Qm + Qa;
  for (int base = 0; base < total; base += 128) {
    float4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = base + u * 32 + lane;
      if (q < total) x[u] = q < Qm ? __ldg(om + q) : __ldg(oa + (q - Qm));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = base + u * 32 + lane;
      if (q < Qm) nm[q] = x[u];
      else if (q < total) na[q - Qm] = x[u];
    }
  }
  if (lane == 0) {
    c.new_mem_ts[v] = __ldg(c.old_mem_ts + v);
    c.new_mail_ts[v] = __ldg(c.old_mail_ts + v);
  }
}

struct GruCommit {  // fused A7 in the GEMM epilogue
  const int32_t* nodes;
  float* mem;
  double* mem_ts;
  float* mail;
  double* mail_ts;
  const double* new_ts;
  const float* new_mail;
  int64_t num_nodes;
  int64_t mail_stride;
  // double-buffered state (optional): save this commit's winner list for the
  // next commit and, when `stamp` is set, catch up the previous commit's rows
  // (prev_nodes from set `old_*`), skipping nodes with stamp[v] == iter
  // (this commit's winners, stamped by k_prep)
  int32_t* save_nodes;
  int32_t* save_num;
  CatchUp cu;  // cu.stamp == nullptr: no catch-up in this kernel
  int32_t skip_meta;  // 1: the epilogue writes only h' rows (mem_ts / mail / mail_ts by k_writeback)
  int32_t* res_nodes;  // optional: winner node ids [U] and U into a result record
  int32_t* res_num;
};
// row F3, deferred mailbox: A5 from the snapshot mail rows (snap_mail, rows as snap_mem)
cudaError_t launch_build_deferred(const GruDesc& d, float* xbuf, const double* ts, int64_t num_events,
                                  const float* snap_mem, const double* snap_mem_ts, const float* snap_mail,
                                  int64_t mail_stride, int64_t snap_step, const int32_t* winner,
                                  const int32_t* num_unique, double* out_ts, cudaStream_t s);
// row F3, deferred mailbox, after the commit: mail[w] = [mem[w] | mem[o] | e], mail_ts[w] = t
void launch_mail_deferred(const int32_t* src, const int32_t* dst, const double* ts, const float* ef, int32_t He,
                          const int32_t* nodes, const int32_t* winner, const int32_t* num_unique, int64_t max_n,
                          const float* mem, int32_t M, float* mail, double* mail_ts, int64_t mail_stride,
                          int64_t num_nodes, cudaStream_t s);
cudaError_t launch_gru_tc(const GruDesc& d, const float* wtc, float* xbuf, const double* ts, int64_t num_events,
                          const float* edge_feat, const float* snap_mem, const double* snap_mem_ts,
                          int64_t snap_step, const float* snap_h, const int32_t* winner,
                          const int32_t* num_unique, float* out_mem, double* out_ts, float* out_mail,
                          int64_t mail_stride, cudaStream_t s, int parts = kGruBuild | kGruGemm,
                          const GruCommit* commit = nullptr, const int32_t* tab_src = nullptr,
                          const int32_t* tab_dst = nullptr);
// features.cu
cudaError_t launch_feature_fetch(const int32_t* sub, const int32_t* eid, int64_t R, int32_t F, const float* nfeat,
                                 int64_t N, int32_t nstride, const float* efeat, int64_t E, int32_t estride,
                                 float* out_n, float* out_e, cudaStream_t s);
// stale.cu
void shard_mit_candidates(const Tcsr& g, const int32_t* src, const int32_t* dst, const double* ts, int64_t B,
                          const double* root_ts, int64_t root_step, double gamma, int32_t F, int32_t* out_ids,
                          cudaStream_t s);
void shard_fetch_finish_table(mspipe_memory* st, const int32_t* ids, int64_t n, float* tab_mem, double* tab_ts,
                              cudaStream_t s);
cudaError_t launch_staleness_error(const int32_t* winner, const int32_t* num_unique, int64_t num_events,
                                  const float* rows_a, int64_t stride_a, const float* rows_b, int64_t stride_b,
                                  int32_t mem_dim, double* out, cudaStream_t s);
cudaError_t launch_stale_hist(const Tcsr& g, const int32_t* src, const int32_t* dst, int64_t E, int64_t B,
                              int32_t max_d, unsigned long long* hist, cudaStream_t s);
// prep.cu
cudaError_t launch_prep(const Tcsr& g, const int32_t* src, const int32_t* dst, const int32_t* neg,
                        const double* ts, int64_t num_events, int32_t fanout, int32_t* out_nbr,
                        int32_t* out_eid, double* out_ts, float* out_dt, int32_t* out_cnt, int32_t* out_sub,
                        int32_t* scratch, int32_t* out_nodes, int32_t* out_winner, int32_t* out_num,
                        const float* mem, const double* mem_ts, int32_t mem_dim, const float* mail,
                        const double* mail_ts, int64_t mail_stride, float* out_mem, double* out_mem_ts,
                        float* out_mail, double* out_mail_ts, cudaStream_t s, int32_t* stamp = nullptr,
                        int32_t stamp_iter = 0, const struct CatchUp* cu = nullptr, int64_t* hint = nullptr);

}  // namespace mspipe

struct mspipe_memory;
namespace mspipe {
// shard.cu
void shard_fetch_plan(mspipe_memory* st, const int32_t* ids, int64_t n, cudaStream_t s);
void shard_fetch_serve(mspipe_memory* st, bool with_mail, cudaStream_t s);
void shard_fetch_finish(mspipe_memory* st, const int32_t* ids, int64_t n, float* out_mem, double* out_mem_ts,
                        float* out_mail, double* out_mail_ts, cudaStream_t s);
void shard_commit_pack(mspipe_memory* st, int64_t commit_version, const int32_t* nodes, const int32_t* winner,
                       const int32_t* num, int64_t max_n, int64_t key_base, const float* new_mem,
                       const double* new_ts, const float* new_mail, cudaStream_t s);
void shard_commit_merge(mspipe_memory* st, int64_t commit_version, cudaStream_t s);
int64_t shard_fetch_rec_bytes(const mspipe_memory* st, bool with_mail);
int64_t shard_commit_rec_bytes(const mspipe_memory* st);
void shard_layout(mspipe_memory* st);
// nccl_xchg.cu
mspipe_status nccl_comm_init(mspipe_memory* st, const void* unique_id);
void nccl_comm_destroy(mspipe_memory* st);
mspipe_status nccl_barrier(mspipe_memory* st, bool fetch, cudaStream_t s);
int32_t nccl_unique_id_bytes();
mspipe_status nccl_get_unique_id(void* out);
}  // namespace mspipe

struct mspipe_memory {
  int64_t num_nodes;
  int32_t mem_dim, edge_dim, mail_dim, k;
  float* mem;
  double* mem_ts;
  float* mail;
  double* mail_ts;
  int64_t mail_stride;
  int32_t rank, world;
  int64_t committed;
  int32_t* scratch;  // [num_nodes] int32, -1 between calls (self-cleaning)
  int64_t* sample_hint;  // [num_nodes] search start per node for the fused prep's sampler (any value is valid)
  int device;
  // ---- world > 1 (shard.cu) ----
  int64_t local_rows;       // rows of this rank's shard: nodes v with v % world == rank
  int64_t sh_cap;           // request / reply slots per peer = ceil(num_nodes / world)
  int64_t sh_capw;          // commit records per peer
  uint8_t* sh_needed;       // [num_nodes] request marks (cleared by the plan)
  int32_t* sh_slot_of;      // [num_nodes] slot of id v in its owner's request list
  int32_t* sh_dest;         // [num_nodes] owner * capw + slot of each local winner
  unsigned long long* sh_keytab;  // [local_rows] LWW key of the committed row
  int32_t sh_with_mail;     // the in-flight fetch carries mail rows
  int64_t sh_fetch_iter;    // iteration of the fetch in flight (window parity)
  // receive window: one allocation (exported by CUDA IPC), per parity p:
  // ids [world][cap] i32 | counts [3][world] i32 | replies [world][cap] | commits [world][capw]
  uint8_t* sh_window;
  int64_t sh_win_bytes, sh_off_ids[2], sh_off_cnt[2], sh_off_rep[2], sh_off_com[2];
  uint8_t** sh_peers;       // [world] device: every rank's window in this process's address space
  void* sh_peer_host[64];   // host copy (entries of other processes opened by cudaIpcOpenMemHandle)
  uint8_t sh_peer_ipc[64];  // 1: sh_peer_host[p] must be closed with cudaIpcCloseMemHandle
  int32_t sh_connected;     // 0: not yet, 1: IPC peers + NCCL barriers, 2: in-process ranks (stream order)
  unsigned long long* sh_sent;  // [3] device: bytes stored into windows (fetch ids, replies, commit records)
  int32_t* sh_bar;          // [2] device: barrier all-reduce operands (commit, fetch)
  void* nccl_comm;          // ncclComm_t of the commit barriers (NULL: in-process rank)
  void* nccl_comm_fetch;    // ncclComm_t of the fetch barriers
  // ---- double-buffered state (mspipe_memory_double_buffer) ----
  // Set 0 = the tables above, set 1 = a second caller-owned set; version c
  // lives in set c & 1.  Commit c first copies the rows of commit c-1 from
  // set (c-1)&1 into set c&1 (catch-up), then writes its own rows there, so a
  // fetch of version c-1 never shares a table with commit c.
  int32_t db;
  float* mem1;
  double* mem_ts1;
  float* mail1;
  double* mail_ts1;
  int32_t* prev_nodes;  // [2][num_nodes] winners of the last commit of each parity
  int32_t* prev_num;    // [2]
  int64_t prev_max[2];  // host bound on prev_num[p] (launch sizing)
  // winner stamps written by mspipe_memory_prep(i) into ring slot i % (k+1)
  // (stamp[v] = i); they let commit i's GEMM kernel do the catch-up itself
  int32_t* stamps;          // [k+1][num_nodes]
  int64_t* stamp_iter;      // [k+1] host: iteration whose winners ring slot r holds (0 = none)
  int64_t caught_up;        // host: the commit whose catch-up a prep has already enqueued (0 = none)
  // library-owned branches beside the caller's stream, per handle (created at
  // mspipe_memory_create, so never lazily under a stream capture): 0 = the
  // commit's write-back branch, 1 = the prep's mitigation branch
  cudaStream_t aux[2];
  cudaEvent_t aux_fork[2], aux_join[2];
};

namespace mspipe {
struct TableSet {
  float* mem;
  double* mem_ts;
  float* mail;
  double* mail_ts;
};
// the tables holding `version` (valid for version == committed, and committed - 1 when double-buffered)
inline TableSet table_set(const mspipe_memory* st, int64_t version) {
  if (st->db && (version & 1)) return {st->mem1, st->mem_ts1, st->mail1, st->mail_ts1};
  return {st->mem, st->mem_ts, st->mail, st->mail_ts};
}
}  // namespace mspipe

struct mspipe_gru {
  mspipe::GruDesc d;
  int32_t precision;
  int64_t max_events;
  float* wpack;  // SIMT layout [Kpad, Npad] (precision FP32_SIMT)
  float* wtc;    // tcgen05 B-operand images (precision FP32_3XTF32)
  float* xbuf;   // tcgen05 A-operand images for <= max_events events
  float* bias;
  float* time_w;
  float* time_b;
};
