// memory.cu — A3 snapshot fetch, A4 mitigation, A2 dedup, A7 write-back.
#include "dedup.cuh"
#include "internal.cuh"

namespace mspipe {

static inline unsigned grid_for(int64_t work_items, int threads, int per_sm) {
  int64_t b = (work_items + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

// ---------------------------------------------------------------------------
// Warp row copy: nrows (<= 32) rows of Q float4.  Row s comes from
// src + (kSrcIds ? id_s : src_row0 + s)·Q and goes to
// dst + (kDstIds ? id_s : dst_row0 + s)·Q, id_s held by lane s (shuffled);
// a negative source id gives a zero row, a negative destination id skips the
// row.  The nrows·Q elements are flattened over the 32 lanes (no idle lanes
// for Q = 25), kU 16-byte loads in flight per lane before their stores, and
// the (row, column) of each element is advanced incrementally (no division).
// ---------------------------------------------------------------------------
template <int kU, bool kSrcIds, bool kDstIds>
__device__ __forceinline__ void warp_copy_rows(const float4* __restrict__ src, int64_t src_row0,
                                               float4* __restrict__ dst, int64_t dst_row0, int32_t Q, int nrows,
                                               int32_t my_id, int lane) {
  const int total = nrows * Q;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  const int q32 = 32 / Q, r32 = 32 - q32 * Q;
  int s = lane / Q, c = lane - (lane / Q) * Q;
  for (int base = 0; base < total; base += 32 * kU) {
    float4 v[kU];
    const int s0 = s, c0 = c;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const bool in = base + u * 32 + lane < total;
      const int32_t id = kSrcIds ? __shfl_sync(0xffffffffu, my_id, s < nrows ? s : 0) : 0;
      const int64_t srow = kSrcIds ? (int64_t)id : src_row0 + s;
      v[u] = (in && srow >= 0) ? __ldg(src + srow * Q + c) : z;
      s += q32;
      c += r32;
      if (c >= Q) {
        c -= Q;
        ++s;
      }
    }
    // the stores walk the same (row, column) sequence again (no per-load index registers)
    s = s0;
    c = c0;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const bool in = base + u * 32 + lane < total;
      const int32_t id = kDstIds ? __shfl_sync(0xffffffffu, my_id, s < nrows ? s : 0) : 0;
      const int64_t drow = kDstIds ? (int64_t)id : dst_row0 + s;
      if (in && drow >= 0) dst[drow * Q + c] = v[u];
      s += q32;
      c += r32;
      if (c >= Q) {
        c -= Q;
        ++s;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// A3 — gather rows of the state tables into dense snapshot buffers
// ("fetches the required ... node memory vectors"; Eq. 2 reads
// s~^(i-k)).  A warp moves kFetchRows rows per step: their ids
// (one per lane), then warp_copy_rows of the mem rows (and the mail rows),
// then the row timestamps.  Each row read is one contiguous 400 B (mem) /
// 1.5 KB (mail) segment and each write is dense.  id -1 = pad (zero row, ts 0).
// ---------------------------------------------------------------------------
constexpr int kFetchRows = 8;
constexpr int kCopyU = 8;
// write-back batches are small (U <= 2B rows, ~1,600 at GDELT): 2 rows per
// warp keeps ~800 warps in flight instead of ~200 (8 rows per warp measured
// 10.6 vs 6.4 us for the commit branch at GDELT)
constexpr int kWbRows = 2;

__global__ void __launch_bounds__(256, 4) k_fetch_gather(
    const int32_t* __restrict__ ids, int64_t n, int64_t N, const float4* __restrict__ mem,
    const double* __restrict__ mem_ts, int32_t Qm, const float4* __restrict__ mail,
    const double* __restrict__ mail_ts, int32_t Qa, float4* __restrict__ out_mem,
    double* __restrict__ out_mem_ts, float4* __restrict__ out_mail,
    double* __restrict__ out_mail_ts) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kFetchRows; base < n;
       base += nwarps * kFetchRows) {
    const int nrows = (int)min64(kFetchRows, n - base);
    int32_t id = lane < nrows ? __ldg(ids + base + lane) : -1;
    if (lane < nrows && (id < -1 || id >= N)) raise_dev(MSPIPE_DEVERR_RANGE);
    if (id >= N || id < -1) id = -1;
    warp_copy_rows<kCopyU, true, false>(mem, 0, out_mem, base, Qm, nrows, id, lane);
    if (Qa > 0) warp_copy_rows<kCopyU, true, false>(mail, 0, out_mail, base, Qa, nrows, id, lane);
    if (lane < nrows) {
      out_mem_ts[base + lane] = id >= 0 ? __ldg(mem_ts + id) : 0.0;
      if (out_mail_ts) out_mail_ts[base + lane] = id >= 0 ? __ldg(mail_ts + id) : 0.0;
    }
  }
}

void launch_fetch(const int32_t* ids, int64_t n, int64_t num_nodes, const float* mem,
                  const double* mem_ts, int32_t mem_dim, const float* mail, const double* mail_ts,
                  int64_t mail_stride, float* out_mem, double* out_mem_ts, float* out_mail,
                  double* out_mail_ts, cudaStream_t s) {
  const int32_t Qm = mem_dim / 4;
  const int32_t Qa = mail ? (int32_t)(mail_stride / 4) : 0;
  const int threads = 256;
  launch_k(k_fetch_gather, dim3(grid_for((n + kFetchRows - 1) / kFetchRows * 32, threads, 4)), dim3(threads), 0, s,
           1, ids, n, num_nodes, (const float4*)mem, mem_ts, Qm, (const float4*)mail, mail_ts, Qa, (float4*)out_mem,
           out_mem_ts, (float4*)out_mail, out_mail_ts);
}

// ---------------------------------------------------------------------------
// A4 — MSPipe-S similarity-based mitigation, one warp per
// target.  Eligibility is one compare; only eligible targets (the Δt tail,
// ~1-p of rows) walk the 2-hop neighbourhood.  Every decision uses
// only ids and timestamps, so eligibility and Ω are bit-exact; the blend is
// f32.
// ---------------------------------------------------------------------------
constexpr int kMitMaxF = 16;
constexpr int kMitMaxC = kMitMaxF * kMitMaxF;
constexpr int kMitWarps = 4;

struct MitWarpSmem {
  int32_t cand[kMitMaxC];
  int32_t kid[kMitMaxC];
  int32_t kc[kMitMaxC];
  double kmts[kMitMaxC];
  int32_t omega[kMitMaxF];
};


__global__ void __launch_bounds__(32 * kMitWarps) k_mitigate(
    Tcsr g, const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
    const double* __restrict__ ts, int64_t B, const float* __restrict__ mem,
    const double* __restrict__ mem_ts, int32_t M, float lambda, double gamma, int32_t n_sim,
    int32_t F, float* __restrict__ out_h, int32_t* __restrict__ out_omega,
    uint8_t* __restrict__ out_elig) {
  __shared__ MitWarpSmem sm_all[kMitWarps];
  const int lane = threadIdx.x & 31;
  MitWarpSmem& sm = sm_all[threadIdx.x >> 5];
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int32_t Q = M / 4;
  const float4* mem4 = (const float4*)mem;
  float4* h4 = (float4*)out_h;
  for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < 2 * B; t += nwarps) {
    const int64_t a = t < B ? t : t - B;
    const int32_t w = t < B ? __ldg(src + a) : __ldg(dst + a);
    const double tstar = __ldg(ts + a);
    const bool wok = w >= 0 && w < g.num_nodes;
    if (!wok && lane == 0) raise_dev(MSPIPE_DEVERR_RANGE);
    const double mtw = wok ? __ldg(mem_ts + w) : 0.0;
    const bool elig = wok && (tstar - mtw) > gamma;  // G11: strictly longer than γ
    int32_t nk = 0;
    if (elig) {
      // N1 = distinct ids of sample(w, t*) \ {w}
      int64_t begw;
      const int64_t endw = lower_bound_ts(g, w, tstar, &begw);
      const int32_t cntw = (int32_t)min64(endw - begw, (int64_t)F);
      int32_t x = (lane < cntw) ? __ldg(g.nbr + (endw - 1 - lane)) : -1;
      if (x == w) x = -1;
      const unsigned grp = __match_any_sync(0xffffffffu, x);
      const bool keep = x >= 0 && lane == __ffs(grp) - 1;
      // candidates: lane l < F owns slots [l*F, (l+1)*F) with the distinct ids of sample(x_l, t*) \ {w}
      if (lane < F) {
        int32_t nl = 0;
        if (keep) {
          int64_t begx;
          const int64_t endx = lower_bound_ts(g, x, tstar, &begx);
          const int32_t cx = (int32_t)min64(endx - begx, (int64_t)F);
          for (int32_t i = 0; i < cx; ++i) {
            const int32_t u = __ldg(g.nbr + (endx - 1 - i));
            if (u == w) continue;
            bool dup = false;
            for (int32_t j = 0; j < nl; ++j) dup |= (sm.cand[lane * F + j] == u);
            if (!dup) sm.cand[lane * F + nl++] = u;
          }
        }
        for (int32_t j = nl; j < F; ++j) sm.cand[lane * F + j] = -1;
      }
      __syncwarp();
      // c(u) = #lists containing u; keep first occurrence of each active u
      const int32_t FF = F * F;
      for (int32_t e0 = 0; e0 < FF; e0 += 32) {
        const int32_t e = e0 + lane;
        const int32_t u = e < FF ? sm.cand[e] : -1;
        bool take = false;
        int32_t c = 0;
        double mu = 0.0;
        if (u >= 0) {
          bool first = true;
          for (int32_t e2 = 0; e2 < FF; ++e2) {
            const int32_t u2 = sm.cand[e2];
            if (u2 == u) {
              ++c;
              if (e2 < e) first = false;
            }
          }
          if (first) {
            mu = __ldg(mem_ts + u);
            take = mu > mtw && (tstar - mu) < gamma;  // active: fresher than w and Δt < γ
          }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, take);
        if (take) {
          const int32_t pos = nk + __popc(bal & ((1u << lane) - 1u));
          sm.kid[pos] = u;
          sm.kc[pos] = c;
          sm.kmts[pos] = mu;
        }
        nk += __popc(bal);
      }
      __syncwarp();
      // rank by (c desc, mem_ts desc, id asc); the first n_sim form Ω
      for (int32_t i = lane; i < nk; i += 32) {
        const int32_t ui = sm.kid[i], ci = sm.kc[i];
        const double mi = sm.kmts[i];
        int32_t rank = 0;
        for (int32_t j = 0; j < nk; ++j) {
          const int32_t cj = sm.kc[j];
          const double mj = sm.kmts[j];
          const int32_t uj = sm.kid[j];
          rank += (cj > ci) || (cj == ci && (mj > mi || (mj == mi && uj < ui)));
        }
        if (rank < n_sim) sm.omega[rank] = ui;
      }
      __syncwarp();
    }
    const int32_t k = min(nk, n_sim);
    if (out_omega && lane < n_sim) out_omega[t * n_sim + lane] = lane < k ? sm.omega[lane] : -1;
    if (out_elig && lane == 0) out_elig[t] = elig ? 1 : 0;
    for (int32_t q = lane; q < Q; q += 32) {
      float4 sw = wok ? __ldg(mem4 + (int64_t)w * Q + q) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (k > 0) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int32_t s2 = 0; s2 < k; ++s2) {
          const float4 v = __ldg(mem4 + (int64_t)sm.omega[s2] * Q + q);
          acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        const float inv = (float)k;
        const float l1 = 1.0f - lambda;
        sw.x = lambda * sw.x + l1 * (acc.x / inv);
        sw.y = lambda * sw.y + l1 * (acc.y / inv);
        sw.z = lambda * sw.z + l1 * (acc.z / inv);
        sw.w = lambda * sw.w + l1 * (acc.w / inv);
      }
      h4[t * Q + q] = sw;
    }
    __syncwarp();
  }
}

void launch_mitigate(const Tcsr& g, const int32_t* src, const int32_t* dst, const double* ts,
                     int64_t num_events, const float* mem, const double* mem_ts, int32_t mem_dim,
                     float lambda, double gamma, int32_t n_sim, int32_t fanout, float* out_h,
                     int32_t* out_omega, uint8_t* out_elig, cudaStream_t s) {
  const int threads = 32 * kMitWarps;
  launch_k(k_mitigate, dim3(grid_for(2 * num_events * 32, threads, 16)), dim3(threads), 0, s, 1, g, src, dst, ts,
           num_events, mem, mem_ts, mem_dim, lambda, gamma, n_sim, fanout, out_h, out_omega, out_elig);
}

// ---------------------------------------------------------------------------
// A2 — deterministic most-recent dedup in one CTA.  Pair p = 2a + role has
// node src_a (role 0) / dst_a (role 1); the winner of node w is max{p} (the
// most recent message, G6).  Phase 1: warp-aggregated atomicMax of p into
// scratch[node] (__match_any_sync groups equal nodes so a hot node costs one
// atomic per warp; max is order-independent).  Phase 2: a pair wins iff
// scratch[node_p] == p; a block scan over contiguous chunks compacts the
// winners in p order.  Phase 3: winners restore scratch[node] = -1.
// ---------------------------------------------------------------------------
constexpr int kDedupThreads = 1024;

template <bool kSmem>
__global__ void __launch_bounds__(kDedupThreads) k_dedup(
    const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int64_t B,
    int32_t* __restrict__ gscratch, int64_t N, int32_t* __restrict__ out_nodes,
    int32_t* __restrict__ out_winner, int32_t* __restrict__ out_num, int32_t* __restrict__ stamp,
    int32_t stamp_iter) {
  extern __shared__ int32_t sscratch[];
  block_dedup<kDedupThreads, kSmem>(src, dst, B, gscratch, sscratch, N, out_nodes, out_winner, out_num);
  if (stamp) {  // double-buffered state: stamp[winner node] = iteration (as k_prep's dedup block)
    __syncthreads();
    const int32_t U = *out_num;
    for (int32_t u = threadIdx.x; u < U; u += kDedupThreads) stamp[out_nodes[u]] = stamp_iter;
  }
}

void launch_dedup(const int32_t* src, const int32_t* dst, int64_t num_events, int32_t* scratch,
                  int64_t num_nodes, int32_t* out_nodes, int32_t* out_winner, int32_t* out_num,
                  cudaStream_t s, int32_t* stamp, int32_t stamp_iter) {
  if (num_nodes <= kDedupSmemNodes) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_dedup<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(kDedupSmemNodes * sizeof(int32_t)));
      attr = true;
    }
    launch_k(k_dedup<true>, dim3(1), dim3(kDedupThreads), num_nodes * sizeof(int32_t), s, 1, src, dst, num_events,
             scratch, num_nodes, out_nodes, out_winner, out_num, stamp, stamp_iter);
  } else {
    launch_k(k_dedup<false>, dim3(1), dim3(kDedupThreads), 0, s, 1, src, dst, num_events, scratch, num_nodes,
             out_nodes, out_winner, out_num, stamp, stamp_iter);
  }
}

// ---------------------------------------------------------------------------
// A7 — write-back of U unique rows (commit of version i, P:L154, P:L820,
// P:L854-L855).  Rows are unique within a batch, so the scatter is a plain
// copy; a warp moves kFetchRows rows per step (loads of all rows first, then
// the stores).  U is read on the device.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 4) k_writeback(
    const int32_t* __restrict__ nodes, const int32_t* __restrict__ num, int64_t max_n,
    const float4* __restrict__ new_mem, const double* __restrict__ new_ts,
    const float4* __restrict__ new_mail, int32_t Qm, int32_t Qa, float4* __restrict__ mem,
    double* __restrict__ mem_ts, float4* __restrict__ mail, double* __restrict__ mail_ts,
    int64_t N) {
  const int64_t U = min64((int64_t)__ldg(num), max_n);
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kWbRows; base < U;
       base += nwarps * kWbRows) {
    const int nrows = (int)min64(kWbRows, U - base);
    int32_t node = lane < nrows ? __ldg(nodes + base + lane) : -1;
    if (lane < nrows && (node < 0 || node >= N)) {
      raise_dev(MSPIPE_DEVERR_RANGE);
      node = -1;
    }
    if (Qm > 0) warp_copy_rows<kCopyU, false, true>(new_mem, base, mem, 0, Qm, nrows, node, lane);
    if (Qa > 0) warp_copy_rows<kCopyU, false, true>(new_mail, base, mail, 0, Qa, nrows, node, lane);
    if (node >= 0) {
      const double t1 = __ldg(new_ts + base + lane);
      mem_ts[node] = t1;
      mail_ts[node] = t1;
    }
  }
}

void launch_writeback(const int32_t* nodes, const int32_t* num, int64_t max_n,
                      const float* new_mem, const double* new_ts, const float* new_mail,
                      int32_t mem_dim, int64_t mail_stride, float* mem, double* mem_ts,
                      float* mail, double* mail_ts, int64_t num_nodes, cudaStream_t s) {
  const int32_t Qm = mem_dim / 4, Qa = (int32_t)(mail_stride / 4);
  const int threads = 256;
  launch_k(k_writeback, dim3(grid_for((max_n + kWbRows - 1) / kWbRows * 32, threads, 4)), dim3(threads), 0, s,
           1, nodes, num, max_n, (const float4*)new_mem, new_ts, (const float4*)new_mail, Qm, Qa, (float4*)mem,
           mem_ts, (float4*)mail, mail_ts, num_nodes);
}

// Double-buffered state, first half of commit c: the rows of commit c-1 (one
// warp per node) from set (c-1)&1 into set c&1, and this commit's winner list
// saved for commit c+1.  Stream order puts it before the commit's own writes.
__global__ void __launch_bounds__(256) k_catchup(const int32_t* __restrict__ prev_nodes,
                                                 const int32_t* __restrict__ prev_num,
                                                 const float4* __restrict__ src_mem, const double* __restrict__ src_mem_ts,
                                                 const float4* __restrict__ src_mail,
                                                 const double* __restrict__ src_mail_ts, float4* __restrict__ dst_mem,
                                                 double* __restrict__ dst_mem_ts, float4* __restrict__ dst_mail,
                                                 double* __restrict__ dst_mail_ts, int32_t Qm, int32_t Qa,
                                                 const int32_t* __restrict__ cur_nodes,
                                                 const int32_t* __restrict__ cur_num, int32_t* __restrict__ save_nodes,
                                                 int32_t* __restrict__ save_num) {
  const int lane = threadIdx.x & 31;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int32_t np = prev_num ? __ldg(prev_num) : 0;  // NULL: only save this commit's list
  for (int64_t w = gtid >> 5; w < np; w += nthreads >> 5) {
    const int32_t v = __ldg(prev_nodes + w);
    for (int c = lane; c < Qm; c += 32) dst_mem[(int64_t)v * Qm + c] = __ldg(src_mem + (int64_t)v * Qm + c);
    for (int c = lane; c < Qa; c += 32) dst_mail[(int64_t)v * Qa + c] = __ldg(src_mail + (int64_t)v * Qa + c);
    if (lane == 0) {
      dst_mem_ts[v] = __ldg(src_mem_ts + v);
      dst_mail_ts[v] = __ldg(src_mail_ts + v);
    }
  }
  const int32_t nc = cur_num ? __ldg(cur_num) : 0;
  for (int64_t i = gtid; i < nc; i += nthreads) save_nodes[i] = __ldg(cur_nodes + i);
  if (gtid == 0) *save_num = nc;
}

void launch_catchup(const int32_t* prev_nodes, const int32_t* prev_num, int64_t prev_max, const float* src_mem,
                    const double* src_mem_ts, const float* src_mail, const double* src_mail_ts, float* dst_mem,
                    double* dst_mem_ts, float* dst_mail, double* dst_mail_ts, int32_t mem_dim, int64_t mail_stride,
                    const int32_t* cur_nodes, const int32_t* cur_num, int64_t cur_max, int32_t* save_nodes,
                    int32_t* save_num, cudaStream_t s) {
  const int threads = 256;
  const int64_t work = prev_max * 32 > cur_max ? prev_max * 32 : cur_max;
  launch_k(k_catchup, dim3(grid_for(work > 0 ? work : 1, threads, 4)), dim3(threads), 0, s, 1, prev_nodes, prev_num,
           (const float4*)src_mem, src_mem_ts, (const float4*)src_mail, src_mail_ts, (float4*)dst_mem, dst_mem_ts,
           (float4*)dst_mail, dst_mail_ts, mem_dim / 4, (int32_t)(mail_stride / 4), cur_nodes, cur_num, save_nodes,
           save_num);
}

// Zero-copy read-back (e2e): the first *num rows of two device arrays straight
// into mapped pinned host memory over PCIe, and *num itself.  Only the rows
// that exist cross the bus (a fixed-size memcpy would move max rows).
__global__ void __launch_bounds__(256) k_rows_to_host(const int32_t* __restrict__ num, int32_t* host_num,
                                                      const uint4* __restrict__ a, uint4* host_a, int64_t a_row_bytes,
                                                      const uint4* __restrict__ b, uint4* host_b,
                                                      int64_t b_row_bytes) {
  const int32_t n = __ldg(num);
  // whole 16-byte words covering the first n rows (the host buffers hold max rows)
  const int64_t na = ((int64_t)n * a_row_bytes + 15) / 16, nt = na + ((int64_t)n * b_row_bytes + 15) / 16;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nt; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < na) host_a[i] = __ldg(a + i);
    else host_b[i - na] = __ldg(b + (i - na));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *host_num = n;
}

void launch_rows_to_host(const int32_t* num, int32_t* host_num, const void* a, void* host_a, int64_t a_row_bytes,
                         const void* b, void* host_b, int64_t b_row_bytes, int64_t max_rows, cudaStream_t s) {
  const int threads = 256;
  const int64_t work = max_rows * (a_row_bytes + b_row_bytes) / 16;
  launch_k(k_rows_to_host, dim3(grid_for(work > 0 ? work : 1, threads, 4)), dim3(threads), 0, s, 1, num, host_num,
           (const uint4*)a, (uint4*)host_a, a_row_bytes, (const uint4*)b, (uint4*)host_b, b_row_bytes);
}

}  // namespace mspipe
