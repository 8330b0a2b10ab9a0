// apan.cu — row F3, the APAN updater (trained "modified from TGL";
// "RNN as the memory update function while incorporating an
// attention mechanism ... asynchronous propagation").  Readings F3-4..F3-8
// (oracle/apan.py):
//   mailbox = a ring of S_mb mails per node (rows [N, S_mb, Dm], times,
//   next slot, filled count); the message of winner w is the attention
//   average of its filled slots, q = W_q S.mem[w], k_s = W_k mail_s,
//   α = softmax(q·k / √M); x = [Σ α mail ‖ cos(ω Δt + ϕ)] feeds the GRU GEMM
//   (k_gru_tc, deferred-mailbox handle: the commit writes h' and mem_ts);
//   after the commit, w's mail [h'_w ‖ h'_o ‖ e] is delivered to w and to its
//   sampled neighbours, the latest key p (F + 1) + s winning per node.
// The projections are plain GEMMs (cuBLAS SGEMM, fp32): q of the winners per
// batch, and k = W_k mail ONCE per delivered mail (a key ring beside the mail
// ring: a mail is read by up to S_mb later updates, its key never changes);
// the per-winner softmax + operand build (mails read straight from the ring)
// and the delivery are kernels here.
#include <cublas_v2.h>

#include "internal.cuh"
#include "tc_layout.cuh"

using namespace mspipe;

namespace {

__device__ __forceinline__ int64_t gw() { return ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; }
__device__ __forceinline__ int64_t nw() { return ((int64_t)gridDim.x * blockDim.x) >> 5; }

// row of winner pair p in the prep's root layout (snapshot rows: times `step`)
__device__ __forceinline__ int64_t root_row(int32_t p, int64_t B) { return (p & 1) ? B + (p >> 1) : (p >> 1); }

// Sw[u] = S.mem[w] (the query input and the GRU hidden input of winner u)
__global__ void k_apan_gather(int64_t B, int32_t M, const int32_t* __restrict__ num,
                              const int32_t* __restrict__ winner, const float* __restrict__ snap_mem, int64_t step,
                              float* Sw) {
  const int lane = threadIdx.x & 31;
  const int32_t U = __ldg(num);
  for (int64_t u = gw(); u < 2 * B; u += nw()) {
    const float* row = snap_mem + root_row(u < U ? __ldg(winner + u) : 0, B) * step * M;
    for (int32_t k = lane; k < M; k += 32) Sw[u * M + k] = u < U ? __ldg(row + k) : 0.f;
  }
}

// warp per GEMM row u (all rows of the M tiles): softmax over the filled slots
// (lane = slot), then x = [Σ α mail | cos(ω Δt + ϕ) | S.mem[w] | 0] into the
// A-operand images (hi | lo), out_ts[u] = t*
__global__ void __launch_bounds__(256) k_apan_build(GruDesc d, int64_t B, int32_t S, const int32_t* __restrict__ num,
                                                    const int32_t* __restrict__ nodes,
                                                    const int32_t* __restrict__ winner,
                                                    const double* __restrict__ ts,
                                                    const double* __restrict__ snap_ts, int64_t step,
                                                    const int32_t* __restrict__ mb_cnt, const float* __restrict__ mb,
                                                    const float* __restrict__ kb, const float* __restrict__ Sw,
                                                    const float* __restrict__ Q, float* xbuf, double* out_ts) {
  __shared__ float sal[8][32];  // the warp's α (lane = slot)
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int32_t U = __ldg(num);
  const int32_t M = d.M, nchunks = d.Kpad / tc::kKC;
  const int64_t rows = (int64_t)((U + tc::kM - 1) / tc::kM) * tc::kM;
  const float scale = rsqrtf((float)M);
  for (int64_t u = gw(); u < rows; u += nw()) {
    if (u >= U) {
      for (int32_t k = lane; k < d.Kpad; k += 32) tc::store_a(xbuf, nchunks, (int32_t)u, k, 0.f);
      continue;
    }
    const int32_t p = __ldg(winner + u), v = __ldg(nodes + u);
    const int32_t c = __ldg(mb_cnt + v);
    float e = -INFINITY;
    if (lane < c) {
      float acc = 0.f;
      const float* q = Q + u * M;
      const float* kr = kb + ((int64_t)v * S + lane) * M;  // k_s = W_k mail_s, cached at delivery
      for (int32_t k = 0; k < M; ++k) acc += __ldg(q + k) * __ldg(kr + k);
      e = acc * scale;
    }
    float mx = e;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float ex = lane < c ? expf(e - mx) : 0.f;
    float den = ex;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
    __syncwarp();
    sal[wib][lane] = lane < c ? ex / den : 0.f;
    __syncwarp();
    const double t = __ldg(ts + (p >> 1));
    const float dt = (float)(t - __ldg(snap_ts + root_row(p, B) * step));  // Δt (G4)
    for (int32_t k = lane; k < d.Kpad; k += 32) {
      float val = 0.f;
      if (k < d.Dm) {
        for (int32_t s = 0; s < c; ++s) val += sal[wib][s] * __ldg(mb + ((int64_t)v * S + s) * d.Dm + k);
      } else if (k < d.Dx) {
        const int32_t q = k - d.Dm;
        val = time_cos(fmaf(__ldg(d.time_w + q), dt, __ldg(d.time_b + q)));
      } else if (k < d.K) {
        val = __ldg(Sw + u * M + (k - d.Dx));
      }
      tc::store_a(xbuf, nchunks, (int32_t)u, k, val);
    }
    if (lane == 0) out_ts[u] = t;
  }
}

// F3-7: mail rows of the winners from the committed memories
__global__ void k_apan_mail(int64_t B, int32_t M, int32_t He, const int32_t* __restrict__ num,
                            const int32_t* __restrict__ nodes, const int32_t* __restrict__ winner,
                            const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                            const float* __restrict__ ef, const float* __restrict__ mem, float* mails) {
  const int lane = threadIdx.x & 31;
  const int32_t U = __ldg(num);
  const int32_t Dm = 2 * M + He;
  for (int64_t u = gw(); u < U; u += nw()) {
    const int32_t p = __ldg(winner + u), ev = p >> 1;
    const int32_t w = __ldg(nodes + u), o = (p & 1) ? __ldg(src + ev) : __ldg(dst + ev);
    float* out = mails + u * Dm;
    for (int32_t k = lane; k < Dm; k += 32)
      out[k] = k < M ? __ldg(mem + (int64_t)w * M + k)
                     : k < 2 * M ? __ldg(mem + (int64_t)o * M + (k - M)) : __ldg(ef + (int64_t)ev * He + (k - 2 * M));
  }
}

// F3-8, candidate (u, s): target = winner u's node (s = 0) or its root's
// neighbour s - 1; key = p (F + 1) + s.  pass 0: atomicMax into best[v];
// pass 1: the candidate holding best[v] writes its mail into v's next slot
__global__ void k_apan_deliver(int64_t B, int32_t F, int32_t S, int32_t Dm, int32_t M, int pass,
                               const int32_t* __restrict__ num, const int32_t* __restrict__ nodes,
                               const int32_t* __restrict__ winner, const int32_t* __restrict__ nbr,
                               const int32_t* __restrict__ cnt, const double* __restrict__ ts,
                               const float* __restrict__ mails, const float* __restrict__ keys, int32_t* best,
                               float* mb, float* kb, double* mb_ts, int32_t* mb_pos, int32_t* mb_cnt) {
  const int lane = threadIdx.x & 31;
  const int32_t U = __ldg(num);
  for (int64_t w = gw(); w < (int64_t)U * (F + 1); w += nw()) {
    const int64_t u = w / (F + 1);
    const int32_t s = (int32_t)(w % (F + 1));
    const int32_t p = __ldg(winner + u);
    const int64_t r = root_row(p, B);
    int32_t v = -1;
    if (s == 0) v = __ldg(nodes + u);
    else if (s - 1 < __ldg(cnt + r)) v = __ldg(nbr + r * F + (s - 1));
    if (v < 0) continue;
    const int32_t key = p * (F + 1) + s;
    if (pass == 0) {
      if (lane == 0) atomicMax(best + v, key);
      continue;
    }
    int win = 0, pos = 0;
    if (lane == 0 && best[v] == key) {
      win = 1;
      pos = mb_pos[v];
      best[v] = -1;
      mb_pos[v] = (pos + 1) % S;
      mb_cnt[v] = min(mb_cnt[v] + 1, S);
      mb_ts[(int64_t)v * S + pos] = __ldg(ts + (p >> 1));
    }
    win = __shfl_sync(0xffffffffu, win, 0);
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (!win) continue;
    float* out = mb + ((int64_t)v * S + pos) * Dm;
    for (int32_t k = lane; k < Dm; k += 32) out[k] = __ldg(mails + u * Dm + k);
    float* ko = kb + ((int64_t)v * S + pos) * M;
    for (int32_t k = lane; k < M; k += 32) ko[k] = __ldg(keys + u * M + k);
  }
}

unsigned blocks_for(int64_t warps) {
  int64_t b = (warps * 32 + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (b > cap) b = cap;
  return (unsigned)(b < 1 ? 1 : b);
}

cublasStatus_t gemm_nt(cublasHandle_t h, int64_t m, int64_t n, int64_t k, const float* A, const float* B, float* C) {
  // row-major C[m, n] = A[m, k] B[n, k]^T
  const float one = 1.f, zero = 0.f;
  return cublasSgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)n, (int)m, (int)k, &one, B, (int)k, A, (int)k, &zero, C,
                     (int)n);
}

}  // namespace

struct mspipe_apan {
  int64_t num_nodes, max_events;
  int32_t M, He, Dm, S;
  float *w_q, *w_k;  // device copies [M, M], [M, Dm]
  float *mb;         // caller-owned mailbox tables
  double* mb_ts;
  int32_t *mb_pos, *mb_cnt;
  float* kb;  // key ring [N, S, M]: k = W_k mail, computed once when the mail is delivered
  float *Sw, *Q, *mails, *keys;
  int32_t* best;
  void* blas_ws;
  cublasHandle_t blas;
};

static void apan_free(mspipe_apan* a) {
  if (!a) return;
  void* bufs[] = {a->w_q, a->w_k, a->kb, a->Sw, a->Q, a->mails, a->keys, a->best, a->blas_ws};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (a->blas) cublasDestroy(a->blas);
  delete a;
}

mspipe_status mspipe_apan_create(mspipe_apan** out, int64_t num_nodes, int32_t mem_dim, int32_t edge_dim,
                                 int32_t slots, int64_t max_events, const float* w_q, const float* w_k, float* mb,
                                 double* mb_ts, int32_t* mb_pos, int32_t* mb_cnt, void* stream) {
  if (!out) return fail(MSPIPE_EINVAL, "apan_create: out is NULL");
  *out = nullptr;
  if (num_nodes <= 0 || mem_dim <= 0 || edge_dim < 0 || slots < 1 || slots > 32 || max_events < 1 ||
      max_events > 8192)
    return fail(MSPIPE_EINVAL, "apan_create: num_nodes=%lld mem_dim=%d slots=%d (1..32) max_events=%lld",
                (long long)num_nodes, mem_dim, slots, (long long)max_events);
  if (!w_q || !w_k || !mb || !mb_ts || !mb_pos || !mb_cnt) return fail(MSPIPE_EINVAL, "apan_create: NULL pointer");
  mspipe_apan* a = new mspipe_apan();
  a->num_nodes = num_nodes;
  a->max_events = max_events;
  a->M = mem_dim;
  a->He = edge_dim;
  a->Dm = 2 * mem_dim + edge_dim;
  a->S = slots;
  a->mb = mb;
  a->mb_ts = mb_ts;
  a->mb_pos = mb_pos;
  a->mb_cnt = mb_cnt;
  const int64_t R = 2 * max_events;
  cudaError_t e = cudaMalloc(&a->w_q, sizeof(float) * (size_t)mem_dim * mem_dim);
  if (e == cudaSuccess) e = cudaMalloc(&a->w_k, sizeof(float) * (size_t)mem_dim * a->Dm);
  if (e == cudaSuccess) e = cudaMalloc(&a->kb, sizeof(float) * (size_t)(num_nodes * slots * mem_dim));
  if (e == cudaSuccess) e = cudaMalloc(&a->keys, sizeof(float) * (size_t)(R * mem_dim));
  if (e == cudaSuccess) e = cudaMalloc(&a->Sw, sizeof(float) * (size_t)(R * mem_dim));
  if (e == cudaSuccess) e = cudaMalloc(&a->Q, sizeof(float) * (size_t)(R * mem_dim));
  if (e == cudaSuccess) e = cudaMalloc(&a->mails, sizeof(float) * (size_t)(R * a->Dm));
  if (e == cudaSuccess) e = cudaMalloc(&a->best, sizeof(int32_t) * (size_t)num_nodes);
  constexpr size_t kWs = 16u << 20;
  if (e == cudaSuccess) e = cudaMalloc(&a->blas_ws, kWs);
  cudaStream_t s = (cudaStream_t)stream;
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(a->w_q, w_q, sizeof(float) * (size_t)mem_dim * mem_dim, cudaMemcpyDefault, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(a->w_k, w_k, sizeof(float) * (size_t)mem_dim * a->Dm, cudaMemcpyDefault, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(a->best, 0xff, sizeof(int32_t) * (size_t)num_nodes, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(a->kb, 0, sizeof(float) * (size_t)(num_nodes * slots * mem_dim), s);
  if (e != cudaSuccess) {
    apan_free(a);
    return cuda_status(e, "apan_create");
  }
  if (cublasCreate(&a->blas) != CUBLAS_STATUS_SUCCESS ||
      cublasSetMathMode(a->blas, CUBLAS_DEFAULT_MATH) != CUBLAS_STATUS_SUCCESS ||
      cublasSetWorkspace(a->blas, a->blas_ws, kWs) != CUBLAS_STATUS_SUCCESS) {
    a->blas = nullptr;
    apan_free(a);
    return fail(MSPIPE_ECUDA, "apan_create: cuBLAS");
  }
  *out = a;
  return MSPIPE_OK;
}

mspipe_status mspipe_apan_destroy(mspipe_apan* a) {
  apan_free(a);
  return MSPIPE_OK;
}

mspipe_status mspipe_message_build_apan(mspipe_apan* a, const mspipe_gru* gru, const double* ts, int64_t num_events,
                                        const float* snap_mem, const double* snap_mem_ts, int64_t snap_step,
                                        const int32_t* nodes, const int32_t* winner, const int32_t* num_unique,
                                        double* out_ts, void* workspace, size_t ws_bytes, void* stream) {
  if (!a || !gru) return fail(MSPIPE_EINVAL, "message_build_apan: NULL handle");
  if (gru->precision != MSPIPE_FP32_3XTF32 || gru->d.mailbox != MSPIPE_MAILBOX_DEFERRED ||
      gru->d.cell != MSPIPE_CELL_GRU)
    return fail(MSPIPE_EUNSUPPORTED, "message_build_apan: needs a deferred-mailbox GRUCell 3xTF32 updater");
  if (gru->d.M != a->M || gru->d.Dm != a->Dm)
    return fail(MSPIPE_EINVAL, "message_build_apan: updater dims differ from the mailbox's");
  if (num_events < 0 || num_events > a->max_events || num_events > gru->max_events || snap_step < 1)
    return fail(MSPIPE_EINVAL, "message_build_apan: num_events=%lld", (long long)num_events);
  if (num_events == 0) return MSPIPE_OK;
  if (!ts || !snap_mem || !snap_mem_ts || !nodes || !winner || !num_unique || !out_ts || !workspace)
    return fail(MSPIPE_EINVAL, "message_build_apan: null input/output");
  if (ws_bytes < mspipe_gru_workspace_size(gru, num_events))
    return fail(MSPIPE_EINVAL, "message_build_apan: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t B = num_events, R = 2 * B;
  k_apan_gather<<<blocks_for(R), 256, 0, s>>>(B, a->M, num_unique, winner, snap_mem, snap_step, a->Sw);
  if (cublasSetStream(a->blas, s) != CUBLAS_STATUS_SUCCESS ||
      cublasSetWorkspace(a->blas, a->blas_ws, 16u << 20) != CUBLAS_STATUS_SUCCESS ||
      gemm_nt(a->blas, R, a->M, a->M, a->Sw, a->w_q, a->Q) != CUBLAS_STATUS_SUCCESS)
    return fail(MSPIPE_ECUDA, "message_build_apan: cuBLAS");
  const int64_t rows = (R + tc::kM - 1) / tc::kM * tc::kM;
  k_apan_build<<<blocks_for(rows), 256, 0, s>>>(gru->d, B, a->S, num_unique, nodes, winner, ts, snap_mem_ts, snap_step,
                                                a->mb_cnt, a->mb, a->kb, a->Sw, a->Q, (float*)workspace, out_ts);
  return cuda_status(cudaGetLastError(), "message_build_apan: launch");
}

mspipe_status mspipe_apan_deliver(mspipe_apan* a, mspipe_memory* st, int64_t commit_version, const int32_t* src,
                                  const int32_t* dst, const double* ts, const float* edge_feat, int64_t num_events,
                                  const int32_t* nodes, const int32_t* winner, const int32_t* num_unique,
                                  const int32_t* nbr, const int32_t* cnt, int32_t fanout, void* stream) {
  if (!a || !st) return fail(MSPIPE_EINVAL, "apan_deliver: NULL handle");
  if (num_events < 0 || num_events > a->max_events || fanout < 0 || fanout > 31)
    return fail(MSPIPE_EINVAL, "apan_deliver: num_events=%lld fanout=%d", (long long)num_events, fanout);
  if (num_events == 0) return MSPIPE_OK;
  if (!src || !dst || !ts || (a->He > 0 && !edge_feat) || !nodes || !winner || !num_unique ||
      (fanout > 0 && (!nbr || !cnt)))
    return fail(MSPIPE_EINVAL, "apan_deliver: null input");
  float* mem = nullptr;
  mspipe_status rc = mspipe_memory_tables(st, commit_version, &mem, nullptr, nullptr, nullptr);
  if (rc != MSPIPE_OK) return rc;
  if (mspipe_memory_local_rows(st) != a->num_nodes)
    return fail(MSPIPE_EUNSUPPORTED, "apan_deliver: sharded memory (world > 1) is not supported");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t B = num_events, R = 2 * B;
  k_apan_mail<<<blocks_for(R), 256, 0, s>>>(B, a->M, a->He, num_unique, nodes, winner, src, dst, edge_feat, mem,
                                            a->mails);
  // the key of every new mail, once (rows >= U: stale but never delivered)
  if (cublasSetStream(a->blas, s) != CUBLAS_STATUS_SUCCESS ||
      cublasSetWorkspace(a->blas, a->blas_ws, 16u << 20) != CUBLAS_STATUS_SUCCESS ||
      gemm_nt(a->blas, R, a->M, a->Dm, a->mails, a->w_k, a->keys) != CUBLAS_STATUS_SUCCESS)
    return fail(MSPIPE_ECUDA, "apan_deliver: cuBLAS");
  for (int pass = 0; pass < 2; ++pass)
    k_apan_deliver<<<blocks_for(R * (fanout + 1)), 256, 0, s>>>(B, fanout, a->S, a->Dm, a->M, pass, num_unique,
                                                                 nodes, winner, nbr, cnt, ts, a->mails, a->keys,
                                                                 a->best, a->mb, a->kb, a->mb_ts, a->mb_pos,
                                                                 a->mb_cnt);
  return cuda_status(cudaGetLastError(), "apan_deliver: launch");
}

mspipe_status mspipe_apan_refresh_keys(mspipe_apan* a, void* stream) {
  if (!a) return fail(MSPIPE_EINVAL, "apan_refresh_keys: NULL handle");
  cudaStream_t s = (cudaStream_t)stream;
  if (cublasSetStream(a->blas, s) != CUBLAS_STATUS_SUCCESS ||
      cublasSetWorkspace(a->blas, a->blas_ws, 16u << 20) != CUBLAS_STATUS_SUCCESS ||
      gemm_nt(a->blas, a->num_nodes * a->S, a->M, a->Dm, a->mb, a->w_k, a->kb) != CUBLAS_STATUS_SUCCESS)
    return fail(MSPIPE_ECUDA, "apan_refresh_keys: cuBLAS");
  return MSPIPE_OK;
}
