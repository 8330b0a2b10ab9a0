// prep.cu — A1 + A2 + A3 of one batch in ONE launch (mspipe_memory_prep).
//
// The per-batch prep is three latency-bound steps whose separate launches
// cost more than their work.  k_prep fuses them:
//   block 0       : A2, the block dedup of the 2B pairs (dedup.cuh);
//   blocks 1..    : one warp per root of the batch ([src | dst | neg]):
//                   A1 (warp_recent_end: 33-ary search of the T-CSR row) and,
//                   with the subgraph ids still in registers, A3: the warp
//                   gathers the 𝒩+1 state rows of its subgraph (root first)
//                   straight into the dense snapshot buffers.
// Reading the tables here is the "fetch": the stage orders this launch between
// write-back(i-1-k) and write-back(i-k) (Eq. 2).
#include "internal.cuh"

namespace mspipe {
#ifdef MSPIPE_PHASES
// debug: per-block phase times of the last k_prep launch (globaltimer ns)
__device__ unsigned long long g_pphase[8192][6];
__device__ __forceinline__ void pphase(int i) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  atomicMax(&g_pphase[blockIdx.x][i], t);
}
#define PPHASE(i) pphase(i)
#define DEDUP_MARK(i) \
  if (threadIdx.x == 0) pphase(i)
#else
#define PPHASE(i)
#endif

}  // namespace mspipe

#include "dedup.cuh"

namespace mspipe {

constexpr int kPrepThreads = 512;
// two blocks per SM (<= 64 registers): at GDELT's 12,000 roots the latency-bound
// root warps need the occupancy (one block per SM ran the roots in ~5 waves), and
// a k_prep block then still fits beside a k_gru_tc CTA
#ifndef MSPIPE_PREP_MINB
#define MSPIPE_PREP_MINB 2
#endif
constexpr int kPrepWarps = kPrepThreads / 32;

struct PrepArgs {
  Tcsr g;
  const int32_t* src;
  const int32_t* dst;
  const int32_t* neg;
  const double* ts;
  int64_t B;
  int32_t F;
  int32_t* out_nbr;
  int32_t* out_eid;
  double* out_ts;
  float* out_dt;
  int32_t* out_cnt;
  int32_t* out_sub;
  int32_t* gscratch;
  int32_t* out_nodes;
  int32_t* out_winner;
  int32_t* out_num;
  const float4* mem;
  const double* mem_ts;
  int32_t Qm;
  const float4* mail;
  const double* mail_ts;
  int32_t Qa;
  float4* out_mem;
  double* out_mem_ts;
  float4* out_mail;
  double* out_mail_ts;
  int32_t* stamp;  // optional: stamp[winner node] = stamp_iter (double-buffered state)
  int32_t stamp_iter;
  CatchUp cu;      // optional (cu.stamp != nullptr): the next commit's catch-up rows
  int32_t Qcu;     // float4 per mail row of the state tables (catch-up)
  int32_t dedup;   // 1: block 0 deduplicates (A2); 0: no dedup block
  int64_t* hint;   // optional [num_nodes]: per-node search start (warp_recent_sample)
  int32_t stream_nbr;  // 1: neighbour rows stored evict-first (read only by a later training stage)
};

// copy `nrows` table rows (ids held by lanes 0..nrows-1, -1 = zero row) of Q
// float4 each into dst rows base..base+nrows-1; kU loads in flight per lane.
__device__ __forceinline__ void warp_gather_rows(const float4* __restrict__ tab, int32_t Q, int32_t my_id,
                                                 int nrows, float4* __restrict__ dst, int64_t dst_row0,
                                                 int lane, int stream_tail = 0) {
  // kU float4 loads in flight per lane before their stores: the whole subgraph
  // (11 rows x 25 float4 for M = 100) in one dependent round instead of three
#ifndef MSPIPE_PREP_KU
#define MSPIPE_PREP_KU 9
#endif
  constexpr int kU = MSPIPE_PREP_KU;
  const int total = nrows * Q;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  // (row s, column c) of this lane's element; the next one is 32 elements on:
  // advance by (q32, r32) with one conditional wrap instead of a division per load
  int s = lane / Q, c = lane - (lane / Q) * Q;
  const int q32 = 32 / Q, r32 = 32 - q32 * Q;
  for (int base = 0; base < total; base += 32 * kU) {
    float4 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int idx = base + u * 32 + lane;
      const int32_t id = __shfl_sync(0xffffffffu, my_id, s < nrows ? s : 0);
      v[u] = (idx < total && id >= 0) ? __ldg(tab + (int64_t)id * Q + c) : z;
      s += q32;
      c += r32;
      if (c >= Q) {
        c -= Q;
        ++s;
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int idx = base + u * 32 + lane;
      if (idx < total) {
        // rows >= 1 (the neighbours) with stream_tail: st.global.cs (evict-first), so the
        // 3B·𝒩 rows nobody reads in this step do not push the root rows and tables out of L2
        if (stream_tail && idx >= Q) __stcs(dst + dst_row0 * Q + idx, v[u]);
        else dst[dst_row0 * Q + idx] = v[u];
      }
    }
  }
}

template <bool kSmem>
__global__ void __launch_bounds__(kPrepThreads, MSPIPE_PREP_MINB) k_prep(PrepArgs a) {
  extern __shared__ int32_t sscratch[];
  if (threadIdx.x == 0) PPHASE(0);
  if (a.dedup && blockIdx.x == 0) {
    block_dedup<kPrepThreads, kSmem>(a.src, a.dst, a.B, a.gscratch, sscratch, a.g.num_nodes, a.out_nodes,
                                     a.out_winner, a.out_num);
    if (threadIdx.x == 0) PPHASE(2);
    if (a.stamp) {
      __syncthreads();  // out_nodes / out_winner / out_num written by this block
      const int32_t U = *a.out_num;
      for (int32_t u = threadIdx.x; u < U; u += kPrepThreads) a.stamp[a.out_nodes[u]] = a.stamp_iter;
    }
    if (threadIdx.x == 0) PPHASE(1);
    return;
  }
  const int lane = threadIdx.x & 31;
  const int64_t R = 3 * a.B;
  const int F = a.F, F1 = a.F + 1;
  const int64_t nwarps = (int64_t)(gridDim.x - a.dedup) * kPrepWarps;
  const int64_t wid = (int64_t)(blockIdx.x - a.dedup) * kPrepWarps + (threadIdx.x >> 5);
  for (int64_t r = wid; r < R; r += nwarps) {
    const int64_t role = r / a.B, ev = r - role * a.B;
    const int32_t v = role == 0 ? __ldg(a.src + ev) : (role == 1 ? __ldg(a.dst + ev) : __ldg(a.neg + ev));
    const double tq = __ldg(a.ts + ev);
    int64_t beg;
    int32_t nbs, eis;
    double tss;
    const int64_t end = a.hint ? warp_recent_sample_hinted(a.g, v, tq, lane, F, &beg, &nbs, &eis, &tss, a.hint)
                               : warp_recent_sample(a.g, v, tq, lane, F, &beg, &nbs, &eis, &tss);
    const int32_t cnt = (int32_t)min64(end - beg, (int64_t)F);
    // A1 outputs; lane s < F = slot s (newest first); lane s in [1, F] also holds subgraph id s
    if (lane < F) {
      const int64_t o = r * F + lane;
      const bool ok = lane < cnt;
      a.out_nbr[o] = ok ? nbs : -1;
      a.out_eid[o] = ok ? eis : -1;
      a.out_ts[o] = ok ? tss : 0.0;
      a.out_dt[o] = ok ? (float)(tq - tss) : 0.0f;
    }
    const int32_t nb_prev = __shfl_up_sync(0xffffffffu, nbs, 1);  // slot lane-1 -> subgraph id lane
    int32_t id = lane == 0 ? v : -1;
    if (lane >= 1 && lane <= F && lane - 1 < cnt) id = nb_prev;
    if (lane == 0) a.out_cnt[r] = cnt;
    if (lane <= F) a.out_sub[r * F1 + lane] = id;
    // A3: the subgraph's snapshot rows (pads and out-of-range ids give zero rows)
    const int32_t gid = (id >= 0 && id < a.g.num_nodes) ? id : -1;
    if (lane <= F) {
      a.out_mem_ts[r * F1 + lane] = gid >= 0 ? __ldg(a.mem_ts + gid) : 0.0;
      if (a.out_mail_ts) a.out_mail_ts[r * F1 + lane] = gid >= 0 ? __ldg(a.mail_ts + gid) : 0.0;
    }
    warp_gather_rows(a.mem, a.Qm, gid, F1, a.out_mem, r * F1, lane, a.stream_nbr);
    if (a.Qa > 0) warp_gather_rows(a.mail, a.Qa, gid, F1, a.out_mail, r * F1, lane);
  }
  if (lane == 0) PPHASE(1);
  if (a.cu.stamp) {  // double-buffered: rows of the previous commit, after this warp's roots
    const int32_t np = __ldg(a.cu.prev_num);
    const int64_t r0 = wid + (R - wid + nwarps - 1) / nwarps * nwarps;  // this warp's first item >= R
    for (int64_t r = r0; r < R + np; r += nwarps) {
      const int32_t v = __ldg(a.cu.prev_nodes + (r - R));
      if (__ldg(a.cu.stamp + v) != a.cu.iter) catchup_row(a.cu, v, a.Qm, a.Qcu, lane);
    }
  }
  if (threadIdx.x == 0) PPHASE(4);
}

cudaError_t launch_prep(const Tcsr& g, const int32_t* src, const int32_t* dst, const int32_t* neg,
                        const double* ts, int64_t num_events, int32_t fanout, int32_t* out_nbr,
                        int32_t* out_eid, double* out_ts, float* out_dt, int32_t* out_cnt, int32_t* out_sub,
                        int32_t* scratch, int32_t* out_nodes, int32_t* out_winner, int32_t* out_num,
                        const float* mem, const double* mem_ts, int32_t mem_dim, const float* mail,
                        const double* mail_ts, int64_t mail_stride, float* out_mem, double* out_mem_ts,
                        float* out_mail, double* out_mail_ts, cudaStream_t s, int32_t* stamp,
                        int32_t stamp_iter, const CatchUp* cu, int64_t* hint) {
  PrepArgs a{g, src, dst, neg, ts, num_events, fanout, out_nbr, out_eid, out_ts, out_dt, out_cnt, out_sub,
             scratch, out_nodes, out_winner, out_num, (const float4*)mem, mem_ts, mem_dim / 4,
             (const float4*)mail, mail_ts, out_mail ? (int32_t)(mail_stride / 4) : 0, (float4*)out_mem, out_mem_ts,
             (float4*)out_mail, out_mail ? out_mail_ts : nullptr, stamp, stamp_iter, CatchUp{},
             (int32_t)(mail_stride / 4)};
  if (cu) a.cu = *cu;
  a.hint = hint;
  // neighbour rows evict-first when a batch's are large (GDELT: 49 MB of rows that only a
  // later training stage reads; measured 96.6 vs 93.1 M events/s), write-back for small
  // batches (wiki: neutral to -1.5 %); MSPIPE_PREP_STCS=0/1 forces it
  {
    const int forced = env_int("MSPIPE_PREP_STCS", -1);
    const int64_t nbr_bytes = 3 * num_events * fanout * (int64_t)(mem_dim * 4 + 8);
    a.stream_nbr = forced >= 0 ? forced : (nbr_bytes > (16ll << 20) ? 1 : 0);
  }
  a.dedup = out_num != nullptr;
  int64_t blocks = (3 * num_events + kPrepWarps - 1) / kPrepWarps;
  // one wave of the two resident blocks per SM; the root warps grid-stride
  // (block 0, the dedup, counts against the wave: 297 blocks on 296 slots left
  // one root block waiting ~13 us for a slot at GDELT)
  const int64_t cap = (int64_t)num_sms() * env_int("MSPIPE_PREP_BPS", 2) - (a.dedup ? 1 : 0);
  if (blocks > cap) blocks = cap;
  if (!a.dedup) return launch_k(k_prep<false>, dim3((unsigned)blocks), dim3(kPrepThreads), 0, s, 1, a);
  blocks += 1;  // block 0: dedup
  if (g.num_nodes <= kDedupSmemNodes && env_int("MSPIPE_PREP_SMEM", 1)) {
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(k_prep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(kDedupSmemNodes * sizeof(int32_t)));
      if (e != cudaSuccess) return e;
      attr = true;
    }
    return launch_k(k_prep<true>, dim3((unsigned)blocks), dim3(kPrepThreads), g.num_nodes * sizeof(int32_t), s, 1,
                    a);
  }
  return launch_k(k_prep<false>, dim3((unsigned)blocks), dim3(kPrepThreads), 0, s, 1, a);
}

}  // namespace mspipe

#ifdef MSPIPE_PHASES
extern "C" __attribute__((visibility("default"))) int mspipe_debug_prep_phases(void* host, int n, int reset) {
  if (reset) {
    static unsigned long long zero[8192][6];
    return (int)cudaMemcpyToSymbol(mspipe::g_pphase, zero, sizeof(zero));
  }
  return (int)cudaMemcpyFromSymbol(host, mspipe::g_pphase, sizeof(unsigned long long) * 6 * n);
}
#endif
