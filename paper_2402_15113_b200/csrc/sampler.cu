// sampler.cu — A1, the recent-𝒩 temporal neighbour sampler (P:L412, P:L810,
// P:L814).
//
// One warp per root.  The sampler is memory-LATENCY bound (dependent probes
// into the time-sorted row), so the warp searches 33-ary: 32 lanes probe 32
// interior positions of the current range at once and a ballot shrinks the
// range 33x per round.  A row of L entries takes ceil(log33(L / 32)) + 1
// dependent rounds instead of log2(L) (wiki: 1-2, LastFM hot items: 3).  The
// first position with ts >= t_q is `end`; the newest min(fanout, end - beg)
// entries before it are the answer (G15: strict <, ties newest-eid first).
// Lanes s < fanout then read entry end-1-s and write output slot s.
#include "internal.cuh"

namespace mspipe {

template <bool kBatch>
__global__ void __launch_bounds__(256) k_sample_recent(
    Tcsr g, const int32_t* __restrict__ roots, const double* __restrict__ qts,
    const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
    const int32_t* __restrict__ neg, const double* __restrict__ ev_ts, int64_t B, int64_t R,
    int32_t F, int32_t* __restrict__ out_nbr, int32_t* __restrict__ out_eid,
    double* __restrict__ out_ts, float* __restrict__ out_dt, int32_t* __restrict__ out_cnt,
    int32_t* __restrict__ out_sub) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < R; r += nwarps) {
    int32_t v;
    double tq;
    if (kBatch) {
      const int64_t role = r / B, a = r - role * B;
      v = role == 0 ? __ldg(src + a) : (role == 1 ? __ldg(dst + a) : __ldg(neg + a));
      tq = __ldg(ev_ts + a);
    } else {
      v = __ldg(roots + r);
      tq = __ldg(qts + r);
    }
    int64_t beg = 0;
    const int64_t end = warp_recent_end(g, v, tq, lane, &beg);
    const int32_t cnt = (int32_t)min64(end - beg, (int64_t)F);
    for (int s = lane; s < F; s += 32) {  // output slot s = entry end-1-s (newest first)
      const int64_t o = r * F + s;
      if (s < cnt) {
        const int64_t q = end - 1 - s;
        const double tsq = __ldg(g.ts + q);
        out_nbr[o] = __ldg(g.nbr + q);
        out_eid[o] = __ldg(g.eid + q);
        out_ts[o] = tsq;
        out_dt[o] = (float)(tq - tsq);
      } else {
        out_nbr[o] = -1;
        out_eid[o] = -1;
        out_ts[o] = 0.0;
        out_dt[o] = 0.0f;
      }
    }
    if (lane == 0) out_cnt[r] = cnt;
    if (out_sub) {
      // subgraph node list [root, nbr_0 .. nbr_{F-1}] (3B(𝒩+1) nodes per batch)
      for (int s = lane; s <= F; s += 32) {
        const int32_t id = s == 0 ? v : ((s - 1 < cnt) ? __ldg(g.nbr + (end - s)) : -1);
        out_sub[r * (F + 1) + s] = id;
      }
    }
  }
}

void launch_sample(const Tcsr& g, const int32_t* roots, const double* qts, const int32_t* src,
                   const int32_t* dst, const int32_t* neg, const double* ev_ts, int64_t num_events,
                   int64_t num_roots, int32_t fanout, int32_t* out_nbr, int32_t* out_eid,
                   double* out_ts, float* out_dt, int32_t* out_cnt, int32_t* out_sub,
                   cudaStream_t s) {
  const int threads = 256;
  int64_t blocks = (num_roots * 32 + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const int32_t* np = nullptr;
  const double* nd = nullptr;
  if (roots)
    launch_k(k_sample_recent<false>, dim3((unsigned)blocks), dim3(threads), 0, s, 1, g, roots, qts, np, np, np, nd,
             (int64_t)1, num_roots, fanout, out_nbr, out_eid, out_ts, out_dt, out_cnt, out_sub);
  else
    launch_k(k_sample_recent<true>, dim3((unsigned)blocks), dim3(threads), 0, s, 1, g, np, nd, src, dst, neg, ev_ts,
             num_events, num_roots, fanout, out_nbr, out_eid, out_ts, out_dt, out_cnt, out_sub);
}

}  // namespace mspipe
