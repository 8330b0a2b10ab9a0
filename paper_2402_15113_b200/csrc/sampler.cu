// sampler.cu — A1, the recent-𝒩 temporal neighbour sampler (P:L412, P:L810,
// P:L814).  One warp serves 32 roots: each lane bisects its root's
// T-CSR row for the first ts >= t_q (so entries before it are exactly the
// events with ts < t_q, G15), then the warp writes the 32 x fanout output
// block cooperatively so every store instruction is contiguous.
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
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp * 32; base < R; base += nwarps * 32) {
    const int64_t r = base + lane;
    int64_t end = 0;
    int32_t cnt = 0;
    int32_t v = -1;
    double tq = 0.0;
    if (r < R) {
      if (kBatch) {
        const int64_t role = r / B, a = r - role * B;
        v = role == 0 ? __ldg(src + a) : (role == 1 ? __ldg(dst + a) : __ldg(neg + a));
        tq = __ldg(ev_ts + a);
      } else {
        v = __ldg(roots + r);
        tq = __ldg(qts + r);
      }
      if (v >= 0 && v < g.num_nodes) {
        const int64_t beg = __ldg(g.indptr + v);
        int64_t lo = beg, hi = __ldg(g.indptr + v + 1);
        while (lo < hi) {  // lower bound of t_q in the row's non-decreasing ts
          const int64_t mid = (lo + hi) >> 1;
          if (__ldg(g.ts + mid) < tq) lo = mid + 1;
          else hi = mid;
        }
        end = lo;
        cnt = (int32_t)min64(end - beg, (int64_t)F);
      } else {
        raise_dev(MSPIPE_DEVERR_RANGE);
      }
      out_cnt[r] = cnt;
    }
    const int nr = (int)min64(32, R - base);
    const int total = 32 * F;
    for (int idx = lane; idx < total; idx += 32) {
      const int rr = idx / F, slot = idx - rr * F;
      const int64_t e = __shfl_sync(0xffffffffu, end, rr);
      const int32_t c = __shfl_sync(0xffffffffu, cnt, rr);
      const double t = __shfl_sync(0xffffffffu, tq, rr);
      if (rr < nr) {
        const int64_t o = base * F + idx;
        if (slot < c) {
          const int64_t q = e - 1 - slot;
          const double tsq = __ldg(g.ts + q);
          out_nbr[o] = __ldg(g.nbr + q);
          out_eid[o] = __ldg(g.eid + q);
          out_ts[o] = tsq;
          out_dt[o] = (float)(t - tsq);
        } else {
          out_nbr[o] = -1;
          out_eid[o] = -1;
          out_ts[o] = 0.0;
          out_dt[o] = 0.0f;
        }
      }
    }
    if (out_sub) {
      const int F1 = F + 1;
      const int tot1 = 32 * F1;
      for (int idx = lane; idx < tot1; idx += 32) {
        const int rr = idx / F1, slot = idx - rr * F1;
        const int64_t e = __shfl_sync(0xffffffffu, end, rr);
        const int32_t c = __shfl_sync(0xffffffffu, cnt, rr);
        const int32_t vv = __shfl_sync(0xffffffffu, v, rr);
        if (rr < nr) {
          int32_t id;
          if (slot == 0) id = vv;
          else id = (slot - 1 < c) ? __ldg(g.nbr + (e - slot)) : -1;
          out_sub[base * F1 + idx] = id;
        }
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
  const int64_t warps = (num_roots + 31) / 32;
  int64_t blocks = (warps * 32 + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (roots)
    k_sample_recent<false><<<(unsigned)blocks, threads, 0, s>>>(g, roots, qts, nullptr, nullptr, nullptr, nullptr, 1,
                                                                 num_roots, fanout, out_nbr, out_eid, out_ts, out_dt,
                                                                 out_cnt, out_sub);
  else
    k_sample_recent<true><<<(unsigned)blocks, threads, 0, s>>>(g, nullptr, nullptr, src, dst, neg, ev_ts, num_events,
                                                                num_roots, fanout, out_nbr, out_eid, out_ts, out_dt,
                                                                out_cnt, out_sub);
}

}  // namespace mspipe
