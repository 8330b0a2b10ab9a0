// stale.cu — the C3 statistic of MSPipe §3.2 (Fig. `fig:overlap`): how
// many of the nodes a batch updates were updated again within the last d
// iterations, i.e. would be read stale under staleness k > d (reading F6).
//
// One thread per (event j, role) endpoint v of the stream.  The T-CSR row of v
// lists v's events in stream order, so a binary search on eid finds the entry
// of event j and its predecessor j' (the previous event of v).  Only the first
// occurrence of v in its batch counts (j' outside the batch); it adds one to
// bin d = i - i' (i, i' the 1-based batches of j, j'), or to bin 0 when v has
// no earlier event.  Bins are accumulated in shared memory per block, then
// added to the global int64 histogram (integer atomics: deterministic).
#include "internal.cuh"

namespace mspipe {

constexpr int kStaleThreads = 256;

__global__ void __launch_bounds__(kStaleThreads) k_stale_hist(Tcsr g, const int32_t* __restrict__ src,
                                                              const int32_t* __restrict__ dst, int64_t E,
                                                              int64_t B, int32_t max_d,
                                                              unsigned long long* __restrict__ hist) {
  extern __shared__ unsigned long long sh[];  // [max_d + 2]
  for (int q = threadIdx.x; q < max_d + 2; q += blockDim.x) sh[q] = 0ull;
  __syncthreads();
  const int64_t P = 2 * E;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = p >> 1;
    const int32_t v = (p & 1) ? __ldg(dst + j) : __ldg(src + j);
    if ((p & 1) && v == __ldg(src + j)) continue;  // self-loop: one endpoint
    if (v < 0 || v >= g.num_nodes) {
      raise_dev(MSPIPE_DEVERR_RANGE);
      continue;
    }
    // first position in row(v) with eid >= j (the entry of event j)
    int64_t lo = __ldg(g.indptr + v), hi = __ldg(g.indptr + v + 1);
    const int64_t beg = lo;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(g.eid + mid) < j) lo = mid + 1;
      else hi = mid;
    }
    const int64_t i = j / B + 1;
    int32_t bin;
    if (lo == beg) {
      bin = 0;
    } else {
      const int64_t jp = __ldg(g.eid + lo - 1);
      const int64_t ip = jp / B + 1;
      if (ip == i) continue;  // not v's first event in this batch
      const int64_t d = i - ip;
      bin = d > max_d ? max_d + 1 : (int32_t)d;
    }
    atomicAdd(sh + bin, 1ull);
  }
  __syncthreads();
  for (int q = threadIdx.x; q < max_d + 2; q += blockDim.x)
    if (sh[q]) atomicAdd(hist + q, sh[q]);
}

cudaError_t launch_stale_hist(const Tcsr& g, const int32_t* src, const int32_t* dst, int64_t E, int64_t B,
                              int32_t max_d, unsigned long long* hist, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * (size_t)(max_d + 2), s);
  if (e != cudaSuccess || E == 0) return e;
  int64_t blocks = (2 * E + kStaleThreads - 1) / kStaleThreads;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  return launch_k(k_stale_hist, dim3((unsigned)blocks), dim3(kStaleThreads),
                  sizeof(unsigned long long) * (size_t)(max_d + 2), s, 1, g, src, dst, E, B, max_d, hist);
}

}  // namespace mspipe

// ---------------------------------------------------------------------------
// Row F1 analytics — the staleness error of MSPipe §5.5 (Fig.
// `fig:staleness_error`; Theorem 1's ε_s): for iteration i,
//     ‖x^(i) − s^(i)‖_F  over the batch's update targets w ∈ U_i,
// x = the memory the updater consumed (the stale read s̃ = S_{v(i)}[w], or the
// mitigated ŝ_w of MSPipe-S) and s = the precise memory S_{i−1}[w] of a k = 0
// run of the same stream (reading F7).  Rows come in root layout: target w of
// pair p = 2a + role is root r = role·n + a, its row at base + r·stride·M.
// One block, f64 accumulation in a fixed order (deterministic).
// ---------------------------------------------------------------------------
namespace mspipe {

constexpr int kErrThreads = 256;

__global__ void __launch_bounds__(kErrThreads) k_staleness_error(const int32_t* __restrict__ winner,
                                                                 const int32_t* __restrict__ num, int64_t n,
                                                                 const float* __restrict__ xa, int64_t stride_a,
                                                                 const float* __restrict__ xb, int64_t stride_b,
                                                                 int32_t M, double* __restrict__ out) {
  __shared__ double part[kErrThreads];
  const int32_t U = *num;
  double acc = 0.0;
  for (int64_t q = threadIdx.x; q < (int64_t)U * M; q += kErrThreads) {
    const int64_t u = q / M, c = q - u * M;
    const int32_t p = __ldg(winner + u);
    const int64_t r = (int64_t)(p & 1) * n + (p >> 1);
    const double d = (double)__ldg(xa + r * stride_a * M + c) - (double)__ldg(xb + r * stride_b * M + c);
    acc = fma(d, d, acc);
  }
  part[threadIdx.x] = acc;
  __syncthreads();
  for (int w = kErrThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sqrt(part[0]);
}

cudaError_t launch_staleness_error(const int32_t* winner, const int32_t* num_unique, int64_t num_events,
                                  const float* rows_a, int64_t stride_a, const float* rows_b, int64_t stride_b,
                                  int32_t mem_dim, double* out, cudaStream_t s) {
  return launch_k(k_staleness_error, dim3(1), dim3(kErrThreads), 0, s, 1, winner, num_unique, num_events, rows_a,
                  stride_a, rows_b, stride_b, mem_dim, out);
}

}  // namespace mspipe
