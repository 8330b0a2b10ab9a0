// features.cu — row F2: the feature-fetch stage ("Fetch feature", stage 2 of
// the paper's pipeline) for the sampled subgraphs: the
// node-feature rows of the 3B(𝒩+1) subgraph nodes (GDELT |d_v| = 413,
// Table `tab:datasets` P:L395) and the edge-feature rows of the 3B·𝒩 sampled
// links.  Pure gather, HBM-bound: one warp per output row, 16-byte
// vector copies with four loads in flight per lane, grid sized to the SMs.
#include "internal.cuh"

namespace mspipe {

constexpr int kFeatThreads = 256;

// copy table row `id` (or zeros for id < 0) of `n4` float4 into dst
__device__ __forceinline__ void warp_copy_row4(const float4* __restrict__ tab, int64_t id, int32_t n4,
                                               float4* __restrict__ dst, int lane) {
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int base = 0; base < n4; base += 128) {
    float4 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = base + q * 32 + lane;
      v[q] = (c < n4 && id >= 0) ? __ldg(tab + id * n4 + c) : z;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = base + q * 32 + lane;
      if (c < n4) dst[c] = v[q];
    }
  }
}

__device__ __forceinline__ void warp_copy_row1(const float* __restrict__ tab, int64_t id, int32_t n,
                                               float* __restrict__ dst, int lane) {
  for (int c = lane; c < n; c += 32) dst[c] = id >= 0 ? __ldg(tab + id * n + c) : 0.f;
}

__global__ void __launch_bounds__(kFeatThreads) k_feature_fetch(
    const int32_t* __restrict__ sub, const int32_t* __restrict__ eid, int64_t R, int32_t F,
    const float* __restrict__ nfeat, int64_t N, int32_t nstride, const float* __restrict__ efeat, int64_t E,
    int32_t estride, float* __restrict__ out_n, float* __restrict__ out_e) {
  const int lane = threadIdx.x & 31;
  const int64_t rows_n = nfeat ? R * (F + 1) : 0;
  const int64_t rows_e = efeat ? R * F : 0;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < rows_n + rows_e; w += nw) {
    const bool node = w < rows_n;
    const int64_t r = node ? w : w - rows_n;
    int64_t id = node ? __ldg(sub + r) : __ldg(eid + r);
    const int64_t lim = node ? N : E;
    if (id >= lim) {
      raise_dev(MSPIPE_DEVERR_RANGE);
      id = -1;
    }
    const int32_t stride = node ? nstride : estride;
    const float* tab = node ? nfeat : efeat;
    float* dst = (node ? out_n : out_e) + r * stride;
    if ((stride & 3) == 0)
      warp_copy_row4(reinterpret_cast<const float4*>(tab), id, stride >> 2, reinterpret_cast<float4*>(dst), lane);
    else
      warp_copy_row1(tab, id, stride, dst, lane);
  }
}

cudaError_t launch_feature_fetch(const int32_t* sub, const int32_t* eid, int64_t R, int32_t F, const float* nfeat,
                                 int64_t N, int32_t nstride, const float* efeat, int64_t E, int32_t estride,
                                 float* out_n, float* out_e, cudaStream_t s) {
  const int64_t rows = (nfeat ? R * (F + 1) : 0) + (efeat ? R * F : 0);
  if (rows == 0) return cudaSuccess;
  int64_t blocks = (rows * 32 + kFeatThreads - 1) / kFeatThreads;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  return launch_k(k_feature_fetch, dim3((unsigned)blocks), dim3(kFeatThreads), 0, s, 1, sub, eid, R, F, nfeat, N,
                  nstride, efeat, E, estride, out_n, out_e);
}

}  // namespace mspipe
