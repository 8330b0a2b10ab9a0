// dedup.cuh — A2 as a block-level device routine (used by k_dedup and k_prep).
//
// Pair p = 2a + role has node src_a (role 0) / dst_a (role 1); the winner of
// node w is max{p} (the most recent message, G6).  Phase 1:
// warp-aggregated atomicMax of p into a node table (__match_any_sync groups
// equal nodes, so a hot node costs one atomic per warp; max is
// order-independent, hence deterministic).  Phase 2: a pair wins iff
// table[node_p] == p; a block scan over contiguous chunks compacts the
// winners in p order.  With kSmem the table lives in shared memory (N <=
// kDedupSmemNodes); otherwise in a self-cleaning global scratch (phase 3 resets
// the touched entries to -1).
#pragma once
#include "internal.cuh"

namespace mspipe {

constexpr int64_t kDedupSmemNodes = 40960;  // node table in shared memory up to 160 KB

template <int NT, bool kSmem>
__device__ __forceinline__ void block_dedup(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                                            int64_t B, int32_t* __restrict__ gscratch, int32_t* sscratch,
                                            int64_t N, int32_t* __restrict__ out_nodes,
                                            int32_t* __restrict__ out_winner, int32_t* __restrict__ out_num) {
  __shared__ int32_t warp_tot[32];
  __shared__ int32_t total_s;
  int32_t* scratch = kSmem ? sscratch : gscratch;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (kSmem) {
    for (int64_t i = tid; i < N; i += NT) sscratch[i] = -1;
    __syncthreads();
  }
  const int64_t P = 2 * B;
  const int64_t Pr = (P + NT - 1) / NT * NT;
  for (int64_t p = tid; p < Pr; p += NT) {
    int32_t node = -1;
    if (p < P) {
      node = (p & 1) ? __ldg(dst + (p >> 1)) : __ldg(src + (p >> 1));
      if (node < 0 || node >= N) {
        raise_dev(MSPIPE_DEVERR_RANGE);
        node = -1;
      }
    }
    const unsigned grp = __match_any_sync(0xffffffffu, node);
    const int leader = 31 - __clz(grp);  // highest lane = largest p of the group
    if (node >= 0 && lane == leader) atomicMax(scratch + node, (int32_t)p);
  }
  if (!kSmem) __threadfence();
  __syncthreads();
  const int64_t C = (P + NT - 1) / NT;  // <= 32: caller guarantees 2B <= 32 * NT
  const int64_t p0 = tid * C;
  uint32_t flags = 0;
  int32_t cnt = 0;
  for (int64_t i = 0; i < C; ++i) {
    const int64_t p = p0 + i;
    if (p >= P) break;
    const int32_t node = (p & 1) ? __ldg(dst + (p >> 1)) : __ldg(src + (p >> 1));
    if (node < 0 || node >= N) continue;
    const int32_t w = kSmem ? sscratch[node] : __ldcg(gscratch + node);
    if (w == (int32_t)p) {
      flags |= 1u << i;
      ++cnt;
    }
  }
  int32_t incl = cnt;  // block exclusive scan of cnt
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const int32_t v = lane < NT / 32 ? warp_tot[lane] : 0;
    int32_t vi = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, vi, d);
      if (lane >= d) vi += y;
    }
    warp_tot[lane] = vi - v;  // exclusive prefix of warp totals
    if (lane == 31) total_s = vi;
  }
  __syncthreads();
  int32_t off = warp_tot[wid] + incl - cnt;
  for (int64_t i = 0; i < C; ++i) {
    if (flags & (1u << i)) {
      const int64_t p = p0 + i;
      out_nodes[off] = (p & 1) ? __ldg(dst + (p >> 1)) : __ldg(src + (p >> 1));
      out_winner[off] = (int32_t)p;
      ++off;
    }
  }
  if (!kSmem) {
    __syncthreads();  // all scratch reads are done before the reset
    for (int64_t i = 0; i < C; ++i) {
      if (flags & (1u << i)) {
        const int64_t p = p0 + i;
        const int32_t node = (p & 1) ? __ldg(dst + (p >> 1)) : __ldg(src + (p >> 1));
        gscratch[node] = -1;
      }
    }
  }
  if (tid == 0) *out_num = total_s;
}

}  // namespace mspipe
