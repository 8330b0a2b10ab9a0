// dedup.cuh — A2 as a block-level device routine (used by k_dedup and k_prep).
//
// Pair p = 2a + role has node src_a (role 0) / dst_a (role 1); the winner of
// node w is max{p} (the most recent message, G6).  Phase 1:
// warp-aggregated atomicMax of p into a node table (__match_any_sync groups
// equal nodes, so a hot node costs one atomic per warp; max is
// order-independent, hence deterministic).  Phase 2: a pair wins iff
// table[node_p] == p; one scan of per-(round, warp) counts compacts the
// winners in p order.  With kSmem the table lives in shared memory (N <=
// kDedupSmemNodes); otherwise in a self-cleaning global scratch (phase 3 resets
// the touched entries to -1).
#pragma once
#include "internal.cuh"

#ifndef DEDUP_MARK
#define DEDUP_MARK(i)  // debug phase marks (prep.cu with MSPIPE_PHASES)
#endif

namespace mspipe {

constexpr int64_t kDedupSmemNodes = 40960;  // node table in shared memory up to 160 KB

template <int NT, bool kSmem>
__device__ __forceinline__ void block_dedup(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                                            int64_t B, int32_t* __restrict__ gscratch, int32_t* sscratch,
                                            int64_t N, int32_t* __restrict__ out_nodes,
                                            int32_t* __restrict__ out_winner, int32_t* __restrict__ out_num) {
  // Pairs are visited in rounds r: thread tid takes p = r * NT + tid, so every
  // load is coalesced and a thread's kR node ids stay in registers for both
  // phases (round 2 kept a contiguous chunk per thread: its phase-2 loads were
  // strided and sequential, 22 us for GDELT's 8,000 pairs).  p order = (round,
  // warp, lane) order, so one exclusive scan of the per-(round, warp) winner
  // counts gives every winner its place in p order.
  constexpr int kR = 32;  // caller guarantees 2B <= 32 * NT
  constexpr int kW = NT / 32;
  __shared__ int32_t cnt_s[kR * kW];
  __shared__ int32_t total_s;
  int32_t* scratch = kSmem ? sscratch : gscratch;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (kSmem) {
    for (int64_t i = tid; i < N; i += NT) sscratch[i] = -1;
  }
  const int64_t P = 2 * B;
  const int R = (int)((P + NT - 1) / NT);
  int32_t node[kR];
  // all loads first (independent, in flight together), the range check after:
  // a raise_dev atomic between them serialised the loads (16 HBM round trips
  // per thread at GDELT, measured 9.8 us)
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const int64_t p = (int64_t)r * NT + tid;
    node[r] = (r < R && p < P) ? ((p & 1) ? __ldg(dst + (p >> 1)) : __ldg(src + (p >> 1))) : -1;
  }
  bool bad = false;
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const int64_t p = (int64_t)r * NT + tid;
    if (r < R && p < P && (node[r] < 0 || node[r] >= N)) {
      bad = true;
      node[r] = -1;
    }
  }
  if (bad) raise_dev(MSPIPE_DEVERR_RANGE);
  if (kSmem) __syncthreads();  // the table is cleared
  DEDUP_MARK(3);
  // phase 1: warp-aggregated atomicMax of p per node (the highest lane of a
  // group of equal nodes holds the group's largest p)
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    if (r >= R) break;  // uniform over the block
    const unsigned grp = __match_any_sync(0xffffffffu, node[r]);
    const int leader = 31 - __clz(grp);
    if (node[r] >= 0 && lane == leader) atomicMax(scratch + node[r], (int32_t)((int64_t)r * NT + tid));
  }
  if (!kSmem) __threadfence();
  __syncthreads();
  DEDUP_MARK(4);
  // phase 2: a pair wins iff the table holds its p; per-(round, warp) counts
  uint32_t flags = 0;
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    if (r >= R) break;
    const int32_t p = (int32_t)((int64_t)r * NT + tid);
    const bool win = node[r] >= 0 && (kSmem ? sscratch[node[r]] : __ldcg(gscratch + node[r])) == p;
    flags |= (win ? 1u : 0u) << r;
    const unsigned b = __ballot_sync(0xffffffffu, win);
    if (lane == 0) cnt_s[r * kW + wid] = __popc(b);
  }
  __syncthreads();
  if (wid == 0) {  // exclusive scan of the R x kW counts in (round, warp) order
    const int E = R * kW;
    const int per = (E + 31) / 32;
    int32_t sum = 0;
    for (int j = 0; j < per; ++j) {
      const int e = lane * per + j;
      if (e < E) sum += cnt_s[e];
    }
    int32_t incl = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    int32_t run = incl - sum;
    for (int j = 0; j < per; ++j) {
      const int e = lane * per + j;
      if (e < E) {
        const int32_t c = cnt_s[e];
        cnt_s[e] = run;
        run += c;
      }
    }
    if (lane == 31) total_s = incl;
  }
  __syncthreads();
  DEDUP_MARK(5);
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    if (r >= R) break;
    const bool win = (flags >> r) & 1u;
    const unsigned b = __ballot_sync(0xffffffffu, win);
    if (win) {
      const int32_t off = cnt_s[r * kW + wid] + __popc(b & ((1u << lane) - 1u));
      out_nodes[off] = node[r];
      out_winner[off] = (int32_t)((int64_t)r * NT + tid);
    }
  }
  if (!kSmem) {
    __syncthreads();  // all scratch reads are done before the reset
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      if (r >= R) break;
      if ((flags >> r) & 1u) gscratch[node[r]] = -1;
    }
  }
  if (tid == 0) *out_num = total_s;
}

}  // namespace mspipe
