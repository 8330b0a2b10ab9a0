// gru_tc.cu — A5 + A6 on the 5th-generation tensor cores (MSPIPE_FP32_3XTF32).
//
// The memory updater is one contraction [U x K] . [K x 4M], K = Dx + M, with
// packed gate blocks (r, z, n_x, n_h) so the GRUCell gates (G5) are applied
// on the accumulator tile.  It runs as tcgen05.mma
// kind::tf32 with fp32 accumulators in TMEM.  fp32 parity (north star:
// 1e-4 relative) comes from the 3xTF32 split  a = a_hi + a_lo,
// a_hi = rna_tf32(a), a_lo = rna_tf32(a - a_hi), and
//   D += A_hi.B_hi + A_hi.B_lo + A_lo.B_hi      (dropped A_lo.B_lo ~ 2^-22).
//
// Two kernels:
//  k_build_x — one warp per (winner row, 4 x 32-wide K chunks): gathers the message
//    x = [s_w | s_o | e | cos(w dt + p) | h] (A5, fused time encoding) from
//    the snapshot rows, writes the A operand as ready-to-copy SWIZZLE_128B
//    K-major images (hi | lo) per (128-row tile, chunk), and the mail row and
//    commit timestamp of the winner (G14).  Thousands of warps hide the
//    gather latency that a per-CTA producer could not.
//  k_gru_tc — CTA = 128 rows x 20 hidden units (N = 80 accumulator columns)
//    x a K range.  One thread streams (A, B) chunk images with cp.async.bulk
//    (TMA engine, mbarrier complete_tx) through a 3-stage ring, one thread
//    issues 12 MMAs per chunk, all 8 warps read TMEM in the epilogue.  U ~ 10^3
//    rows is only a handful of M tiles, so K is split S ways over a cluster
//    (1,1,S); the S partial tiles are summed through distributed shared memory
//    in fixed rank order (deterministic) and each rank applies the gates to
//    128/S rows.
#include <cuda_bf16.h>
#include <stdlib.h>

#include "internal.cuh"
#include "tc_layout.cuh"

#include <algorithm>

namespace mspipe {

namespace tc {

// hidden units per tile: 20 divides the paper's memory width (M = 100) into
// five tiles with no padding (16 needed seven tiles, 112 columns)
constexpr int kJ = 20;
constexpr int kN = 4 * kJ;              // accumulator columns (UMMA N = 80: M = 128 needs N % 16 == 0)
constexpr int kQ = kJ / 4;              // float4 quads of a gate row
constexpr int kRecvRow = kN / 4 + 1;    // float4 per received row: 21 (odd: conflict-free pushes and reads)
constexpr int kBTile = kN * kKC * 4;    // 10 KB
constexpr int kBBlock = 2 * kBTile;
constexpr int kStageBytes = kABlock + kBBlock;  // 52 KB
constexpr int kStages = 3;
// 8 warps: warp 0 loads, warp 1 issues the MMAs, warps 2..7 prefetch the
// epilogue's inputs; in the epilogue warps w and w + 4 read the two 32-column
// halves of the same TMEM lane quarter (w % 4), so the gate math of a tile
// (expf / tanhf / division chains of 128 rows x 20 units) spreads over 256
// threads: with 4 warps, one warp per scheduler left every dependent step of
// those chains exposed (measured: 3.5 of ~15 us per GDELT tile)
constexpr int kThreads = 256;
constexpr int kPfThreads = kThreads - 64;  // warps 2..7
constexpr int kHBufBytes = kM * kJ * 4;   // h rows of the tile's hidden units (prefetched)
constexpr int kRecvBytes = kM * kRecvRow * 16;  // K-split partials received from the cluster (S x 128/S rows)
constexpr int kSmemBytes =
    kStages * kStageBytes + 1024 /*align*/ + 1024 /*barriers*/ + kHBufBytes + kRecvBytes + kN * 4 /*biases*/;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra.uni WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// wait with cluster-scope acquire: the phase was completed by st.async bytes from other CTAs
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra.uni WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// 32 TMEM lanes x 8 consecutive fp32 columns -> 8 registers per thread.
#define MSPIPE_TMEM_LD8(taddr, r)                                                                        \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"                \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) \
               : "r"(taddr))
// 32 TMEM lanes x 32 consecutive fp32 columns -> 32 registers per thread.
#define MSPIPE_TMEM_LD32(taddr, r)                                                                          \
  asm volatile(                                                                                             \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "                                                             \
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"                                            \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"                          \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),    \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),           \
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),         \
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),         \
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                                               \
      : "r"(taddr))
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// generic address of the same shared-memory location in CTA `rank` of the cluster
__device__ __forceinline__ const void* mapa_generic(const void* p, uint32_t rank) {
  uint64_t r;
  asm volatile("mapa.u64 %0, %1, %2;\n" : "=l"(r) : "l"(reinterpret_cast<uint64_t>(p)), "r"(rank));
  return reinterpret_cast<const void*>(r);
}
// asynchronous remote store whose bytes complete a transaction on the
// destination CTA's mbarrier (remote_bar: mapa'd address of that barrier)
__device__ __forceinline__ void st_async_f4(uint32_t addr, float x, float y, float z, float w, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1,%2,%3,%4}, [%5];\n" ::"r"(addr),
               "f"(x), "f"(y), "f"(z), "f"(w), "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void st_dsmem_f4(uint32_t addr, float x, float y, float z, float w) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"r"(addr), "f"(x), "f"(y), "f"(z), "f"(w)
               : "memory");
}
// Not volatile and no memory clobber so the compiler may batch these loads;
// they stay after the cluster barrier through their address dependence on mapa.
__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t addr) {
  float4 v;
  asm("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];\n"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "r"(addr));
  return v;
}
// SWIZZLE_128B K-major smem descriptor (sm_100: version 1, SBO = 1024 B, LBO field 16 B).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
// kind::tf32 instruction descriptor: D f32, A/B tf32, K-major, M = 128, N = kN.
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kN >> 3) << 17) |
                            ((uint32_t)(kM >> 4) << 24);
// kind::f16 instruction descriptor (MSPIPE_BF16): D f32, A/B bf16, K-major, M = 128, N = kN.
constexpr uint32_t kIdescBf = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kN >> 3) << 17) |
                              ((uint32_t)(kM >> 4) << 24);
constexpr int kBTile16 = kN * kKC16 * 2;             // 10 KB
// bf16 mode splits both operands, x = hi + lo (two bf16), and issues
// A_lo.B_hi + A_hi.B_lo + A_hi.B_hi (the bf16 analogue of 3xTF32): ~16
// mantissa bits per operand, so h' lands within the C.6 per-element rule
// (2e-2|o| + 1e-3) that plain bf16 operands miss by 3-10x
constexpr int kABlock16 = 2 * kATile16;              // 32 KB: hi | lo
constexpr int kBBlock16 = 2 * kBTile16;              // 20 KB: hi | lo
constexpr int kStageBytes16 = kABlock16 + kBBlock16;  // 52 KB
}  // namespace tc

#ifdef MSPIPE_PHASES
__device__ unsigned long long g_phase[8192][16];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PHASE_T(i)                                                                           \
  g_phase[(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x][i] = gtimer()
#define PHASE(i) \
  if (threadIdx.x == 0) PHASE_T(i)
#else
#define PHASE_T(i)
#define PHASE(i)
#endif

int gru_tc_jtiles(const GruDesc& d) { return (d.M + tc::kJ - 1) / tc::kJ; }
__device__ __forceinline__ int gru_tc_jtiles_dev(const GruDesc& d) { return (d.M + tc::kJ - 1) / tc::kJ; }

// ---------------------------------------------------------------------------
// weight packing: per (hidden tile jt, K chunk c) a 16 KB block
// [hi image 8 KB | lo image 8 KB] of the B operand, N = 64 rows n = g*16 + jj
// (gate g in r, z, n_x, n_h), K-major SWIZZLE_128B; bias[jt*64 + n].
// ---------------------------------------------------------------------------
// B-operand value of row n = g*16 + jj of hidden tile jt at K index k (0 outside)
__device__ __forceinline__ float wval(const float* __restrict__ w_ih, const float* __restrict__ w_hh,
                                      const GruDesc& d, int32_t g, int32_t j, int32_t k) {
  const int32_t M = d.M;
  if (j >= M) return 0.f;
  if (d.cell == MSPIPE_CELL_RNN) {  // RNNCell: n_x = W_ih x, n_h = W_hh h
    if (k < d.Dx) return g == 2 ? w_ih[(int64_t)j * d.Dx + k] : 0.f;
    if (k < d.K) return g == 3 ? w_hh[(int64_t)j * M + (k - d.Dx)] : 0.f;
    return 0.f;
  }
  if (k < d.Dx) return g < 3 ? w_ih[(int64_t)(g * M + j) * d.Dx + k] : 0.f;
  if (k < d.K) {
    const int32_t q = k - d.Dx;
    if (g == 0) return w_hh[(int64_t)j * M + q];
    if (g == 1) return w_hh[(int64_t)(M + j) * M + q];
    if (g == 3) return w_hh[(int64_t)(2 * M + j) * M + q];
  }
  return 0.f;
}

// bf16 weights (MSPIPE_BF16): per (jt, 64-wide K chunk) one 8 KB SWIZZLE_128B
// K-major image of the 64 B-operand rows, round-to-nearest bf16
__global__ void k_gru_pack_bf16(const float* __restrict__ w_ih, const float* __restrict__ w_hh, GruDesc d,
                                int32_t jtiles, uint8_t* __restrict__ wtc) {
  const int32_t nchunks = d.Kpad / tc::kKC16;
  const int64_t total = (int64_t)jtiles * nchunks * tc::kN * tc::kKC16;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t kk = (int32_t)(t % tc::kKC16);
    const int32_t n = (int32_t)((t / tc::kKC16) % tc::kN);
    const int32_t c = (int32_t)((t / (tc::kKC16 * tc::kN)) % nchunks);
    const int32_t jt = (int32_t)(t / ((int64_t)tc::kKC16 * tc::kN * nchunks));
    const float v = wval(w_ih, w_hh, d, n / tc::kJ, jt * tc::kJ + n % tc::kJ, c * tc::kKC16 + kk);
    uint8_t* blk = wtc + ((int64_t)jt * nchunks + c) * tc::kBBlock16;
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    const uint32_t off = tc::sw128_off16((uint32_t)n, (uint32_t)kk);
    *reinterpret_cast<__nv_bfloat16*>(blk + off) = hi;
    *reinterpret_cast<__nv_bfloat16*>(blk + tc::kBTile16 + off) = __float2bfloat16_rn(v - __bfloat162float(hi));
  }
}

__global__ void k_gru_pack_tc(const float* __restrict__ w_ih, const float* __restrict__ w_hh,
                              const float* __restrict__ b_ih, const float* __restrict__ b_hh, GruDesc d,
                              int32_t jtiles, float* __restrict__ wtc, float* __restrict__ bias) {
  const int32_t nchunks = d.Kpad / tc::kKC;
  const int64_t total = (int64_t)jtiles * nchunks * tc::kN * tc::kKC;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t kk = (int32_t)(t % tc::kKC);
    const int32_t n = (int32_t)((t / tc::kKC) % tc::kN);
    const int32_t c = (int32_t)((t / (tc::kKC * tc::kN)) % nchunks);
    const int32_t jt = (int32_t)(t / ((int64_t)tc::kKC * tc::kN * nchunks));
    const int32_t g = n / tc::kJ, jj = n % tc::kJ, j = jt * tc::kJ + jj, k = c * tc::kKC + kk;
    const int32_t M = d.M;
    const float v = wval(w_ih, w_hh, d, g, j, k);
    const float hi = tc::tf32_rna(v);
    const float lo = tc::tf32_rna(v - hi);
    char* blk = reinterpret_cast<char*>(wtc) + ((int64_t)jt * nchunks + c) * tc::kBBlock;
    const uint32_t off = tc::sw128_off((uint32_t)n, (uint32_t)kk);
    *reinterpret_cast<float*>(blk + off) = hi;
    *reinterpret_cast<float*>(blk + tc::kBTile + off) = lo;
    if (c == 0 && kk == 0) {
      float b = 0.f;
      if (j < M && d.cell == MSPIPE_CELL_RNN) {
        if (g == 2) b = b_ih[j];
        else if (g == 3) b = b_hh[j];
      } else if (j < M) {
        if (g == 0) b = b_ih[j] + b_hh[j];
        else if (g == 1) b = b_ih[M + j] + b_hh[M + j];
        else if (g == 2) b = b_ih[2 * M + j];
        else b = b_hh[2 * M + j];
      }
      bias[jt * tc::kN + n] = b;
    }
  }
}

size_t gru_tc_bias_floats(const GruDesc& d) { return (size_t)gru_tc_jtiles(d) * tc::kN; }

size_t gru_tc_packed_floats(const GruDesc& d) {
  if (d.bf16) return (size_t)gru_tc_jtiles(d) * (d.Kpad / tc::kKC16) * (tc::kBBlock16 / 4);
  return (size_t)gru_tc_jtiles(d) * (d.Kpad / tc::kKC) * (tc::kBBlock / 4);
}

size_t gru_tc_xbuf_floats(const GruDesc& d, int64_t max_events) {
  const int64_t mtiles = (2 * max_events + tc::kM - 1) / tc::kM;
  if (d.bf16) return (size_t)mtiles * (d.Kpad / tc::kKC16) * (tc::kABlock16 / 4);
  return (size_t)mtiles * (d.Kpad / tc::kKC) * (tc::kABlock / 4);
}

void launch_gru_pack_tc(const float* w_ih, const float* w_hh, const float* b_ih, const float* b_hh,
                        const GruDesc& d, float* wtc, float* bias, cudaStream_t s) {
  const int threads = 256;
  const int64_t total = (int64_t)gru_tc_packed_floats(d) / 2;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 4096) blocks = 4096;
  if (!d.bf16) {
    k_gru_pack_tc<<<(unsigned)blocks, threads, 0, s>>>(w_ih, w_hh, b_ih, b_hh, d, gru_tc_jtiles(d), wtc, bias);
    return;
  }
  // bf16: the weight images, then the biases (k_gru_pack_tc's bias pass over one chunk, into scratch)
  const int64_t total16 = (int64_t)gru_tc_jtiles(d) * (d.Kpad / tc::kKC16) * tc::kN * tc::kKC16;
  int64_t b16 = (total16 + threads - 1) / threads;
  if (b16 > 4096) b16 = 4096;
  k_gru_pack_bf16<<<(unsigned)b16, threads, 0, s>>>(w_ih, w_hh, d, gru_tc_jtiles(d), (uint8_t*)wtc);
  GruDesc one = d;
  one.Kpad = tc::kKC;  // a single 32-wide chunk: k_gru_pack_tc then writes every bias once
  float* scratch = nullptr;
  if (cudaMallocAsync(&scratch, sizeof(float) * gru_tc_jtiles(d) * (tc::kBBlock / 4), s) != cudaSuccess) return;
  k_gru_pack_tc<<<(unsigned)gru_tc_jtiles(d), threads, 0, s>>>(w_ih, w_hh, b_ih, b_hh, one, gru_tc_jtiles(d),
                                                               scratch, bias);
  cudaFreeAsync(scratch, s);
}

// ---------------------------------------------------------------------------
struct TcArgs {
  GruDesc d;
  const float* wtc;   // packed B blocks
  float* xbuf;        // A blocks [mtile][chunk][hi | lo]
  const double* ts;
  int64_t B;
  const float* ef;
  const float* snap_mem;
  const double* snap_ts;
  int64_t step;
  const float* snap_h;
  const int32_t* winner;
  const int32_t* num_unique;
  float* out_mem;
  double* out_ts;
  float* out_mail;
  int64_t mail_stride;
  // fused A7 (commit_mem != nullptr): h' goes straight to mem[node]; the
  // commit ts and mail rows staged by k_build_x (new_ts, new_mail) are copied
  // to mem_ts / mail_ts / mail[node]
  const int32_t* nodes;
  float* commit_mem;
  double* commit_mem_ts;
  float* commit_mail;
  double* commit_mail_ts;
  const double* new_ts;
  const float* new_mail;
  int64_t num_nodes;
  // double-buffered state (GruCommit)
  int32_t* save_nodes;
  int32_t* save_num;
  CatchUp cu;
  // build from the state tables (mspipe_message_build_tables): tsrc/tdst are
  // the batch's endpoints, snap_mem / snap_ts the tables of the version read,
  // indexed by node id instead of by snapshot row
  const int32_t* tsrc;
  const int32_t* tdst;
  // GEMM: h (the GRU hidden input) is new_mail[u][0:M] (= S.mem[w], G14)
  int32_t h_from_mail;
  int32_t cpb;  // K chunks per TMEM accumulator buffer (k_gru_tc, tf32)
  int32_t skip_meta;  // fused A7: mem_ts / mail / mail_ts written by a concurrent k_writeback instead
  int32_t* res_nodes;  // optional result record: winner node ids [U] and U (host read-back)
  int32_t* res_num;
};

// row index of the state S.mem[w] of pair (ev, role) in snap_mem (times M) /
// snap_ts: the snapshot row (root layout, stride `step`) or, building from the
// tables, the node id itself
__device__ __forceinline__ int64_t snap_row(const TcArgs& a, int32_t ev, int role) {
  if (a.tsrc) return role ? __ldg(a.tdst + ev) : __ldg(a.tsrc + ev);
  return (role ? a.B + ev : (int64_t)ev) * a.step;
}

// Double-buffered commit: copy the previous commit's rows (old set -> this
// commit's set) except this commit's own winners, which the epilogue writes.
// Warp `wq` of `nw` participating warps; one warp per row.
__device__ __forceinline__ void catch_up(const TcArgs& a, int64_t wq, int64_t nw, int lane) {
  const int32_t np = __ldg(a.cu.prev_num);
  const int32_t Qm = a.d.M / 4, Qa = (int32_t)(a.mail_stride / 4);
  for (int64_t r = wq; r < np; r += nw) {
    const int32_t v = __ldg(a.cu.prev_nodes + r);
    if (__ldg(a.cu.stamp + v) != a.cu.iter) catchup_row(a.cu, v, Qm, Qa, lane);
  }
}

// A5 value of winner pair p, column k of x = [s_w | s_o | e | cos(w dt + p) | h]
__device__ __forceinline__ float msg_val(const TcArgs& a, int32_t p, int32_t k) {
  const GruDesc& d = a.d;
  const int32_t M = d.M;
  const int32_t ev = p >> 1, role = p & 1;
  if (k < M) return __ldg(a.snap_mem + snap_row(a, ev, role) * M + k);
  if (k < 2 * M) return __ldg(a.snap_mem + snap_row(a, ev, role ^ 1) * M + (k - M));
  if (k < d.Dm) return __ldg(a.ef + (int64_t)ev * d.He + (k - 2 * M));
  if (k < d.Dx) {
    const float dt = (float)(__ldg(a.ts + ev) - __ldg(a.snap_ts + snap_row(a, ev, role)));  // Δt (G4)
    const int q = k - d.Dm;
    return time_cos(fmaf(__ldg(d.time_w + q), dt, __ldg(d.time_b + q)));
  }
  if (k < d.K) {
    const int q = k - d.Dx;
    return a.snap_h ? __ldg(a.snap_h + (role ? a.B + ev : (int64_t)ev) * M + q)
                    : __ldg(a.snap_mem + snap_row(a, ev, role) * M + q);
  }
  return 0.f;
}

// A5 with bf16 operands (MSPIPE_BF16): one warp per (row, 64-wide chunk), two
// columns per lane; the mail row and commit ts stay fp32.
__device__ __forceinline__ void build_bf16(const TcArgs& a) {
  const GruDesc& d = a.d;
  const int32_t U = __ldg(a.num_unique);
  const int32_t nchunks = d.Kpad / tc::kKC16;
  const int32_t mtiles = (U + tc::kM - 1) / tc::kM;
  const int64_t items = (int64_t)mtiles * nchunks * tc::kM;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < items; w += nwarps) {
    const int32_t row = (int32_t)(w % tc::kM);
    const int32_t c = (int32_t)((w / tc::kM) % nchunks);
    const int32_t mt = (int32_t)(w / ((int64_t)tc::kM * nchunks));
    const int32_t u = mt * tc::kM + row;
    const int32_t k0 = c * tc::kKC16 + 2 * lane;
    float v0 = 0.f, v1 = 0.f;
    if (u < U) {
      const int32_t p = __ldg(a.winner + u);
      v0 = msg_val(a, p, k0);
      v1 = msg_val(a, p, k0 + 1);
      if (a.out_mail) {
        if (k0 < a.mail_stride) a.out_mail[(int64_t)u * a.mail_stride + k0] = k0 < d.Dm ? v0 : 0.f;
        if (k0 + 1 < a.mail_stride) a.out_mail[(int64_t)u * a.mail_stride + k0 + 1] = k0 + 1 < d.Dm ? v1 : 0.f;
      }
      if (c == 0 && lane == 0) a.out_ts[u] = __ldg(a.ts + (p >> 1));
    }
    uint8_t* blk = reinterpret_cast<uint8_t*>(a.xbuf) + ((int64_t)mt * nchunks + c) * tc::kABlock16;
    const __nv_bfloat162 hi = __floats2bfloat162_rn(v0, v1);
    const float2 hf = __bfloat1622float2(hi);
    const uint32_t off = tc::sw128_off16((uint32_t)row, (uint32_t)(2 * lane));
    *reinterpret_cast<__nv_bfloat162*>(blk + off) = hi;
    *reinterpret_cast<__nv_bfloat162*>(blk + tc::kATile16 + off) = __floats2bfloat162_rn(v0 - hf.x, v1 - hf.y);
  }
}

// A5: one warp per (row, kBuildChunks chunks).  lane = column inside a chunk.
// kBuildChunks = 4 (default) or 20 (MSPIPE_BUILD_ROW=1: one warp per whole row
// for Kpad <= 640, the row's metadata resolved once, 20 loads in flight per lane)
constexpr int kBuildChunks = 4;
constexpr int kBuildRowChunks = 20;
template <int kBuildChunks>
__global__ void __launch_bounds__(256) k_build_x(TcArgs a) {
  if (a.d.bf16) {
    build_bf16(a);
    return;
  }
  const GruDesc& d = a.d;
  const int32_t U = __ldg(a.num_unique);
  const int32_t nchunks = d.Kpad / tc::kKC;
  const int32_t ngroups = (nchunks + kBuildChunks - 1) / kBuildChunks;
  const int32_t mtiles = (U + tc::kM - 1) / tc::kM;
  // one warp per (row, group of kBuildChunks K chunks): the row's pair, rows
  // and Δt are resolved once for 128 columns (the per-item index work was
  // half of the kernel's issue slots with one chunk per item), kBuildChunks
  // loads in flight per lane.  items < 2^31: 32-bit index arithmetic.
  const uint32_t items = (uint32_t)mtiles * (uint32_t)ngroups * tc::kM;
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const int32_t M = d.M;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < items; w += nwarps) {
    const int32_t row = (int32_t)(w % tc::kM);
    const uint32_t gm = w / tc::kM;
    const int32_t mt = (int32_t)(gm / (uint32_t)ngroups);
    const int32_t cg = (int32_t)(gm - (uint32_t)mt * (uint32_t)ngroups);
    const int32_t u = mt * tc::kM + row;
    float v[kBuildChunks];
#pragma unroll
    for (int q = 0; q < kBuildChunks; ++q) v[q] = 0.f;
    if (u < U) {
      const int32_t p = __ldg(a.winner + u);
      const int32_t ev = p >> 1, role = p & 1;
      const float* sw = a.snap_mem + snap_row(a, ev, role) * M;
      const float* so = a.snap_mem + snap_row(a, ev, role ^ 1) * M;
      const float* hrow = a.snap_h ? a.snap_h + (role ? a.B + ev : (int64_t)ev) * M : sw;
      const float* erow = a.ef + (int64_t)ev * d.He;
      const double t_ev = __ldg(a.ts + ev);
      const float dt = (float)(t_ev - __ldg(a.snap_ts + snap_row(a, ev, role)));  // Δt (G4)
#pragma unroll
      for (int q = 0; q < kBuildChunks; ++q) {  // loads first (all in flight), then the encoding
        const int32_t k = (cg * kBuildChunks + q) * tc::kKC + lane;
        if (k < M) v[q] = __ldg(sw + k);
        else if (k < 2 * M) v[q] = __ldg(so + (k - M));
        else if (k < d.Dm) v[q] = __ldg(erow + (k - 2 * M));
        else if (k >= d.Dx && k < d.K) v[q] = __ldg(hrow + (k - d.Dx));
      }
#pragma unroll
      for (int q = 0; q < kBuildChunks; ++q) {
        const int32_t k = (cg * kBuildChunks + q) * tc::kKC + lane;
        if (k >= d.Dm && k < d.Dx) {
          const int qq = k - d.Dm;
          v[q] = time_cos(fmaf(__ldg(d.time_w + qq), dt, __ldg(d.time_b + qq)));
        }
        if (k < a.mail_stride) a.out_mail[(int64_t)u * a.mail_stride + k] = k < d.Dm ? v[q] : 0.f;
      }
      if (cg == 0 && lane == 0) a.out_ts[u] = t_ev;
    }
    const uint32_t off = tc::sw128_off((uint32_t)row, (uint32_t)lane);
#pragma unroll
    for (int q = 0; q < kBuildChunks; ++q) {
      const int32_t c = cg * kBuildChunks + q;
      if (c >= nchunks) break;
      const float hi = tc::tf32_rna(v[q]);
      const float lo = tc::tf32_rna(v[q] - hi);
      char* blk = reinterpret_cast<char*>(a.xbuf) + ((int64_t)mt * nchunks + c) * tc::kABlock;
      *reinterpret_cast<float*>(blk + off) = hi;
      *reinterpret_cast<float*>(blk + tc::kATile + off) = lo;
    }
  }
}

// Gate nonlinearities.  MSPIPE_FAST_GATES (default): σ(x) = 1 / (1 + e^-x)
// and tanh(x) = 1 - 2 / (1 + e^2x) from the MUFU exponential (__expf) and
// reciprocal (rcp.approx, 1 ulp): ~1e-7 absolute on σ and tanh against the
// 1e-4|o| + 1e-6 rule.  The IEEE division (and __frcp_rn) put a slow-path
// branch around every reciprocal, which serialised the 12 reciprocals of a
// 4-unit item: ~2 us of a 12 us GDELT tile (phase marks).
#ifndef MSPIPE_FAST_GATES
#define MSPIPE_FAST_GATES 1
#endif
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float gate_sigmoid(float x) {
  if (MSPIPE_FAST_GATES) return rcp_approx(1.0f + __expf(-x));
  return 1.0f / (1.0f + expf(-x));
}
__device__ __forceinline__ float gate_tanh(float x) {
  if (MSPIPE_FAST_GATES) return 1.0f - 2.0f * rcp_approx(1.0f + __expf(2.0f * x));
  return tanhf(x);
}

// GRUCell gates (G5): r = σ(.), z = σ(.), n = tanh(x_n + r h_n), h' = (1 - z) n + z h.
__device__ __forceinline__ float4 gates4(const float* pr, const float* pz, const float* pnx, const float* pnh,
                                         float4 h, int32_t cell) {
  const float* hv = &h.x;
  float out[4];
  if (cell == MSPIPE_CELL_RNN) {  // RNNCell (row F3): h' = tanh(W_ih x + b_ih + W_hh h + b_hh)
#pragma unroll
    for (int e = 0; e < 4; ++e) out[e] = gate_tanh(pnx[e] + pnh[e]);
    return make_float4(out[0], out[1], out[2], out[3]);
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float r = gate_sigmoid(pr[e]);
    const float z = gate_sigmoid(pz[e]);
    const float n = gate_tanh(pnx[e] + r * pnh[e]);
    out[e] = (1.0f - z) * n + z * hv[e];
  }
  return make_float4(out[0], out[1], out[2], out[3]);
}

// h' of winner u, hidden units j0..j0+3: to out_mem (winner order) and, when
// the write-back is fused (A7), to the state row of its node.
__device__ __forceinline__ void store_h4(const TcArgs& a, int32_t u, int32_t node, int32_t j0, float4 h) {
  if (a.out_mem) *reinterpret_cast<float4*>(a.out_mem + (int64_t)u * a.d.M + j0) = h;
  if (a.commit_mem && node >= 0) *reinterpret_cast<float4*>(a.commit_mem + (int64_t)node * a.d.M + j0) = h;
}

// fused A7, rest of the row: mem_ts = mail_ts = t*, mail row = staged x[0:Dm];
// the float4 columns of the mail row are spread over the hidden tiles.
// (Prefetching these into shared memory during the main loop was measured
// slower: the extra loads delay the warps' arrival at the cluster barrier.)
__device__ __forceinline__ void commit_rows(const TcArgs& a, int32_t m0, int32_t U, int rb, int re, int jt, int J,
                                            const int32_t* rownode) {
  if (!a.new_mail) {  // deferred mailbox (row F3): mem_ts only; the mail rows follow the commit
    if (jt == 0)
      for (int mm = rb + (int)threadIdx.x; mm < re; mm += blockDim.x) {
        const int32_t u = m0 + mm, node = rownode[mm];
        if (u < U && node >= 0) a.commit_mem_ts[node] = __ldg(a.new_ts + u);
      }
    return;
  }
  const int Q = (int)(a.mail_stride / 4);
  const int c0 = jt * Q / J, c1 = (jt + 1) * Q / J, nq = c1 - c0;
  const float4* __restrict__ src = reinterpret_cast<const float4*>(a.new_mail);
  float4* __restrict__ dst = reinterpret_cast<float4*>(a.commit_mail);
  // 4 loads in flight per thread before their stores (a load-store-load loop
  // serialises on L2 latency: 13 round trips per thread for 128 rows)
  const int total = (re - rb) * nq;
  for (int base = threadIdx.x; base < total; base += 4 * blockDim.x) {
    float4 v[4];
    int64_t to[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int it = base + q * blockDim.x;
      to[q] = -1;
      if (it < total) {
        const int mm = rb + it / nq, c = c0 + it % nq;
        const int32_t u = m0 + mm, node = rownode[mm];
        if (u < U && node >= 0) {
          v[q] = __ldg(src + (int64_t)u * Q + c);
          to[q] = (int64_t)node * Q + c;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (to[q] >= 0) dst[to[q]] = v[q];
  }
  if (jt == 0)
    for (int mm = rb + (int)threadIdx.x; mm < re; mm += blockDim.x) {
      const int32_t u = m0 + mm, node = rownode[mm];
      if (u < U && node >= 0) {
        const double t = __ldg(a.new_ts + u);
        a.commit_mem_ts[node] = t;
        a.commit_mail_ts[node] = t;
      }
    }
}

// kBf: bf16 operands (MSPIPE_BF16): 64-wide K chunks of 52 KB stages (hi | lo), one
// accumulator per CTA for its K range (bf16 tolerance, north star 2e-2); the
// K split and partial-sum exchange are the tf32 kernel's.
// Persistent over tiles: grid (S, clusters); cluster c takes tiles
// q = c, c + clusters, ... of the mt_act x J tiles of the U rows (U read on
// the device), so no CTA is launched for the empty tiles of the 2B bound.
// Per tile: the loader streams the K chunks of (mt, jt) through the stage
// ring (chunk counter continued across tiles, so stage phases carry over) and
// issues the next tile's first kStages chunks as soon as this tile's MMAs are
// done, overlapping them with the epilogue; the K-split partials go through
// one receive buffer, so one cluster barrier per tile orders every push after
// the owner's reads of the tile before.
#ifndef MSPIPE_MAIL_PF
#define MSPIPE_MAIL_PF 1
#endif
constexpr bool kMailPf = MSPIPE_MAIL_PF != 0;
// K-split partials pushed with st.async completing bytes on the owner's
// mbarrier (no cluster barrier between the pushes and the reduction)
#ifndef MSPIPE_ASYNC_PUSH
#define MSPIPE_ASYNC_PUSH 1
#endif
constexpr bool kAsyncPush = MSPIPE_ASYNC_PUSH != 0;
// K-split partials of the CTA's own rows stored locally (not through st.async)
#ifndef MSPIPE_LOCAL_PUSH
#define MSPIPE_LOCAL_PUSH 1
#endif
constexpr bool kLocalPush = MSPIPE_LOCAL_PUSH != 0;

// __launch_bounds__ without a min-blocks clause: ptxas then keeps k_gru_tc at 167
// registers (213 with ", 1"), so a 256-thread k_build_x block (40 registers) of the
// next batch fits beside the GEMM CTA in the SM's 64K-register file (the GEMM's
// shared memory leaves room for it: k_build_x uses none).  -DMSPIPE_GEMM_MINB=n: a
// min-blocks bound of n (1: the old 213 registers; 2: 128 registers, small spills).
#ifdef MSPIPE_GEMM_MINB
#define MSPIPE_GEMM_BOUNDS __launch_bounds__(tc::kThreads, MSPIPE_GEMM_MINB)
#else
#define MSPIPE_GEMM_BOUNDS __launch_bounds__(tc::kThreads)
#endif
template <bool kBf>
__global__ void MSPIPE_GEMM_BOUNDS k_gru_tc(TcArgs a) {
  using namespace tc;
  constexpr int SB = kBf ? kStageBytes16 : kStageBytes;
  constexpr int AB = kBf ? kABlock16 : kABlock;
  constexpr int BB = kBf ? kBBlock16 : kBBlock;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * SB);
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  uint64_t* rfull = acc_full + 2;  // K-split partials of the tile received (st.async bytes)
  int32_t* rownode = reinterpret_cast<int32_t*>(smem + kStages * SB + 512);  // [128] node of each row
  float4* hbuf = reinterpret_cast<float4*>(smem + kStages * SB + 1024);  // [128 rows][kQ]
  // [S ranks x 128/S rows][kRecvRow float4]: row stride 84 words, so the 8
  // rows of a quarter-warp's 16-byte accesses fall on 8 distinct bank quads
  float4* recv = reinterpret_cast<float4*>(smem + kStages * SB + 1024 + kHBufBytes);
  // this tile's gate biases, prefetched during the main loop
  float* sbias = reinterpret_cast<float*>(smem + kStages * SB + 1024 + kHBufBytes + kRecvBytes);

  const GruDesc& d = a.d;
  PHASE(9);
  // U (written by the previous step's prep) is a cold HBM read: it is consumed
  // only after the setup and the first tile's speculative loads below
  const int32_t U = __ldg(a.num_unique);
  const int J = gru_tc_jtiles_dev(d);
  const int S = gridDim.x;
  const int split = blockIdx.x;
  const int64_t cta_q = (int64_t)blockIdx.y * S + split;
  const int64_t n_cta = (int64_t)gridDim.y * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t nchunks = d.Kpad / (kBf ? kKC16 : kKC);
  const int32_t c0 = split * nchunks / S, c1 = (split + 1) * nchunks / S;
  const int32_t nc = c1 - c0;  // tf32: <= kMaxChunks buffers of cpb chunks
  // tf32: K chunk ci accumulates into TMEM buffer ci / cpb (cpb chunks per
  // kN-column buffer; 1 unless the K range exceeds kMaxChunks buffers)
  const int cpb = a.cpb > 0 ? a.cpb : 1;
  const int nbuf = (nc + cpb - 1) / cpb;
  const int need = (kBf ? 1 : nbuf) * kN;  // allocation: a power of two >= 32 columns
  const uint32_t tcols = need <= 32 ? 32u : need <= 64 ? 64u : need <= 128 ? 128u : need <= 256 ? 256u : 512u;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(rfull, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, tcols);
  PHASE(0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // kAsyncPush: the peers may target rfull only once it is initialised; the
  // matching wait comes right before this CTA's first push (long satisfied)
  if (kAsyncPush && S > 1) cluster_arrive_relaxed();
  const uint32_t tmem = *tmem_slot;
  const int rank = S > 1 ? (int)cluster_rank() : 0;

  // loader: chunk ci of the tile with sequence number ti (global chunk counter g = ti*nc + ci)
  auto load_chunk = [&](int64_t ti, int32_t mt_l, int jt_l, int ci) {
    const int64_t g = ti * nc + ci;
    const int s = (int)(g % kStages);
    const uint32_t ph = (uint32_t)(g / kStages) & 1u;
    mbar_wait(&empty[s], ph ^ 1u);
    uint8_t* st = smem + s * SB;
    mbar_arrive_expect_tx(&full[s], SB);
    bulk_g2s(st, reinterpret_cast<const char*>(a.xbuf) + ((int64_t)mt_l * nchunks + c0 + ci) * AB, AB, &full[s]);
    bulk_g2s(st + AB, reinterpret_cast<const char*>(a.wtc) + ((int64_t)jt_l * nchunks + c0 + ci) * BB, BB, &full[s]);
  };
  // the cluster's first tile (q = blockIdx.y) is issued before U is known: the
  // workspace holds every M tile of the 2B bound, so the reads are in bounds
  int pre = 0;  // chunks of the current tile the loader already issued
  if (warp == 0 && lane == 0)
    for (; pre < nc && pre < kStages; ++pre) load_chunk(0, (int32_t)(blockIdx.y / J), (int)(blockIdx.y % J), pre);
  const int64_t mt_act = U > 0 ? (U + kM - 1) / kM : 0;
  const int64_t tiles = mt_act * J;
  if (cta_q == 0 && threadIdx.x == 0) {
    if (a.save_num) *a.save_num = U;
    if (a.res_num) *a.res_num = U;
  }
  if ((int64_t)blockIdx.y >= tiles) {  // no tile for this cluster (uniform across it)
    if (warp == 0 && lane == 0)
      for (int s = 0; s < pre; ++s) mbar_wait(&full[s], 0u);  // drain the speculative copies
    if (a.cu.stamp && warp >= 2) catch_up(a, cta_q * (kPfThreads / 32) + (warp - 2), n_cta * (kPfThreads / 32), lane);
    if (kAsyncPush && S > 1) cluster_wait();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tmem, tcols);
    return;
  }
  int64_t ti = 0;
  for (int64_t q = blockIdx.y; q < tiles; q += gridDim.y, ++ti) {
    const int32_t mt = (int32_t)(q / J);
    const int jt = (int)(q % J);
    const int32_t m0 = mt * kM;
    if (warp == 0 && lane == 0) {
      for (int ci = pre; ci < nc; ++ci) load_chunk(ti, mt, jt, ci);
    } else if (warp == 1 && lane == 0) {
      // MMA issuer.  Each K chunk accumulates into its OWN 64-column TMEM
      // buffer (12 MMAs): the tensor core's accumulation truncates, so the error
      // grows with the MMAs per accumulator (measured: max 5.2e-6 for 222 MMAs,
      // 1.0e-6 for 28); the epilogue then adds the buffers in fp32 registers
      // with round-to-nearest, in chunk order.
      for (int ci = 0; ci < nc; ++ci) {
        const int64_t g = ti * nc + ci;
        const int s = (int)(g % kStages);
        const uint32_t ph = (uint32_t)(g / kStages) & 1u;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t base = smem_u32(smem + s * SB);
        if (kBf) {  // 4 k-steps of K = 16 (32 B along K), 3 split MMAs each, into the single accumulator
          const uint64_t da_hi = sw128_desc(base), da_lo = sw128_desc(base + kATile16);
          const uint64_t db_hi = sw128_desc(base + AB), db_lo = sw128_desc(base + AB + kBTile16);
#pragma unroll
          for (int kk = 0; kk < kKC16 / 16; ++kk) {
            const uint64_t adv = (uint64_t)(kk * 32) >> 4;
            mma_bf16(tmem, da_lo + adv, db_hi + adv, kIdescBf, (ci | kk) != 0);
            mma_bf16(tmem, da_hi + adv, db_lo + adv, kIdescBf, 1u);
            mma_bf16(tmem, da_hi + adv, db_hi + adv, kIdescBf, 1u);
          }
        } else {
          const uint64_t da_hi = sw128_desc(base), da_lo = sw128_desc(base + kATile);
          const uint64_t db_hi = sw128_desc(base + kABlock), db_lo = sw128_desc(base + kABlock + kBTile);
          const uint32_t tacc = tmem + (uint32_t)((ci / cpb) * kN);
#pragma unroll
          for (int kk = 0; kk < kKC / 8; ++kk) {
            const uint64_t adv = (uint64_t)(kk * 32) >> 4;  // 8 tf32 = 32 B along K inside the swizzle row
            mma_tf32(tacc, da_lo + adv, db_hi + adv, kIdesc, (kk != 0 || ci % cpb != 0) ? 1u : 0u);
            mma_tf32(tacc, da_hi + adv, db_lo + adv, kIdesc, 1u);
            mma_tf32(tacc, da_hi + adv, db_hi + adv, kIdesc, 1u);
          }
        }
        mma_commit(&empty[s]);
      }
      mma_commit(acc_full);
      PHASE_T(2);
    } else if (warp >= 2) {
      // idle warps: prefetch h (the GRU hidden input: snap_h, the snapshot
      // row, or the staged mail row, G13/G14) of the rows this CTA will
      // finalise, 4 hidden units per item
      const int rb = rank * kM / S, re = (rank + 1) * kM / S;
      if (kMailPf && a.commit_mem && a.new_mail) {
        // warm the commit epilogue's mail-row slices (staged by k_build_x a step ago) into L2
        const int Q = (int)(a.mail_stride / 4);
        const int cq0 = jt * Q / J, nq = (jt + 1) * Q / J - cq0;
        for (int mm = rb + (int)threadIdx.x - 64; mm < re; mm += kPfThreads)
          if (m0 + mm < U && nq > 0)
            l2_prefetch(a.new_mail + ((int64_t)(m0 + mm) * Q + cq0) * 4, (uint32_t)nq * 16u);
      }
      for (int it = threadIdx.x - 64; it < (re - rb) * kQ; it += kPfThreads) {
        const int mm = rb + it / kQ, qq = it % kQ;
        const int32_t u = m0 + mm, j0 = jt * kJ + qq * 4;
        float4 hv = make_float4(0.f, 0.f, 0.f, 0.f);
        if (u < U && j0 < d.M) {  // M % 4 == 0: a quad is all valid or all padding
          const float* hrow;
          if (a.h_from_mail) {
            hrow = a.new_mail + (int64_t)u * a.mail_stride;
          } else {
            const int32_t p = __ldg(a.winner + u);
            const int64_t rw = (p & 1) ? a.B + (p >> 1) : (p >> 1);
            hrow = a.snap_h ? a.snap_h + rw * d.M : a.snap_mem + rw * a.step * d.M;
          }
          hv = __ldg(reinterpret_cast<const float4*>(hrow + j0));
        }
        hbuf[mm * kQ + qq] = hv;
        if (qq == 0) {
          const int32_t node = (a.commit_mem && u < U) ? __ldg(a.nodes + u) : -1;
          rownode[mm] = node;
          if (a.save_nodes && jt == 0 && node >= 0) a.save_nodes[u] = node;
          if (a.res_nodes && jt == 0 && u < U) a.res_nodes[u] = node;
        }
      }
      for (int i = threadIdx.x - 64; i < kN; i += kPfThreads) sbias[i] = __ldg(d.bias + jt * kN + i);
      if (ti == 0 && a.cu.stamp) catch_up(a, cta_q * (kPfThreads / 32) + (warp - 2), n_cta * (kPfThreads / 32), lane);
    }
    __syncwarp();

    // ---------------- epilogue: TMEM -> registers (thread = row)
    mbar_wait(acc_full, (uint32_t)(ti & 1));
    PHASE(3);
    tc_fence_after();
    if (warp == 0 && lane == 0) {  // the stages are free: start the next tile's loads now
      pre = 0;
      const int64_t qn = q + gridDim.y;
      if (qn < tiles) {
        for (; pre < nc && pre < kStages; ++pre) load_chunk(ti + 1, (int32_t)(qn / J), (int)(qn % J), pre);
      }
    }
    // thread = (row m of lane quarter warp % 4, column half warp / 4): the
    // half's kN/2 = 40 columns as five 8-column loads per buffer (column
    // offsets multiples of 8)
    constexpr int kHC = kN / 2;
    const int half = warp >> 2;
    const int m = (warp & 3) * 32 + lane;
    const uint32_t tbase = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(half * kHC);
    uint32_t r0[kHC];
#pragma unroll
    for (int c8 = 0; c8 < kHC / 8; ++c8) MSPIPE_TMEM_LD8(tbase + 8 * c8, (r0 + 8 * c8));
    tmem_wait_ld();
    for (int bi = 1; bi < (kBf ? 1 : nbuf); ++bi) {
      uint32_t t0[kHC];
#pragma unroll
      for (int c8 = 0; c8 < kHC / 8; ++c8) MSPIPE_TMEM_LD8(tbase + bi * kN + 8 * c8, (t0 + 8 * c8));
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < kHC; ++i)
        r0[i] = __float_as_uint(__fadd_rn(__uint_as_float(r0[i]), __uint_as_float(t0[i])));
    }
    PHASE(4);
    const float* bias = sbias;
    // this thread's half row (kHC / 4 = 10 float4, index half * 10 + c4) goes
    // to recv[src_rank][m - rb(owner)][.] of the rank that finalises row m;
    // S = 1: into this CTA's own buffer
    constexpr int kH4 = kHC / 4;
    if (S > 1) {
      // Fire-and-forget remote stores instead of latency-bound remote loads.
      const int R = kM / S;
      const int owner = m / R, lm = m % R;
      const uint32_t dst = mapa(smem_u32(recv) + (uint32_t)((rank * R + lm) * kRecvRow + half * kH4) * 16u,
                                (uint32_t)owner);
      if (kAsyncPush) {
        if (ti == 0) cluster_wait();  // every rfull of the cluster is initialised
        // the peers' rows: (S - 1) x R rows x kN floats (S x R without kLocalPush)
        if (threadIdx.x == 0) mbar_arrive_expect_tx(rfull, (uint32_t)((kLocalPush ? S - 1 : S) * R * kN * 4));
      }
      if (kLocalPush && owner == rank) {
        // this CTA's own rows: plain shared stores (the __syncthreads below
        // orders them before the reduction); only the peers' rows travel
        float4* own = recv + (rank * R + lm) * kRecvRow + half * kH4;
#pragma unroll
        for (int c4 = 0; c4 < kH4; ++c4)
          own[c4] = make_float4(__uint_as_float(r0[4 * c4]), __uint_as_float(r0[4 * c4 + 1]),
                                __uint_as_float(r0[4 * c4 + 2]), __uint_as_float(r0[4 * c4 + 3]));
      } else if (kAsyncPush) {
        const uint32_t rbar = mapa(smem_u32(rfull), (uint32_t)owner);
#pragma unroll
        for (int c4 = 0; c4 < kH4; ++c4)
          st_async_f4(dst + 16u * (uint32_t)c4, __uint_as_float(r0[4 * c4]), __uint_as_float(r0[4 * c4 + 1]),
                      __uint_as_float(r0[4 * c4 + 2]), __uint_as_float(r0[4 * c4 + 3]), rbar);
      } else {
#pragma unroll
        for (int c4 = 0; c4 < kH4; ++c4)
          st_dsmem_f4(dst + 16u * (uint32_t)c4, __uint_as_float(r0[4 * c4]), __uint_as_float(r0[4 * c4 + 1]),
                      __uint_as_float(r0[4 * c4 + 2]), __uint_as_float(r0[4 * c4 + 3]));
      }
    } else {
#pragma unroll
      for (int c4 = 0; c4 < kH4; ++c4)
        recv[m * kRecvRow + half * kH4 + c4] =
            make_float4(__uint_as_float(r0[4 * c4]), __uint_as_float(r0[4 * c4 + 1]), __uint_as_float(r0[4 * c4 + 2]),
                        __uint_as_float(r0[4 * c4 + 3]));
    }
    PHASE(1);
    tc_fence_before();
    __syncthreads();  // hbuf complete; every TMEM read of this tile done (the next tile's MMAs may start)
    PHASE(5);
    {
      if (S > 1 && kAsyncPush) {
        mbar_wait_cluster(rfull, (uint32_t)(ti & 1));  // all S x R partial rows have landed
      } else if (S > 1) {
#ifdef MSPIPE_PHASES
        asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
        PHASE(7);
        asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
#else
        cluster_sync_all();  // all pushes into recv are visible
#endif
      }
      PHASE(6);
      const int R = kM / S;
      const int rb = rank * R;
      for (int it = threadIdx.x; it < R * kQ; it += kThreads) {
        const int lm = it / kQ, qq = it % kQ;
        const int mm = rb + lm;
        const int32_t u = m0 + mm;
        const int32_t j0 = jt * kJ + qq * 4;
        if (u >= U || j0 >= d.M) continue;
        float4 acc[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) acc[g] = recv[(0 * R + lm) * kRecvRow + g * kQ + qq];
        for (int sr = 1; sr < S; ++sr)  // fixed rank order: deterministic sum
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const float4 v = recv[(sr * R + lm) * kRecvRow + g * kQ + qq];
            acc[g].x += v.x;
            acc[g].y += v.y;
            acc[g].z += v.z;
            acc[g].w += v.w;
          }
        if (it == (int)threadIdx.x) PHASE(11);
        float pr[4], pz[4], pnx[4], pnh[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int jj = qq * 4 + e;
          pr[e] = (&acc[0].x)[e] + bias[jj];
          pz[e] = (&acc[1].x)[e] + bias[kJ + jj];
          pnx[e] = (&acc[2].x)[e] + bias[2 * kJ + jj];
          pnh[e] = (&acc[3].x)[e] + bias[3 * kJ + jj];
        }
#if defined(MSPIPE_PHASES) && defined(MSPIPE_DBG_NOSTORE)  // phase experiments only: the math without the stores
        {
          const float4 hv = gates4(pr, pz, pnx, pnh, hbuf[mm * kQ + qq], d.cell);
          if (hv.x == 12345.f) store_h4(a, u, rownode[mm], j0, hv);
        }
#elif defined(MSPIPE_PHASES) && defined(MSPIPE_DBG_NOMATH)  // phase experiments only: the stores without the math
        store_h4(a, u, rownode[mm], j0, make_float4(pr[0], pz[1], pnx[2], pnh[3]));
#else
        if (d.gates) {  // row F4: the backward of the gates reads the pre-activations (biases included)
          float4* gs = reinterpret_cast<float4*>(d.gates + (int64_t)u * 4 * d.M + j0);
          const int32_t q4 = d.M / 4;
          gs[0] = make_float4(pr[0], pr[1], pr[2], pr[3]);
          gs[q4] = make_float4(pz[0], pz[1], pz[2], pz[3]);
          gs[2 * q4] = make_float4(pnx[0], pnx[1], pnx[2], pnx[3]);
          gs[3 * q4] = make_float4(pnh[0], pnh[1], pnh[2], pnh[3]);
        }
        store_h4(a, u, rownode[mm], j0, gates4(pr, pz, pnx, pnh, hbuf[mm * kQ + qq], d.cell));
#endif
      }
      PHASE(10);
      if (a.commit_mem && !a.skip_meta) commit_rows(a, m0, U, rb, rb + R, jt, J, rownode);
      PHASE(8);
    }
    __syncthreads();  // hbuf / rownode / sbias are rewritten by the next tile's prefetch
    // single receive buffer: every CTA's reads of it precede the next tile's pushes
    if (S > 1 && q + gridDim.y < tiles) cluster_sync_all();
  }
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, tcols);
  }
}

// Row F3, deferred mailbox (TGL's TGN), A5: x = [S.mail[w] (Dm) | cos(w dt + p) | h = S.mem[w]],
// dt = t* - S.mem_ts[w]; one warp per (winner row, K chunk), as k_build_x.
__global__ void __launch_bounds__(256) k_build_deferred(GruDesc d, float* xbuf, const double* ts, int64_t B,
                                                        const float* snap_mem, const double* snap_ts,
                                                        const float* snap_mail, int64_t mail_stride, int64_t step,
                                                        const int32_t* winner, const int32_t* num_unique,
                                                        double* out_ts) {
  const int32_t U = __ldg(num_unique);
  const int32_t nchunks = d.Kpad / tc::kKC;
  const int64_t items = (int64_t)U * nchunks;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < items; w += nwarps) {
    const int32_t u = (int32_t)(w / nchunks), c = (int32_t)(w % nchunks);
    const int32_t k = c * tc::kKC + lane;
    const int32_t p = __ldg(winner + u);
    const int64_t ev = p >> 1;
    const int64_t rw = (p & 1) ? B + ev : ev;  // the winner's root row of the subgraph
    float v = 0.f;
    if (k < d.Dm) v = __ldg(snap_mail + rw * step * mail_stride + k);
    else if (k < d.Dx) {
      const float dt = (float)(__ldg(ts + ev) - __ldg(snap_ts + rw * step));
      v = time_cos(fmaf(__ldg(d.time_w + (k - d.Dm)), dt, __ldg(d.time_b + (k - d.Dm))));
    } else if (k < d.K) v = __ldg(snap_mem + rw * step * d.M + (k - d.Dx));
    tc::store_a(xbuf, nchunks, u, k, v);
    if (c == 0 && lane == 0) out_ts[u] = __ldg(ts + ev);
  }
}

cudaError_t launch_build_deferred(const GruDesc& d, float* xbuf, const double* ts, int64_t num_events,
                                  const float* snap_mem, const double* snap_mem_ts, const float* snap_mail,
                                  int64_t mail_stride, int64_t snap_step, const int32_t* winner,
                                  const int32_t* num_unique, double* out_ts, cudaStream_t s) {
  const int64_t warps = 2 * num_events * (d.Kpad / tc::kKC);
  int64_t blocks = (warps * 32 + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return launch_k(k_build_deferred, dim3((unsigned)blocks), dim3(256), 0, s, 1, d, xbuf, ts, num_events, snap_mem,
                  snap_mem_ts, snap_mail, mail_stride, snap_step, winner, num_unique, out_ts);
}

// Row F3, deferred mailbox, after the commit: the new mail of winner w (event
// ev, other endpoint o) from the committed memories, [mem[w] | mem[o] | e_ev]
// (o was updated in the same commit), mail_ts[w] = t_ev.  One warp per winner.
__global__ void __launch_bounds__(256) k_mail_deferred(const int32_t* src, const int32_t* dst, const double* ts,
                                                       const float* ef, int32_t He, const int32_t* nodes,
                                                       const int32_t* winner, const int32_t* num_unique,
                                                       const float* mem, int32_t M, float* mail, double* mail_ts,
                                                       int64_t mail_stride, int64_t num_nodes) {
  const int32_t U = __ldg(num_unique);
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < U; u += nwarps) {
    const int32_t w = __ldg(nodes + u), p = __ldg(winner + u);
    const int64_t ev = p >> 1;
    const int32_t o = (p & 1) ? __ldg(src + ev) : __ldg(dst + ev);
    if (w < 0 || w >= num_nodes || o < 0 || o >= num_nodes) continue;
    float* row = mail + (int64_t)w * mail_stride;
    for (int c = lane; c < mail_stride; c += 32) {
      float v = 0.f;
      if (c < M) v = mem[(int64_t)w * M + c];
      else if (c < 2 * M) v = mem[(int64_t)o * M + (c - M)];
      else if (c < 2 * M + He) v = __ldg(ef + ev * He + (c - 2 * M));
      row[c] = v;
    }
    if (lane == 0) mail_ts[w] = __ldg(ts + ev);
  }
}

void launch_mail_deferred(const int32_t* src, const int32_t* dst, const double* ts, const float* ef, int32_t He,
                          const int32_t* nodes, const int32_t* winner, const int32_t* num_unique, int64_t max_n,
                          const float* mem, int32_t M, float* mail, double* mail_ts, int64_t mail_stride,
                          int64_t num_nodes, cudaStream_t s) {
  int64_t blocks = (max_n * 32 + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  launch_k(k_mail_deferred, dim3((unsigned)blocks), dim3(256), 0, s, 1, src, dst, ts, ef, He, nodes, winner,
           num_unique, mem, M, mail, mail_ts, mail_stride, num_nodes);
}

// ---------------------------------------------------------------------------

constexpr int kMaxChunks = 512 / tc::kN;  // 6 buffers of 80 TMEM columns (the SM's TMEM: 512)

// co-resident clusters of S CTAs of k_gru_tc (cached per S; env MSPIPE_TC_CLUSTERS overrides)
static int64_t gru_tc_clusters(int S, bool bf16) {
  const int forced = env_int("MSPIPE_TC_CLUSTERS", 0);  // experiments: read at every launch
  if (forced > 0) return forced;
  static int64_t cache[2][17] = {};
  int64_t& c = cache[bf16 ? 1 : 0][S & 15];
  if (c > 0) return c;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)S, 1, 1);
  cfg.blockDim = dim3(tc::kThreads);
  cfg.dynamicSmemBytes = tc::kSmemBytes;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = (unsigned)S;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  const cudaError_t e = bf16 ? cudaOccupancyMaxActiveClusters(&n, k_gru_tc<true>, &cfg)
                             : cudaOccupancyMaxActiveClusters(&n, k_gru_tc<false>, &cfg);
  if (e != cudaSuccess || n <= 0) {
    (void)cudaGetLastError();
    n = num_sms() / S;
  }
  return c = n;
}

int gru_tc_splits(int64_t max_rows, const GruDesc& d, bool shared_buffers) {
  // K-split = cluster size.  Powers of two pack the GPCs (measured: 5-CTA
  // clusters of 1-CTA-per-SM blocks spill into a second wave, 4 do not).
  const int forced = env_int("MSPIPE_TC_SPLITS", 0);  // experiments only: read at every launch
  const int nchunks = d.Kpad / (d.bf16 ? tc::kKC16 : tc::kKC);
  // tf32: up to three K chunks share a TMEM buffer (36 MMAs per accumulator:
  // measured 0.47 of the 1e-4 tolerance at GDELT; four (48 MMAs) exceeded it
  // on one element); bf16: a single accumulator
  const int64_t s_min = d.bf16 ? 1 : (nchunks + 3 * kMaxChunks - 1) / (3 * kMaxChunks);
  if (forced > 0) return forced;  // below s_min the chunks share TMEM buffers (TcArgs::cpb)
  // big batches (GDELT's 2B = 8000, ~13 M tiles x 5 hidden tiles): S = 2, the
  // 130 CTAs in one wave, two K chunks per TMEM buffer (measured with the
  // 20-unit tile: 43.3 vs 44.6 us per GDELT step at S = 2 / 1, and S = 1
  // needs four chunks per buffer)
  if (shared_buffers && !d.bf16 && max_rows >= 4096)
    return (int)std::max<int64_t>(env_int("MSPIPE_TC_BIG_S", 2), s_min);
  const int64_t tiles = ((max_rows + tc::kM - 1) / tc::kM) * gru_tc_jtiles(d);
  int64_t s = 1;
  while (s < 8 && tiles * s * 2 <= 2 * (int64_t)num_sms() && s * 2 <= nchunks / 2) s *= 2;
  while (s < s_min) s *= 2;
  return (int)s;
}

cudaError_t launch_gru_tc(const GruDesc& d, const float* wtc, float* xbuf, const double* ts, int64_t num_events,
                          const float* edge_feat, const float* snap_mem, const double* snap_mem_ts,
                          int64_t snap_step, const float* snap_h, const int32_t* winner,
                          const int32_t* num_unique, float* out_mem, double* out_ts, float* out_mail,
                          int64_t mail_stride, cudaStream_t s, int parts, const GruCommit* commit,
                          const int32_t* tab_src, const int32_t* tab_dst) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_gru_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         tc::kSmemBytes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_gru_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::kSmemBytes);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_gru_tc<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_gru_tc<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  TcArgs a{d, wtc, xbuf, ts, num_events, edge_feat, snap_mem, snap_mem_ts, snap_step, snap_h, winner,
           num_unique, out_mem, out_ts, out_mail, mail_stride};
  if (commit) {
    a.nodes = commit->nodes;
    a.commit_mem = commit->mem;
    a.commit_mem_ts = commit->mem_ts;
    a.commit_mail = commit->mail;
    a.commit_mail_ts = commit->mail_ts;
    a.new_ts = commit->new_ts;
    a.new_mail = commit->new_mail;
    a.num_nodes = commit->num_nodes;
    a.mail_stride = commit->mail_stride;
    a.save_nodes = commit->save_nodes;
    a.save_num = commit->save_num;
    a.cu = commit->cu;
    a.h_from_mail = snap_mem == nullptr && snap_h == nullptr;
    a.skip_meta = commit->skip_meta;
    a.res_nodes = commit->res_nodes;
    a.res_num = commit->res_num;
  }
  a.tsrc = tab_src;
  a.tdst = tab_dst;
  const int64_t max_rows = 2 * num_events;
  const int64_t mtiles = (max_rows + tc::kM - 1) / tc::kM;
  if (parts & kGruBuild) {
    const int64_t nch = d.Kpad / (d.bf16 ? tc::kKC16 : tc::kKC);
    const int64_t warps = mtiles * (d.bf16 ? nch : (nch + kBuildChunks - 1) / kBuildChunks) * tc::kM;
    int64_t blocks = (warps * 32 + 255) / 256;
    const int64_t cap = (int64_t)num_sms() * env_int("MSPIPE_BUILD_BPS", 8);
    if (blocks > cap) blocks = cap;
    const bool row = !d.bf16 && env_int("MSPIPE_BUILD_ROW", 0) && d.Kpad / tc::kKC <= kBuildRowChunks;
    // items of 2 K chunks for small batches (more warps hide the gather latency: wiki 37.1 vs
    // 36.7 M events/s), 4 for large (GDELT 98.1 vs 96.4 M, r02zs); MSPIPE_BUILD_CHUNKS forces it
    const int bc = env_int("MSPIPE_BUILD_CHUNKS", max_rows <= 2048 ? 2 : kBuildChunks);
    const bool two = !d.bf16 && !row && bc == 2;
    if (two) {
      const int64_t w2 = mtiles * ((nch + 1) / 2) * tc::kM;
      blocks = std::min<int64_t>((w2 * 32 + 255) / 256, cap);
    }
    cudaError_t e = row   ? launch_k(k_build_x<kBuildRowChunks>, dim3((unsigned)blocks), dim3(256), 0, s, 1, a)
                    : two ? launch_k(k_build_x<2>, dim3((unsigned)blocks), dim3(256), 0, s, 1, a)
                          : launch_k(k_build_x<kBuildChunks>, dim3((unsigned)blocks), dim3(256), 0, s, 1, a);
    if (e != cudaSuccess) return e;
  }
  if (!(parts & kGruGemm)) return cudaSuccess;
  const int S = gru_tc_splits(max_rows, d, true);  // k_gru_tc: TMEM buffers may hold several chunks
  if (!d.bf16) {
    const int nchunks = d.Kpad / tc::kKC;
    const int nc_max = (nchunks + S - 1) / S;
    a.cpb = (nc_max + kMaxChunks - 1) / kMaxChunks;
  }
  // persistent grid: as many S-CTA clusters as are co-resident (one CTA per
  // SM: the stage ring fills shared memory), at most one per tile of the bound
  const int64_t max_tiles = mtiles * gru_tc_jtiles(d);
  const int64_t nclust = std::min<int64_t>(max_tiles, gru_tc_clusters(S, d.bf16));
  if (d.bf16)
    return launch_k(k_gru_tc<true>, dim3((unsigned)S, (unsigned)nclust), dim3(tc::kThreads), tc::kSmemBytes, s,
                    (unsigned)S, a);
  return launch_k(k_gru_tc<false>, dim3((unsigned)S, (unsigned)nclust), dim3(tc::kThreads), tc::kSmemBytes, s,
                  (unsigned)S, a);
}

}  // namespace mspipe

#ifdef MSPIPE_PHASES
extern "C" __attribute__((visibility("default"))) int mspipe_debug_phases(void* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, mspipe::g_phase, sizeof(unsigned long long) * 16 * n);
}
#endif
