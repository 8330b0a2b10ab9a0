// train.cu — row F4: the MTGNN training stage of one iteration on the GPU
// ("the memory updater computes the updated memory, the MTGNN layer computes
// the embeddings, and the loss and backward steps are performed (including
// all-reduce)"; Eq. 2 h = emb(s~_v, s~_u | u ∈ N(v))).
// Readings T1-T7 (oracle/train.py):
//   T1 s~ of a subgraph node = the batch's GRU output h' if it is a winner,
//      else the fetched snapshot row;  T2 gradients reach the GRU weights
//      through h' only;  T3 single-head temporal attention, H = emb_dim;
//   T4 TGN link decoder;  T5 mean BCE on logits;  T6 SGD;  T7 DP mean.
//
// The contractions (projections, their weight and input gradients, the
// GRU weight gradient) are plain GEMMs on cuBLAS, row-major through the
// transposed-operand identity: the three over the 3B·𝒩 neighbour slots (the
// K|V projection, its weight gradient and its input gradient: ~85 % of the
// step's FLOPs) in 3xTF32 on the tensor cores (operands split into tf32
// hi | lo by their producers, three TF32 GEMMs accumulated in fp32: fp32
// accuracy), the small rest in SGEMM (default math: no TF32).  The gathers, the
// per-root attention (≤ 𝒩 = 10 neighbours, one warp per root), the decoder's
// nonlinearity and loss, the deterministic scatter of the node gradients into
// the winners' h' rows (stable radix sort of (winner, slot) pairs, then one
// warp per winner sums its slots in slot order) and the GRU's gate backward
// are hand-written kernels.  Every reduction has a fixed order: the step is
// bitwise deterministic.
#include <cublas_v2.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>

#include "internal.cuh"
#include "tc_layout.cuh"

using namespace mspipe;

namespace {

constexpr int kTrThreads = 256;
constexpr int32_t kNoWinner = 0x7fff;  // sort key of a slot whose node is not a winner (2B <= 16384 < 2^15)
enum { P_WQ, P_WK, P_WV, P_WO, P_BO, P_W1, P_B1, P_W2, P_B2, P_WIH, P_WHH, P_BIH, P_BHH, P_N };

struct Dims {
  int32_t M, He, Dt, Dx, K, H, F;
};

int64_t layout(const Dims& d, int64_t off[P_N]) {
  const int64_t M = d.M, H = d.H, Z = d.M + d.Dt;
  const int64_t sz[P_N] = {H * M, H * Z, H * Z, H * (H + M), H, H * 2 * H, H, H, 1,
                           3 * M * d.Dx, 3 * M * M, 3 * M, 3 * M};
  int64_t o = 0;
  for (int i = 0; i < P_N; ++i) {
    off[i] = o;
    o += (sz[i] + 3) / 4 * 4;  // 16-byte aligned tensors
  }
  return o;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int64_t gwarp() { return ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; }
__device__ __forceinline__ int64_t nwarps() { return ((int64_t)gridDim.x * blockDim.x) >> 5; }
__device__ __forceinline__ int64_t gthread() { return (int64_t)blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int64_t nthreads() { return (int64_t)gridDim.x * blockDim.x; }

// wmap[node] = winner row u (set) or -1 (clear)
__global__ void k_tr_map(const int32_t* __restrict__ nodes, const int32_t* __restrict__ num, int32_t* wmap,
                         int set) {
  const int32_t U = __ldg(num);
  for (int64_t u = gthread(); u < U; u += nthreads()) wmap[__ldg(nodes + u)] = set ? (int32_t)u : -1;
}

// T1 + the attention inputs: one warp per root r and slot s in [0, F]:
//   s == 0: sroot[r] = s~(root);  s >= 1: zn[r, s-1] = [s~(nbr) ‖ φ(Δt)] or 0;
//   key[slot] = winner row of the slot's node (kNoWinner if none), val[slot] = slot
__global__ void __launch_bounds__(kTrThreads) k_tr_gather(
    Dims d, int64_t R, const int32_t* __restrict__ sub, const float* __restrict__ sdt,
    const int32_t* __restrict__ cnt, const float* __restrict__ snap, const int32_t* __restrict__ wmap,
    const float* __restrict__ hn, const float* __restrict__ tw, const float* __restrict__ tb, float* sroot,
    float* zn, float* zn_lo, int32_t* key, int32_t* val) {
  const int lane = threadIdx.x & 31;
  const int32_t F = d.F, M = d.M, Z = d.M + d.Dt;
  for (int64_t slot = gwarp(); slot < R * (F + 1); slot += nwarps()) {  // one warp per (root, slot)
    const int64_t r = slot / (F + 1);
    const int32_t s = (int32_t)(slot % (F + 1));
    const int32_t c = __ldg(cnt + r);
    {
      const int32_t id = __ldg(sub + slot);
      const bool valid = id >= 0 && (s == 0 || s - 1 < c);
      const int32_t u = valid ? __ldg(wmap + id) : -1;
      if (lane == 0) {
        key[slot] = u >= 0 ? u : kNoWinner;
        val[slot] = (int32_t)slot;
      }
      const float* row = u >= 0 ? hn + (int64_t)u * M : snap + slot * M;
      if (s == 0) {
        float* out = sroot + r * M;
        for (int32_t k = lane; k < M; k += 32) out[k] = valid ? __ldg(row + k) : 0.f;
      } else {  // neighbour rows feed the 3xTF32 projections: tf32 hi | lo images
        float* out = zn + (r * F + s - 1) * Z;
        float* olo = zn_lo + (r * F + s - 1) * Z;
        const float dt = __ldg(sdt + r * F + s - 1);
        for (int32_t k = lane; k < Z; k += 32) {
          const float v = !valid ? 0.f
                          : k < M ? __ldg(row + k) : time_cos(fmaf(__ldg(tw + k - M), dt, __ldg(tb + k - M)));
          const float hi = tc::tf32_rna(v);
          out[k] = hi;
          olo[k] = tc::tf32_rna(v - hi);
        }
      }
    }
  }
}

// T3 forward, one warp per root: α = softmax(q·k_u / √H) over the cnt valid
// neighbours (lane u holds score u, F <= 31), a = Σ α_u v_u, zo[r] = [a ‖ s~(root)]
__global__ void __launch_bounds__(kTrThreads) k_tr_attn_fwd(Dims d, int64_t R, const int32_t* __restrict__ cnt,
                                                            const float* __restrict__ q,
                                                            const float* __restrict__ kv,
                                                            const float* __restrict__ sroot, float* alpha,
                                                            float* zo) {
  __shared__ float s_al[kTrThreads / 32][32];  // the warp's α (lane = neighbour): no shuffles in ragged loops
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int32_t F = d.F, H = d.H, M = d.M;
  const float scale = rsqrtf((float)H);
  for (int64_t r = gwarp(); r < R; r += nwarps()) {
    const int32_t c = __ldg(cnt + r);
    const float* qr = q + r * H;
    float my = -INFINITY;
    for (int32_t u = 0; u < c; ++u) {
      const float* kr = kv + (r * F + u) * 2 * H;
      float p = 0.f;
      for (int32_t h = lane; h < H; h += 32) p += __ldg(qr + h) * __ldg(kr + h);
      p = warp_sum(p) * scale;
      if (lane == u) my = p;
    }
    float mx = my;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float e = lane < c ? expf(my - mx) : 0.f;
    const float den = warp_sum(e);
    const float a_l = lane < c ? e / den : 0.f;
    if (lane < F) alpha[r * F + lane] = a_l;
    __syncwarp();
    s_al[wib][lane] = a_l;
    __syncwarp();
    float* out = zo + r * (H + M);
    for (int32_t h = lane; h < H; h += 32) {
      float acc = 0.f;
      for (int32_t u = 0; u < c; ++u) acc += s_al[wib][u] * __ldg(kv + (r * F + u) * 2 * H + H + h);
      out[h] = acc;
    }
    if (c == 0)
      for (int32_t h = lane; h < H; h += 32) out[h] = 0.f;
    for (int32_t k = lane; k < M; k += 32) out[H + k] = __ldg(sroot + r * M + k);
  }
}

// T4 input: pair p < B = (src_p, dst_p), pair B + j = (src_j, neg_j); emb rows + b_o
__global__ void k_tr_dec_in(int64_t B, int32_t H, const float* __restrict__ emb, const float* __restrict__ b_o,
                            float* za) {
  const int64_t total = 2 * B * 2 * H;
  for (int64_t t = gthread(); t < total; t += nthreads()) {
    const int64_t p = t / (2 * H);
    const int32_t c = (int32_t)(t % (2 * H));
    const int64_t j = p % B;
    const int64_t root = c < H ? j : (p < B ? B + j : 2 * B + j);
    const int32_t h = c < H ? c : c - H;
    za[t] = __ldg(emb + root * H + h) + __ldg(b_o + h);
  }
}

__device__ __forceinline__ double softplus_d(double x) { return fmax(x, 0.0) + log1p(exp(-fabs(x))); }

// T4 + T5, one warp per pair: y = tanh(pre + b_1), logit = w_2·y + b_2, the
// BCE term (f64), dlogit = (σ(logit) - label) / 2B, dpre = dlogit w_2 (1 - y²)
__global__ void __launch_bounds__(kTrThreads) k_tr_dec_out(int64_t B, int32_t H, const float* __restrict__ pre,
                                                           const float* __restrict__ b_1,
                                                           const float* __restrict__ w_2,
                                                           const float* __restrict__ b_2, float* y,
                                                           float* logit, float* dlogit, double* term,
                                                           float* dpre) {
  const int lane = threadIdx.x & 31;
  for (int64_t p = gwarp(); p < 2 * B; p += nwarps()) {
    float acc = 0.f;
    for (int32_t h = lane; h < H; h += 32) {
      const float v = tanhf(__ldg(pre + p * H + h) + __ldg(b_1 + h));
      y[p * H + h] = v;
      acc += __ldg(w_2 + h) * v;
    }
    const float l = warp_sum(acc) + __ldg(b_2);
    const bool pos = p < B;
    const float g = (1.f / (1.f + expf(-l)) - (pos ? 1.f : 0.f)) / (float)(2 * B);
    if (lane == 0) {
      logit[p] = l;
      dlogit[p] = g;
      term[p] = pos ? softplus_d(-(double)l) : softplus_d((double)l);
    }
    for (int32_t h = lane; h < H; h += 32) {
      const float v = y[p * H + h];
      dpre[p * H + h] = g * __ldg(w_2 + h) * (1.f - v * v);
    }
  }
}

// mean of the 2B loss terms in a fixed order (one block)
__global__ void __launch_bounds__(1024) k_tr_loss(int64_t n, const double* __restrict__ term, double* loss) {
  __shared__ double part[1024];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += term[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = part[0] / (double)n;
}

// dE of the 3B roots from the decoder input gradient dza [2B, 2H]
__global__ void k_tr_dec_scatter(int64_t B, int32_t H, const float* __restrict__ dza, float* demb) {
  const int64_t total = 3 * B * H;
  for (int64_t t = gthread(); t < total; t += nthreads()) {
    const int64_t r = t / H;
    const int32_t h = (int32_t)(t % H);
    float v;
    if (r < B) v = __ldg(dza + r * 2 * H + h) + __ldg(dza + (B + r) * 2 * H + h);
    else if (r < 2 * B) v = __ldg(dza + (r - B) * 2 * H + H + h);
    else v = __ldg(dza + (r - B) * 2 * H + H + h);
    demb[t] = v;
  }
}

// T3 backward, one warp per root: da = dzo[r, :H];
//   dα_u = da·v_u, dv_u = α_u da, dscore_u = α_u (dα_u - Σ α dα),
//   dq = Σ dscore_u k_u / √H, dk_u = dscore_u q / √H
__global__ void __launch_bounds__(kTrThreads) k_tr_attn_bwd(Dims d, int64_t R, const int32_t* __restrict__ cnt,
                                                            const float* __restrict__ q,
                                                            const float* __restrict__ kv,
                                                            const float* __restrict__ alpha,
                                                            const float* __restrict__ dzo, float* dq,
                                                            float* dkv, float* dkv_lo) {
  __shared__ float s_ds[kTrThreads / 32][32], s_al[kTrThreads / 32][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int32_t F = d.F, H = d.H, M = d.M;
  const float scale = rsqrtf((float)H);
  for (int64_t r = gwarp(); r < R; r += nwarps()) {
    const int32_t c = __ldg(cnt + r);
    const float* da = dzo + r * (H + M);
    float my_da = 0.f;  // dα of lane u
    for (int32_t u = 0; u < c; ++u) {
      float p = 0.f;
      for (int32_t h = lane; h < H; h += 32) p += __ldg(da + h) * __ldg(kv + (r * F + u) * 2 * H + H + h);
      p = warp_sum(p);
      if (lane == u) my_da = p;
    }
    const float al = lane < F ? __ldg(alpha + r * F + lane) : 0.f;
    const float sdot = warp_sum(lane < c ? al * my_da : 0.f);
    const float ds = lane < c ? al * (my_da - sdot) : 0.f;
    __syncwarp();
    s_ds[wib][lane] = ds;
    s_al[wib][lane] = al;
    __syncwarp();
    for (int32_t h = lane; h < H; h += 32) {
      float acc = 0.f;
      for (int32_t u = 0; u < c; ++u) acc += s_ds[wib][u] * __ldg(kv + (r * F + u) * 2 * H + h);
      dq[r * H + h] = acc * scale;
    }
    for (int32_t u = 0; u < F; ++u) {
      const float dsu = s_ds[wib][u];
      const float au = s_al[wib][u];
      float* o = dkv + (r * F + u) * 2 * H;
      float* ol = dkv_lo + (r * F + u) * 2 * H;
      for (int32_t h = lane; h < H; h += 32) {
        const float dk = u < c ? dsu * __ldg(q + r * H + h) * scale : 0.f;
        const float dv = u < c ? au * __ldg(da + h) : 0.f;
        const float kh = tc::tf32_rna(dk), vh = tc::tf32_rna(dv);
        o[h] = kh;
        o[H + h] = vh;
        ol[h] = tc::tf32_rna(dk - kh);
        ol[H + h] = tc::tf32_rna(dv - vh);
      }
    }
  }
}

// dh'[u] = Σ over the slots whose node is winner u (keys sorted).  A hot node
// is referenced by tens of thousands of neighbour slots, so every winner's
// segment is cut into pieces of kPiece slots, each summed by one block (8 slot
// lanes x float4 column groups, the lanes' partials added in lane order), and
// the pieces of a winner are added in piece order: a fixed order, so the sum
// is deterministic.  Rows u in [U, 2B) are zero (the GEMMs run over 2B rows).
constexpr int kSegLanes = kTrThreads / 32;
constexpr int64_t kPiece = 512;

// segment bounds of every winner from the sorted keys in one parallel pass:
// position i starts a run when key[i] != key[i - 1] (lo of key[i], hi of key[i - 1]);
// winners without slots keep lo = hi = 0 (lo_hi zeroed first)
__global__ void k_tr_seg_bounds(int64_t nslots, const int32_t* __restrict__ skey, int64_t* lo_hi) {
  for (int64_t i = gthread(); i <= nslots; i += nthreads()) {
    const int32_t k = i < nslots ? __ldg(skey + i) : kNoWinner;
    const int32_t kp = i > 0 ? __ldg(skey + i - 1) : -1;
    if (k == kp) continue;
    if (kp >= 0 && kp != kNoWinner) lo_hi[2 * kp + 1] = i;
    if (k != kNoWinner) lo_hi[2 * k] = i;
  }
}

// one block: the exclusive scan of the winners' piece counts
__global__ void __launch_bounds__(1024) k_tr_seg_plan(int64_t B2, const int32_t* __restrict__ num,
                                                       const int64_t* __restrict__ lo_hi, int64_t* poff) {
  __shared__ int64_t carry;
  __shared__ int64_t wsum[32];
  const int32_t U = __ldg(num);
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < B2; base += blockDim.x) {
    const int64_t u = base + threadIdx.x;
    int64_t n = 0;
    if (u < U) n = (lo_hi[2 * u + 1] - lo_hi[2 * u] + kPiece - 1) / kPiece;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t x = n;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      int64_t v = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      wsum[lane] = v;
    }
    __syncthreads();
    const int64_t incl = x + (w > 0 ? wsum[w - 1] : 0);
    if (u < B2) poff[u] = carry + incl - n;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry += incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) poff[B2] = carry;
}

// pass 1: block per piece p (grid-stride over the bound): rows of slots [start, end)
__global__ void __launch_bounds__(kTrThreads) k_tr_seg_piece(Dims d, int64_t B2, const int64_t* __restrict__ lo_hi,
                                                             const int64_t* __restrict__ poff,
                                                             const int32_t* __restrict__ sval,
                                                             const float* __restrict__ dzo,
                                                             const float* __restrict__ dzn, float* part) {
  __shared__ float4 lanes[kSegLanes][32];
  const int g = threadIdx.x & 31, sl = threadIdx.x >> 5;
  const int32_t F = d.F, H = d.H, M = d.M, Q = d.M / 4;
  const int64_t total = poff[B2];
  for (int64_t p = blockIdx.x; p < total; p += gridDim.x) {
    int64_t a = 0, b = B2;  // the winner u with poff[u] <= p < poff[u + 1]
    while (a < b) {
      const int64_t m = (a + b) >> 1;
      if (poff[m + 1] <= p) a = m + 1; else b = m;
    }
    const int64_t u = a;
    const int64_t start = lo_hi[2 * u] + (p - poff[u]) * kPiece;
    const int64_t end = min(start + kPiece, lo_hi[2 * u + 1]);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (g < Q)
      for (int64_t i = start + sl; i < end; i += kSegLanes) {
        const int64_t slot = __ldg(sval + i);
        const int64_t r = slot / (F + 1);
        const int32_t s = (int32_t)(slot % (F + 1));
        const float4 v = s == 0 ? __ldg(reinterpret_cast<const float4*>(dzo + r * (H + M) + H) + g)
                                : __ldg(reinterpret_cast<const float4*>(dzn + (r * F + s - 1) * M) + g);
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
    lanes[sl][g] = acc;
    __syncthreads();
    if (sl == 0 && g < Q) {
      float4 t = lanes[0][g];
      for (int q = 1; q < kSegLanes; ++q) {
        t.x += lanes[q][g].x;
        t.y += lanes[q][g].y;
        t.z += lanes[q][g].z;
        t.w += lanes[q][g].w;
      }
      reinterpret_cast<float4*>(part + p * M)[g] = t;
    }
    __syncthreads();
  }
}

// pass 2: thread per (u, float4 group): the winner's pieces in piece order
__global__ void k_tr_seg_final(int32_t M, int64_t B2, const int64_t* __restrict__ poff,
                               const float* __restrict__ part, float* dhn) {
  const int32_t Q = M / 4;
  for (int64_t t = gthread(); t < B2 * Q; t += nthreads()) {
    const int64_t u = t / Q;
    const int32_t g = (int32_t)(t % Q);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t p = poff[u]; p < poff[u + 1]; ++p) {
      const float4 v = reinterpret_cast<const float4*>(part + p * M)[g];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    reinterpret_cast<float4*>(dhn + u * M)[g] = acc;
  }
}

// the GEMM operand X = [x | h] of winner row u, column k (A image: hi + lo)
__device__ __forceinline__ float x_elem(const float* xbuf, int32_t nchunks, int64_t u, int32_t k) {
  const char* blk = reinterpret_cast<const char*>(xbuf) + ((u / tc::kM) * nchunks + k / tc::kKC) * tc::kABlock;
  const uint32_t off = tc::sw128_off((uint32_t)(u % tc::kM), (uint32_t)(k % tc::kKC));
  return __ldg(reinterpret_cast<const float*>(blk + off)) + __ldg(reinterpret_cast<const float*>(blk + tc::kATile + off));
}

// GRU backward of the gates (chain rule of torch.nn.GRUCell, G5) per (u, j):
//   D[u] = [d pre_r | d pre_z | d pre_n(x) | d (W_hn h + b_hn)], and X plain [2B, K]
__global__ void k_tr_gru_bwd(Dims d, int64_t B2, int32_t nchunks, const int32_t* __restrict__ num,
                             const float* __restrict__ xbuf, const float* __restrict__ gates,
                             const float* __restrict__ dhn, float* D, float* xp) {
  const int32_t U = __ldg(num);
  const int32_t M = d.M, K = d.K;
  for (int64_t t = gthread(); t < B2 * K; t += nthreads()) {
    const int64_t u = t / K;
    const int32_t k = (int32_t)(t % K);
    xp[t] = u < U ? x_elem(xbuf, nchunks, u, k) : 0.f;
  }
  for (int64_t t = gthread(); t < B2 * M; t += nthreads()) {
    const int64_t u = t / M;
    const int32_t j = (int32_t)(t % M);
    float* o = D + u * 4 * M;
    if (u >= U) {
      o[j] = o[M + j] = o[2 * M + j] = o[3 * M + j] = 0.f;
      continue;
    }
    const float* g = gates + u * 4 * M;
    const float r = 1.f / (1.f + expf(-__ldg(g + j)));
    const float z = 1.f / (1.f + expf(-__ldg(g + M + j)));
    const float ghn = __ldg(g + 3 * M + j);
    const float n = tanhf(__ldg(g + 2 * M + j) + r * ghn);
    const float h = x_elem(xbuf, nchunks, u, d.Dx + j);
    const float dh = __ldg(dhn + t);
    const float dn = dh * (1.f - z);
    const float dz = dh * (h - n);
    const float dan = dn * (1.f - n * n);
    o[j] = dan * ghn * r * (1.f - r);
    o[M + j] = dz * z * (1.f - z);
    o[2 * M + j] = dan;
    o[3 * M + j] = dan * r;
  }
}

// bias gradients from the column sums cs = D^T 1 [4M]: b_ih = [r, z, n_x], b_hh = [r, z, n_h]
__global__ void k_tr_gru_bias(int32_t M, const float* __restrict__ cs, float* gbih, float* gbhh) {
  for (int64_t t = gthread(); t < 3 * M; t += nthreads()) {
    gbih[t] = cs[t];
    gbhh[t] = t < 2 * M ? cs[t] : cs[M + t];
  }
}

__global__ void k_tr_sgd(int64_t n, float lr, const float* __restrict__ g, float* p) {
  for (int64_t t = gthread(); t < n; t += nthreads()) p[t] -= lr * g[t];
}

__global__ void k_tr_fill(int64_t n, float v, float* p) {
  for (int64_t t = gthread(); t < n; t += nthreads()) p[t] = v;
}

__global__ void k_tr_split(int64_t n, const float* __restrict__ x, float* hi, float* lo) {
  for (int64_t t = gthread(); t < n; t += nthreads()) {
    const float v = x[t];
    const float h = tc::tf32_rna(v);
    hi[t] = h;
    lo[t] = tc::tf32_rna(v - h);
  }
}

// row-major C = op(A) op(B) on the tensor cores in 3xTF32 (A = A_hi + A_lo, B = B_hi + B_lo,
// every part tf32-representable, so each product is exact and the sums are fp32):
//   C = A_lo B_hi + A_hi B_lo + A_hi B_hi   (the dropped A_lo B_lo ~ 2^-22 relative)
cublasStatus_t gemm_tf32(cublasHandle_t h, bool ta, bool tb, int64_t m, int64_t n, int64_t k, const float* A,
                         int64_t lda, const float* B, int64_t ldb, float beta, float* C, int64_t ldc) {
  const float one = 1.f;
  return cublasGemmEx(h, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N, (int)n, (int)m, (int)k, &one,
                      B, CUDA_R_32F, (int)ldb, A, CUDA_R_32F, (int)lda, &beta, C, CUDA_R_32F, (int)ldc,
                      CUBLAS_COMPUTE_32F_FAST_TF32, CUBLAS_GEMM_DEFAULT);
}
cublasStatus_t gemm3(cublasHandle_t h, bool ta, bool tb, int64_t m, int64_t n, int64_t k, const float* Ahi,
                     const float* Alo, int64_t lda, const float* Bhi, const float* Blo, int64_t ldb, float* C,
                     int64_t ldc) {
  cublasStatus_t st = gemm_tf32(h, ta, tb, m, n, k, Alo, lda, Bhi, ldb, 0.f, C, ldc);
  if (st == CUBLAS_STATUS_SUCCESS) st = gemm_tf32(h, ta, tb, m, n, k, Ahi, lda, Blo, ldb, 1.f, C, ldc);
  if (st == CUBLAS_STATUS_SUCCESS) st = gemm_tf32(h, ta, tb, m, n, k, Ahi, lda, Bhi, ldb, 1.f, C, ldc);
  return st;
}

// long-K weight gradient C[m, n] = A^T B (A [K, m], B [K, n] row-major) in 3xTF32: the
// tensor core's fp32 accumulation truncates, so K is cut into chunks of kChunkK rows
// (64 MMA k-steps each), one strided-batched GEMM per term writes the chunk partials,
// and the partials are added on the CUDA cores in chunk order (deterministic)
constexpr int64_t kChunkK = 512;
cublasStatus_t gemm3_tn_chunked(cublasHandle_t h, int64_t m, int64_t n, int64_t K, const float* Ahi,
                                const float* Alo, int64_t lda, const float* Bhi, const float* Blo, int64_t ldb,
                                float* part, int64_t nparts) {
  const float one = 1.f, zero = 0.f;
  const float* As[3] = {Alo, Ahi, Ahi};
  const float* Bs[3] = {Bhi, Blo, Bhi};
  for (int t = 0; t < 3; ++t) {
    cublasStatus_t st = cublasGemmStridedBatchedEx(
        h, CUBLAS_OP_N, CUBLAS_OP_T, (int)n, (int)m, (int)kChunkK, &one, Bs[t], CUDA_R_32F, (int)ldb, kChunkK * ldb,
        As[t], CUDA_R_32F, (int)lda, kChunkK * lda, t ? &one : &zero, part, CUDA_R_32F, (int)n, m * n, (int)nparts,
        CUBLAS_COMPUTE_32F_FAST_TF32, CUBLAS_GEMM_DEFAULT);
    if (st != CUBLAS_STATUS_SUCCESS) return st;
  }
  (void)K;
  return CUBLAS_STATUS_SUCCESS;
}

// out[i] = Σ_p part[p][i] in p order (+ tail[i] when given: the last, partial chunk)
__global__ void k_tr_sum_parts(int64_t n, int64_t nparts, const float* __restrict__ part,
                               const float* __restrict__ tail, float* out) {
  for (int64_t i = gthread(); i < n; i += nthreads()) {
    float acc = 0.f;
    for (int64_t p = 0; p < nparts; ++p) acc += part[p * n + i];
    if (tail) acc += tail[i];
    out[i] = acc;
  }
}

// row-major C[m, n] = alpha op(A)[m, k] op(B)[k, n] + beta C (column-major cuBLAS on the transposes)
cublasStatus_t gemm_rm(cublasHandle_t h, bool ta, bool tb, int64_t m, int64_t n, int64_t k, const float* A,
                       int64_t lda, const float* B, int64_t ldb, float beta, float* C, int64_t ldc) {
  const float one = 1.f;
  return cublasSgemm(h, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N, (int)n, (int)m, (int)k,
                     &one, B, (int)ldb, A, (int)lda, &beta, C, (int)ldc);
}

// colsum of row-major X [rows, cols] (ld) into y [cols]: X^T 1
cublasStatus_t colsum(cublasHandle_t h, int64_t rows, int64_t cols, const float* X, int64_t ld, const float* ones,
                      float* y) {
  const float one = 1.f, zero = 0.f;
  return cublasSgemv(h, CUBLAS_OP_N, (int)cols, (int)rows, &one, X, (int)ld, ones, 1, &zero, y, 1);
}

unsigned grid_for(int64_t work, int per_block) {
  int64_t b = (work + per_block - 1) / per_block;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (b > cap) b = cap;
  return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace

struct mspipe_train {
  Dims d;
  int64_t num_nodes, max_events;
  int64_t off[P_N];
  int64_t total;
  float* params;  // caller-owned device [total]
  float* grads;   // caller-owned device [total]
  // workspace (handle-owned)
  int32_t* wmap;
  float *sroot, *zn, *q, *kv, *alpha, *zo, *emb, *za, *pre, *y, *logit, *dlogit, *dpre, *dza, *demb, *dzo, *dq, *dkv,
      *dzn, *dhn, *D, *xp, *ones, *cs;
  float *zn_lo, *dkv_lo, *wkv_hi, *wkv_lo;  // 3xTF32 parts (zn / dkv hold the hi parts)
  float* wpart;                             // chunk partials of dW_k | dW_v [RF / kChunkK + 1, 2H, Z]
  double* term;
  int32_t *key, *val, *skey, *sval;
  int64_t *lo_hi, *poff;  // per winner: its sorted segment, exclusive scan of its piece counts
  float* part;            // piece sums [slots / kPiece + 2B + 1, M]
  void* sort_tmp;
  size_t sort_bytes;
  void* blas_ws;  // cuBLAS workspace owned here: no allocation inside a CUDA-graph capture
  cublasHandle_t blas;
};

static void train_free(mspipe_train* t) {
  if (!t) return;
  void* bufs[] = {t->wmap, t->sroot, t->zn, t->q, t->kv, t->alpha, t->zo, t->emb, t->za, t->pre, t->y, t->logit,
                  t->dlogit, t->dpre, t->dza, t->demb, t->dzo, t->dq, t->dkv, t->dzn, t->dhn, t->D, t->xp, t->ones,
                  t->cs, t->term, t->key, t->val, t->skey, t->sval, t->sort_tmp, t->blas_ws, t->lo_hi, t->poff, t->part,
                  t->zn_lo, t->dkv_lo, t->wkv_hi, t->wkv_lo, t->wpart};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (t->blas) cublasDestroy(t->blas);
  delete t;
}

int64_t mspipe_train_layout(int32_t mem_dim, int32_t edge_dim, int32_t time_dim, int32_t emb_dim,
                            int64_t* offsets) {
  if (mem_dim <= 0 || edge_dim < 0 || time_dim <= 0 || emb_dim <= 0) return -1;
  const int32_t Dx = 2 * mem_dim + edge_dim + time_dim;
  Dims d{mem_dim, edge_dim, time_dim, Dx, Dx + mem_dim, emb_dim, 0};
  int64_t off[P_N];
  const int64_t total = layout(d, off);
  if (offsets)
    for (int i = 0; i < P_N; ++i) offsets[i] = off[i];
  return total;
}

mspipe_status mspipe_train_create(mspipe_train** out, const mspipe_gru* gru, int64_t num_nodes, int32_t emb_dim,
                                  int32_t fanout, int64_t max_events, float* params, float* grads, void* stream) {
  if (!out) return fail(MSPIPE_EINVAL, "train_create: out is NULL");
  *out = nullptr;
  if (!gru || !params || !grads) return fail(MSPIPE_EINVAL, "train_create: NULL gru / params / grads");
  if (gru->precision != MSPIPE_FP32_3XTF32 || gru->d.cell != MSPIPE_CELL_GRU ||
      gru->d.mailbox != MSPIPE_MAILBOX_IMMEDIATE)
    return fail(MSPIPE_EUNSUPPORTED, "train_create: needs a GRUCell, immediate-mailbox, MSPIPE_FP32_3XTF32 updater");
  if (gru->d.M > 128) return fail(MSPIPE_EUNSUPPORTED, "train_create: mem_dim <= 128 (one float4 group per lane)");
  if (num_nodes <= 0 || emb_dim <= 0 || fanout < 1 || fanout > 31 || max_events <= 0 ||
      max_events > gru->max_events || 2 * max_events > kNoWinner)
    return fail(MSPIPE_EINVAL, "train_create: num_nodes=%lld emb_dim=%d fanout=%d max_events=%lld",
                (long long)num_nodes, emb_dim, fanout, (long long)max_events);
  mspipe_train* t = new mspipe_train();
  const GruDesc& g = gru->d;
  t->d = Dims{g.M, g.He, g.Dt, g.Dx, g.K, emb_dim, fanout};
  t->num_nodes = num_nodes;
  t->max_events = max_events;
  t->total = layout(t->d, t->off);
  t->params = params;
  t->grads = grads;
  const int64_t B = max_events, R = 3 * B, F = fanout, M = g.M, H = emb_dim, Z = g.M + g.Dt;
  const int64_t slots = R * (F + 1);
  cudaError_t e = cudaSuccess;
  auto af = [&](float** p, int64_t n) {
    if (e == cudaSuccess) e = cudaMalloc(p, sizeof(float) * (size_t)(n > 0 ? n : 1));
  };
  if (e == cudaSuccess) e = cudaMalloc(&t->wmap, sizeof(int32_t) * (size_t)num_nodes);
  af(&t->sroot, R * M);
  af(&t->zn, R * F * Z);
  af(&t->q, R * H);
  af(&t->kv, R * F * 2 * H);
  af(&t->alpha, R * F);
  af(&t->zo, R * (H + M));
  af(&t->emb, R * H);
  af(&t->za, 2 * B * 2 * H);
  af(&t->pre, 2 * B * H);
  af(&t->y, 2 * B * H);
  af(&t->logit, 2 * B);
  af(&t->dlogit, 2 * B);
  af(&t->dpre, 2 * B * H);
  af(&t->dza, 2 * B * 2 * H);
  af(&t->demb, R * H);
  af(&t->dzo, R * (H + M));
  af(&t->dq, R * H);
  af(&t->dkv, R * F * 2 * H);
  af(&t->dzn, R * F * M);
  af(&t->zn_lo, R * F * Z);
  af(&t->dkv_lo, R * F * 2 * H);
  af(&t->wkv_hi, 2 * H * Z);
  af(&t->wkv_lo, 2 * H * Z);
  af(&t->wpart, (R * F / kChunkK + 1) * 2 * H * Z);
  af(&t->dhn, 2 * B * M);
  af(&t->D, 2 * B * 4 * M);
  af(&t->xp, 2 * B * g.K);
  af(&t->ones, std::max<int64_t>(R * F, 4 * M));
  af(&t->cs, 4 * M);
  if (e == cudaSuccess) e = cudaMalloc(&t->term, sizeof(double) * (size_t)(2 * B + 1));
  if (e == cudaSuccess) e = cudaMalloc(&t->key, sizeof(int32_t) * (size_t)slots);
  if (e == cudaSuccess) e = cudaMalloc(&t->val, sizeof(int32_t) * (size_t)slots);
  if (e == cudaSuccess) e = cudaMalloc(&t->skey, sizeof(int32_t) * (size_t)slots);
  if (e == cudaSuccess) e = cudaMalloc(&t->sval, sizeof(int32_t) * (size_t)slots);
  if (e == cudaSuccess) e = cudaMalloc(&t->lo_hi, sizeof(int64_t) * (size_t)(4 * B));
  if (e == cudaSuccess) e = cudaMalloc(&t->poff, sizeof(int64_t) * (size_t)(2 * B + 1));
  af(&t->part, (slots / kPiece + 2 * B + 1) * M);
  if (e == cudaSuccess)
    e = cub::DeviceRadixSort::SortPairs(nullptr, t->sort_bytes, t->key, t->skey, t->val, t->sval, (int)slots, 0, 15);
  if (e == cudaSuccess) e = cudaMalloc(&t->sort_tmp, t->sort_bytes);
  constexpr size_t kBlasWs = 32u << 20;
  if (e == cudaSuccess) e = cudaMalloc(&t->blas_ws, kBlasWs);
  if (e != cudaSuccess) {
    train_free(t);
    return cuda_status(e, "train_create: allocation");
  }
  if (cublasCreate(&t->blas) != CUBLAS_STATUS_SUCCESS ||
      cublasSetMathMode(t->blas, CUBLAS_DEFAULT_MATH) != CUBLAS_STATUS_SUCCESS ||
      cublasSetWorkspace(t->blas, t->blas_ws, kBlasWs) != CUBLAS_STATUS_SUCCESS) {
    t->blas = nullptr;
    train_free(t);
    return fail(MSPIPE_ECUDA, "train_create: cublasCreate failed");
  }
  cudaStream_t s = (cudaStream_t)stream;
  e = cudaMemsetAsync(t->wmap, 0xff, sizeof(int32_t) * (size_t)num_nodes, s);
  if (e == cudaSuccess) {
    const int64_t n1 = std::max<int64_t>(R * F, 4 * M);
    k_tr_fill<<<grid_for(n1, 256), 256, 0, s>>>(n1, 1.f, t->ones);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {  // the updater's images follow the master weights from the start
    launch_gru_pack_tc(params + t->off[P_WIH], params + t->off[P_WHH], params + t->off[P_BIH], params + t->off[P_BHH],
                       gru->d, gru->wtc, gru->bias, s);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    train_free(t);
    return cuda_status(e, "train_create: init");
  }
  *out = t;
  return MSPIPE_OK;
}

mspipe_status mspipe_train_destroy(mspipe_train* t) {
  train_free(t);
  return MSPIPE_OK;
}

mspipe_status mspipe_gru_save_gates(mspipe_gru* gru, float* gates) {
  if (!gru) return fail(MSPIPE_EINVAL, "gru_save_gates: NULL handle");
  if (gates && (gru->precision == MSPIPE_FP32_SIMT || gru->d.cell != MSPIPE_CELL_GRU))
    return fail(MSPIPE_EUNSUPPORTED, "gru_save_gates: tensor-core GRUCell handles only");
  gru->d.gates = gates;
  return MSPIPE_OK;
}

#define TR_BLAS(call)                                                                 \
  do {                                                                                \
    if ((call) != CUBLAS_STATUS_SUCCESS) return fail(MSPIPE_ECUDA, "train_step: cuBLAS " #call); \
  } while (0)

mspipe_status mspipe_train_step(mspipe_train* t, const mspipe_gru* gru, int64_t num_events, const int32_t* sub_ids,
                                const float* sub_dt, const int32_t* sub_cnt, const float* snap_mem,
                                const int32_t* nodes, const int32_t* num_unique, const float* new_mem,
                                const void* workspace, size_t ws_bytes, const float* gates, double* out_loss,
                                float* out_logits, void* stream) {
  if (!t || !gru) return fail(MSPIPE_EINVAL, "train_step: NULL handle");
  if (num_events < 0 || num_events > t->max_events)
    return fail(MSPIPE_EINVAL, "train_step: num_events=%lld > max %lld", (long long)num_events,
                (long long)t->max_events);
  if (gru->d.M != t->d.M || gru->d.K != t->d.K || gru->d.bf16)
    return fail(MSPIPE_EINVAL, "train_step: the GRU handle does not match this training stage");
  if (!sub_ids || !sub_dt || !sub_cnt || !snap_mem || !nodes || !num_unique || !new_mem || !workspace || !gates ||
      !out_loss)
    return fail(MSPIPE_EINVAL, "train_step: null input/output");
  if (ws_bytes < mspipe_gru_workspace_size(gru, num_events))
    return fail(MSPIPE_EINVAL, "train_step: workspace of %zu bytes too small", ws_bytes);
  if (num_events == 0) return MSPIPE_OK;
  cudaStream_t s = (cudaStream_t)stream;
  // cublasSetStream resets the workspace to the default pool: re-attach ours
  if (cublasSetStream(t->blas, s) != CUBLAS_STATUS_SUCCESS ||
      cublasSetWorkspace(t->blas, t->blas_ws, 32u << 20) != CUBLAS_STATUS_SUCCESS)
    return fail(MSPIPE_ECUDA, "train_step: cublasSetStream / cublasSetWorkspace");
  const Dims& d = t->d;
  const int64_t B = num_events, R = 3 * B, F = d.F, M = d.M, H = d.H, Z = d.M + d.Dt, B2 = 2 * B;
  const int64_t slots = R * (F + 1);
  const float* P = t->params;
  float* G = t->grads;
  const float *wq = P + t->off[P_WQ], *wkv = P + t->off[P_WK], *wo = P + t->off[P_WO], *bo = P + t->off[P_BO],
              *w1 = P + t->off[P_W1], *b1 = P + t->off[P_B1], *w2 = P + t->off[P_W2], *b2 = P + t->off[P_B2];
  // w_k and w_v are adjacent ([2H, Z] as one matrix) iff H*Z is a multiple of 4 (16-byte tensor alignment)
  const bool kv_adj = t->off[P_WV] == t->off[P_WK] + H * Z;
  if (!kv_adj) return fail(MSPIPE_EUNSUPPORTED, "train_step: emb_dim * (mem_dim + time_dim) must be a multiple of 4");
  // forward ------------------------------------------------------------------
  k_tr_map<<<grid_for(B2, 256), 256, 0, s>>>(nodes, num_unique, t->wmap, 1);
  k_tr_gather<<<grid_for(R * (F + 1) * 32, kTrThreads), kTrThreads, 0, s>>>(d, R, sub_ids, sub_dt, sub_cnt, snap_mem, t->wmap,
                                                                 new_mem, gru->time_w, gru->time_b, t->sroot, t->zn, t->zn_lo,
                                                                 t->key, t->val);
  TR_BLAS(gemm_rm(t->blas, false, true, R, H, M, t->sroot, M, wq, M, 0.f, t->q, H));
  k_tr_split<<<grid_for(2 * H * Z, 256), 256, 0, s>>>(2 * H * Z, wkv, t->wkv_hi, t->wkv_lo);
  TR_BLAS(gemm3(t->blas, false, true, R * F, 2 * H, Z, t->zn, t->zn_lo, Z, t->wkv_hi, t->wkv_lo, Z, t->kv, 2 * H));
  k_tr_attn_fwd<<<grid_for(R * 32, kTrThreads), kTrThreads, 0, s>>>(d, R, sub_cnt, t->q, t->kv, t->sroot, t->alpha,
                                                                   t->zo);
  TR_BLAS(gemm_rm(t->blas, false, true, R, H, H + M, t->zo, H + M, wo, H + M, 0.f, t->emb, H));
  k_tr_dec_in<<<grid_for(B2 * 2 * H, 256), 256, 0, s>>>(B, (int32_t)H, t->emb, bo, t->za);
  TR_BLAS(gemm_rm(t->blas, false, true, B2, H, 2 * H, t->za, 2 * H, w1, 2 * H, 0.f, t->pre, H));
  k_tr_dec_out<<<grid_for(B2 * 32, kTrThreads), kTrThreads, 0, s>>>(B, (int32_t)H, t->pre, b1, w2, b2, t->y, t->logit,
                                                                   t->dlogit, t->term, t->dpre);
  k_tr_loss<<<1, 1024, 0, s>>>(B2, t->term, out_loss);
  if (out_logits) {
    cudaError_t e = cudaMemcpyAsync(out_logits, t->logit, sizeof(float) * (size_t)B2, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_status(e, "train_step: logits");
  }
  // backward ----------------------------------------------------------
  TR_BLAS(colsum(t->blas, B2, H, t->y, H, t->dlogit, G + t->off[P_W2]));       // dw_2 = y^T dlogit
  TR_BLAS(colsum(t->blas, B2, 1, t->dlogit, 1, t->ones, G + t->off[P_B2]));    // db_2 = Σ dlogit
  TR_BLAS(gemm_rm(t->blas, true, false, H, 2 * H, B2, t->dpre, H, t->za, 2 * H, 0.f, G + t->off[P_W1], 2 * H));
  TR_BLAS(colsum(t->blas, B2, H, t->dpre, H, t->ones, G + t->off[P_B1]));
  TR_BLAS(gemm_rm(t->blas, false, false, B2, 2 * H, H, t->dpre, H, w1, 2 * H, 0.f, t->dza, 2 * H));
  k_tr_dec_scatter<<<grid_for(R * H, 256), 256, 0, s>>>(B, (int32_t)H, t->dza, t->demb);
  TR_BLAS(gemm_rm(t->blas, true, false, H, H + M, R, t->demb, H, t->zo, H + M, 0.f, G + t->off[P_WO], H + M));
  TR_BLAS(colsum(t->blas, R, H, t->demb, H, t->ones, G + t->off[P_BO]));
  TR_BLAS(gemm_rm(t->blas, false, false, R, H + M, H, t->demb, H, wo, H + M, 0.f, t->dzo, H + M));
  k_tr_attn_bwd<<<grid_for(R * 32, kTrThreads), kTrThreads, 0, s>>>(d, R, sub_cnt, t->q, t->kv, t->alpha, t->dzo,
                                                                   t->dq, t->dkv, t->dkv_lo);
  TR_BLAS(gemm_rm(t->blas, true, false, H, M, R, t->dq, H, t->sroot, M, 0.f, G + t->off[P_WQ], M));
  TR_BLAS(gemm_rm(t->blas, false, false, R, M, H, t->dq, H, wq, M, 1.f, t->dzo + H, H + M));  // ds~(root) += W_q^T dq
  {  // dW_k | dW_v = dKV^T Z over the 3B·𝒩 slots: chunked 3xTF32, partials added in order
    const int64_t RF = R * F, full = RF / kChunkK, rem = RF - full * kChunkK;
    if (full > 0)
      TR_BLAS(gemm3_tn_chunked(t->blas, 2 * H, Z, RF, t->dkv, t->dkv_lo, 2 * H, t->zn, t->zn_lo, Z, t->wpart, full));
    float* tail = nullptr;
    if (rem > 0) {
      tail = t->wpart + full * 2 * H * Z;
      TR_BLAS(gemm3(t->blas, true, false, 2 * H, Z, rem, t->dkv + full * kChunkK * 2 * H,
                    t->dkv_lo + full * kChunkK * 2 * H, 2 * H, t->zn + full * kChunkK * Z, t->zn_lo + full * kChunkK * Z,
                    Z, tail, Z));
    }
    k_tr_sum_parts<<<grid_for(2 * H * Z, 256), 256, 0, s>>>(2 * H * Z, full, t->wpart, tail, G + t->off[P_WK]);
  }
  TR_BLAS(gemm3(t->blas, false, false, R * F, M, 2 * H, t->dkv, t->dkv_lo, 2 * H, t->wkv_hi, t->wkv_lo, Z, t->dzn, M));
  // T2: node gradients into the winners' h' rows, deterministic order
  size_t sb = t->sort_bytes;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(t->sort_tmp, sb, t->key, t->skey, t->val, t->sval, (int)slots, 0, 15, s);
  if (e != cudaSuccess) return cuda_status(e, "train_step: sort");
  e = cudaMemsetAsync(t->lo_hi, 0, sizeof(int64_t) * (size_t)(2 * B2), s);
  if (e != cudaSuccess) return cuda_status(e, "train_step: segment bounds");
  k_tr_seg_bounds<<<grid_for(slots + 1, 256), 256, 0, s>>>(slots, t->skey, t->lo_hi);
  k_tr_seg_plan<<<1, 1024, 0, s>>>(B2, num_unique, t->lo_hi, t->poff);
  const int64_t max_pieces = slots / kPiece + B2 + 1;
  k_tr_seg_piece<<<(unsigned)std::min<int64_t>(max_pieces, (int64_t)num_sms() * 8), kTrThreads, 0, s>>>(
      d, B2, t->lo_hi, t->poff, t->sval, t->dzo, t->dzn, t->part);
  k_tr_seg_final<<<grid_for(B2 * (M / 4), 256), 256, 0, s>>>((int32_t)M, B2, t->poff, t->part, t->dhn);
  const int32_t nchunks = gru->d.Kpad / tc::kKC;
  k_tr_gru_bwd<<<grid_for(B2 * d.K, 256), 256, 0, s>>>(d, B2, nchunks, num_unique, (const float*)workspace, gates,
                                                      t->dhn, t->D, t->xp);
  const int64_t K = d.K, Dx = d.Dx;
  TR_BLAS(gemm_rm(t->blas, true, false, 3 * M, Dx, B2, t->D, 4 * M, t->xp, K, 0.f, G + t->off[P_WIH], Dx));
  TR_BLAS(gemm_rm(t->blas, true, false, 2 * M, M, B2, t->D, 4 * M, t->xp + Dx, K, 0.f, G + t->off[P_WHH], M));
  TR_BLAS(gemm_rm(t->blas, true, false, M, M, B2, t->D + 3 * M, 4 * M, t->xp + Dx, K, 0.f,
                  G + t->off[P_WHH] + 2 * M * M, M));
  TR_BLAS(colsum(t->blas, B2, 4 * M, t->D, 4 * M, t->ones, t->cs));
  k_tr_gru_bias<<<grid_for(3 * M, 256), 256, 0, s>>>((int32_t)M, t->cs, G + t->off[P_BIH], G + t->off[P_BHH]);
  k_tr_map<<<grid_for(B2, 256), 256, 0, s>>>(nodes, num_unique, t->wmap, 0);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e, "train_step: launch");
  return MSPIPE_OK;
}

mspipe_status mspipe_train_sgd(mspipe_train* t, mspipe_gru* gru, float lr, void* stream) {
  if (!t || !gru) return fail(MSPIPE_EINVAL, "train_sgd: NULL handle");
  if (gru->d.M != t->d.M || gru->d.K != t->d.K || gru->d.bf16)
    return fail(MSPIPE_EINVAL, "train_sgd: the GRU handle does not match this training stage");
  cudaStream_t s = (cudaStream_t)stream;
  k_tr_sgd<<<grid_for(t->total, 256), 256, 0, s>>>(t->total, lr, t->grads, t->params);
  const float* P = t->params;
  launch_gru_pack_tc(P + t->off[P_WIH], P + t->off[P_WHH], P + t->off[P_BIH], P + t->off[P_BHH], gru->d, gru->wtc,
                     gru->bias, s);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e, "train_sgd: launch");
  return MSPIPE_OK;
}
