// gru_simt.cu — A5 + A6 on CUDA cores in fp32 (MSPIPE_FP32_SIMT): the
// correctness baseline of the memory updater.
//
// One GEMM  [U x K] . [K x 4M]  with K = Dx + M rows of packed weights
// [[W_ir W_iz W_in 0], [W_hr W_hz 0 W_hn]] so each output column group
// (r_pre, z_pre, n_x, n_h) of hidden unit j is produced by the same thread
// and the GRU gates are applied in registers (no pre-activation round trip).
// The A operand x = [s_w ‖ s_o ‖ e ‖ cos(ω Δt + φ) ‖ h] is never
// materialised: each K-chunk of it is built straight into shared memory
// from the snapshot rows, the edge-feature rows and the time encoder.
#include "internal.cuh"

namespace mspipe {

constexpr int kMT = 32;        // winner rows per CTA
constexpr int kJT = 32;        // hidden units per CTA
constexpr int kNT = 4 * kJT;   // packed columns per CTA
constexpr int kKC = 32;        // K chunk
constexpr int kThreads = 128;  // 4 warps: warp w owns rows 8w..8w+7, lane owns hidden unit

// ---------------------------------------------------------------------------
// weight packing: wpack[k][jt*128 + g*32 + jj], j = jt*32 + jj, g in (r, z, n_x, n_h)
// ---------------------------------------------------------------------------
__global__ void k_gru_pack(const float* __restrict__ w_ih, const float* __restrict__ w_hh,
                           const float* __restrict__ b_ih, const float* __restrict__ b_hh,
                           GruDesc d, float* __restrict__ wpack, float* __restrict__ bias) {
  const int64_t total = (int64_t)d.Kpad * d.Npad;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t k = (int32_t)(t / d.Npad), n = (int32_t)(t % d.Npad);
    const int32_t jt = n / kNT, g = (n % kNT) / kJT, jj = n % kJT, j = jt * kJT + jj;
    const int32_t M = d.M;
    float v = 0.f;
    if (j < M) {
      if (k < d.Dx) {
        if (g < 3) v = w_ih[(int64_t)(g * M + j) * d.Dx + k];
      } else if (k < d.K) {
        const int32_t kk = k - d.Dx;
        if (g == 0) v = w_hh[(int64_t)j * M + kk];
        else if (g == 1) v = w_hh[(int64_t)(M + j) * M + kk];
        else if (g == 3) v = w_hh[(int64_t)(2 * M + j) * M + kk];
      }
    }
    wpack[t] = v;
    if (k == 0) {
      float b = 0.f;
      if (j < M) {
        if (g == 0) b = b_ih[j] + b_hh[j];
        else if (g == 1) b = b_ih[M + j] + b_hh[M + j];
        else if (g == 2) b = b_ih[2 * M + j];
        else b = b_hh[2 * M + j];
      }
      bias[n] = b;
    }
  }
}

void launch_gru_pack(const float* w_ih, const float* w_hh, const float* b_ih, const float* b_hh,
                     const GruDesc& d, float* wpack, float* bias, cudaStream_t s) {
  const int threads = 256;
  int64_t blocks = ((int64_t)d.Kpad * d.Npad + threads - 1) / threads;
  if (blocks > 4096) blocks = 4096;
  k_gru_pack<<<(unsigned)blocks, threads, 0, s>>>(w_ih, w_hh, b_ih, b_hh, d, wpack, bias);
}

// ---------------------------------------------------------------------------
struct RowInfo {
  int32_t rw[kMT];  // snapshot row of the winner node (root layout)
  int32_t ro[kMT];  // snapshot row of the other endpoint
  int32_t ev[kMT];  // event index a inside the batch
  float dt[kMT];    // Δt = (float)(t* - S.mem_ts[w])
};

struct GruArgs {
  GruDesc d;
  const double* ts;
  int64_t B;
  const float* ef;
  const float* snap_mem;
  const double* snap_ts;
  int64_t step;
  const float* snap_h;
};

__device__ __forceinline__ float x_elem(const GruArgs& a, const RowInfo& ri, int m, int k) {
  const int32_t rw = ri.rw[m];
  if (rw < 0) return 0.f;
  const GruDesc& d = a.d;
  const int32_t M = d.M;
  if (k < M) return __ldg(a.snap_mem + (int64_t)rw * a.step * M + k);
  if (k < 2 * M) return __ldg(a.snap_mem + (int64_t)ri.ro[m] * a.step * M + (k - M));
  if (k < d.Dm) return __ldg(a.ef + (int64_t)ri.ev[m] * d.He + (k - 2 * M));
  if (k < d.Dx) {
    const int q = k - d.Dm;
    return time_cos(fmaf(__ldg(d.time_w + q), ri.dt[m], __ldg(d.time_b + q)));
  }
  if (k < d.K) {
    const int kk = k - d.Dx;
    return a.snap_h ? __ldg(a.snap_h + (int64_t)rw * M + kk)
                    : __ldg(a.snap_mem + (int64_t)rw * a.step * M + kk);
  }
  return 0.f;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

__global__ void __launch_bounds__(kThreads) k_gru_simt(
    GruArgs a, const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
    const int32_t* __restrict__ winner, const int32_t* __restrict__ num_unique,
    float* __restrict__ out_mem, double* __restrict__ out_ts, float* __restrict__ out_mail,
    int64_t mail_stride) {
  __shared__ __align__(16) float As[2][kMT][kKC + 4];
  __shared__ __align__(16) float Bs[2][kKC][kNT];
  __shared__ RowInfo ri;
  const int32_t U = __ldg(num_unique);
  const int32_t m0 = blockIdx.x * kMT;
  if (m0 >= U) return;
  const int jt = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, ty = tid >> 5;
  const GruDesc& d = a.d;
  const int32_t M = d.M;
  if (tid < kMT) {
    const int32_t u = m0 + tid;
    if (u < U) {
      const int32_t p = __ldg(winner + u);
      const int32_t ev = p >> 1, role = p & 1;
      const int32_t rw = role ? (int32_t)a.B + ev : ev;
      const int32_t ro = role ? ev : (int32_t)a.B + ev;
      ri.rw[tid] = rw;
      ri.ro[tid] = ro;
      ri.ev[tid] = ev;
      ri.dt[tid] = (float)(__ldg(a.ts + ev) - __ldg(a.snap_ts + (int64_t)rw * a.step));
    } else {
      ri.rw[tid] = -1;
      ri.ro[tid] = -1;
      ri.ev[tid] = 0;
      ri.dt[tid] = 0.f;
    }
  }
  __syncthreads();

  const float* wcol = d.wpack + (int64_t)jt * kNT;
  auto issue_B = [&](int stage, int kc) {
    // 32 x 128 floats = 1024 x 16 B; 8 per thread
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int idx = tid + i * kThreads;
      const int r = idx >> 5, c4 = idx & 31;
      cp_async16(&Bs[stage][r][c4 * 4], wcol + (int64_t)(kc * kKC + r) * d.Npad + c4 * 4);
    }
    cp_async_commit();
  };
  float areg[8];
  auto fetch_A = [&](int kc) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int idx = tid + i * kThreads;
      areg[i] = x_elem(a, ri, idx >> 5, kc * kKC + (idx & 31));
    }
  };
  auto store_A = [&](int stage) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int idx = tid + i * kThreads;
      As[stage][idx >> 5][idx & 31] = areg[i];
    }
  };

  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int g = 0; g < 4; ++g) acc[i][g] = 0.f;

  const int nK = d.Kpad / kKC;
  issue_B(0, 0);
  fetch_A(0);
  store_A(0);
  for (int kc = 0; kc < nK; ++kc) {
    const int s = kc & 1;
    if (kc + 1 < nK) issue_B(s ^ 1, kc + 1);
    else cp_async_commit();
    cp_async_wait1();
    __syncthreads();
    if (kc + 1 < nK) fetch_A(kc + 1);
#pragma unroll
    for (int kk = 0; kk < kKC; kk += 4) {
      float4 av[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) av[i] = *reinterpret_cast<const float4*>(&As[s][ty * 8 + i][kk]);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float bv[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) bv[g] = Bs[s][kk + q][g * kJT + lane];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float x = q == 0 ? av[i].x : (q == 1 ? av[i].y : (q == 2 ? av[i].z : av[i].w));
#pragma unroll
          for (int g = 0; g < 4; ++g) acc[i][g] = fmaf(x, bv[g], acc[i][g]);
        }
      }
    }
    if (kc + 1 < nK) store_A(s ^ 1);
    __syncthreads();
  }

  // epilogue: GRUCell gates (G5), h' = (1 - z) n + z h
  const int32_t j = jt * kJT + lane;
  if (j < M) {
    const float br = __ldg(d.bias + jt * kNT + lane);
    const float bz = __ldg(d.bias + jt * kNT + kJT + lane);
    const float bnx = __ldg(d.bias + jt * kNT + 2 * kJT + lane);
    const float bnh = __ldg(d.bias + jt * kNT + 3 * kJT + lane);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = ty * 8 + i;
      const int32_t u = m0 + m;
      if (u < U) {
        const float r = 1.0f / (1.0f + expf(-(acc[i][0] + br)));
        const float z = 1.0f / (1.0f + expf(-(acc[i][1] + bz)));
        const float n = tanhf(acc[i][2] + bnx + r * (acc[i][3] + bnh));
        const float h = x_elem(a, ri, m, d.Dx + j);
        out_mem[(int64_t)u * M + j] = (1.0f - z) * n + z * h;
      }
    }
  }
  // mail row = x[0:Dm] (G14) and the commit timestamp t*, written once (jt == 0)
  if (jt == 0) {
    const int rows = min(kMT, U - m0);
    for (int idx = tid; idx < rows * (int)mail_stride; idx += kThreads) {
      const int m = idx / (int)mail_stride, c = idx - m * (int)mail_stride;
      out_mail[(int64_t)(m0 + m) * mail_stride + c] = c < d.Dm ? x_elem(a, ri, m, c) : 0.f;
    }
    if (tid < rows) out_ts[m0 + tid] = __ldg(a.ts + ri.ev[tid]);
  }
}

void launch_gru_simt(const GruDesc& d, const int32_t* src, const int32_t* dst, const double* ts,
                     int64_t num_events, const float* edge_feat, const float* snap_mem,
                     const double* snap_mem_ts, int64_t snap_step, const float* snap_h,
                     const int32_t* nodes, const int32_t* winner, const int32_t* num_unique,
                     float* out_mem, double* out_ts, float* out_mail, int64_t mail_stride,
                     cudaStream_t s) {
  (void)nodes;
  GruArgs a{d, ts, num_events, edge_feat, snap_mem, snap_mem_ts, snap_step, snap_h};
  const int64_t max_rows = 2 * num_events;
  dim3 grid((unsigned)((max_rows + kMT - 1) / kMT), (unsigned)(d.Npad / kNT));
  launch_k(k_gru_simt, grid, dim3(kThreads), 0, s, 1, a, src, dst, winner, num_unique, out_mem, out_ts, out_mail,
           mail_stride);
}

}  // namespace mspipe
