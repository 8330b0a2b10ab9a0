// tc_layout.cuh — the GEMM A-operand image layout shared by its producers
// (k_build_x in gru_tc.cu, the fused build in prep.cu) and its consumer
// (k_gru_tc): per (128-row tile, 32-wide K chunk) one SWIZZLE_128B K-major
// block, tf32 hi image then lo image (3xTF32 split, a = hi + lo).
#pragma once
#include <stdint.h>

namespace mspipe {
namespace tc {

constexpr int kM = 128;                 // rows per tile (UMMA M)
constexpr int kKC = 32;                 // fp32 per 128 B swizzle row = one K chunk
constexpr int kATile = kM * kKC * 4;    // 16 KB
constexpr int kABlock = 2 * kATile;     // hi | lo

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// byte offset of element (row, k) inside a 128-row x 32-fp32 SWIZZLE_128B tile
__host__ __device__ __forceinline__ uint32_t sw128_off(uint32_t row, uint32_t k) {
  return row * 128u + ((((k >> 2) ^ (row & 7u)) & 7u) << 4) + (k & 3u) * 4u;
}

// A operand of GEMM row u, column k = value v, split hi | lo
__device__ __forceinline__ void store_a(float* xbuf, int32_t nchunks, int32_t u, int32_t k, float v) {
  const float hi = tf32_rna(v);
  const float lo = tf32_rna(v - hi);
  char* blk = reinterpret_cast<char*>(xbuf) + ((int64_t)(u / kM) * nchunks + k / kKC) * kABlock;
  const uint32_t off = sw128_off((uint32_t)(u % kM), (uint32_t)(k % kKC));
  *reinterpret_cast<float*>(blk + off) = hi;
  *reinterpret_cast<float*>(blk + kATile + off) = lo;
}

// bf16 operands (MSPIPE_BF16): one 128 B swizzle row holds 64 bf16 = one K chunk
constexpr int kKC16 = 64;
constexpr int kATile16 = kM * kKC16 * 2;  // 16 KB

__host__ __device__ __forceinline__ uint32_t sw128_off16(uint32_t row, uint32_t k) {
  return row * 128u + ((((k >> 3) ^ (row & 7u)) & 7u) << 4) + (k & 7u) * 2u;
}

}  // namespace tc
}  // namespace mspipe
