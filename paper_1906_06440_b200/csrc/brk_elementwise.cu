// brk_elementwise.cu — the small bandwidth-bound kernels around the BRGEMM passes:
//   * blocked column sum (bias gradient) with optional ReLU mask, any block factors
//   * SGD apply  w -= lr * dw  (after a data-parallel allreduce of dw)
#include <cuda_bf16.h>

#include "brk_internal.h"

namespace brk {
namespace {

// fp32 -> TF32 (10-bit mantissa) round-to-nearest, ties away (cvt.rna.tf32.f32), kept as fp32 bits
__global__ void round_tf32_kernel(const float* __restrict__ src, float* __restrict__ dst, int64_t n) {
  const int64_t nv = n / 4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nv;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 v = reinterpret_cast<const float4*>(src)[i];
    uint32_t r[4];
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r[0]) : "f"(v.x));
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r[1]) : "f"(v.y));
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r[2]) : "f"(v.z));
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r[3]) : "f"(v.w));
    reinterpret_cast<float4*>(dst)[i] = make_float4(__uint_as_float(r[0]), __uint_as_float(r[1]),
                                                    __uint_as_float(r[2]), __uint_as_float(r[3]));
  }
  if (blockIdx.x == 0 && threadIdx.x < n - nv * 4) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(src[nv * 4 + threadIdx.x]));
    dst[nv * 4 + threadIdx.x] = __uint_as_float(r);
  }
}

__device__ __forceinline__ float ld_any(const void* p, int64_t i, int bf16) {
  return bf16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]) : static_cast<const float*>(p)[i];
}
__device__ __forceinline__ void st_any(void* p, int64_t i, float v, int bf16) {
  if (bf16) static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
  else static_cast<float*>(p)[i] = v;
}

// Column sums in two deterministic passes: pass 1, CTA (column tile, row split)
// sums its rows per column (threads = consecutive columns: coalesced rows of
// the blocked layout); pass 2 adds the split partials in split order.
__device__ __forceinline__ int64_t blk_off(int n, int k, int Kb, int b_n, int b_k) {
  return (static_cast<int64_t>(n / b_n) * Kb + k / b_k) * b_n * b_k + static_cast<int64_t>(n % b_n) * b_k + k % b_k;
}

__global__ void colsum_partial_kernel(const void* dy, const void* y, void* dz_out, float* part, int N, int K,
                                      int b_n, int b_k, int bf16, int rows_per) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const int Kb = K / b_k;
  const int n0 = blockIdx.y * rows_per, n1 = min(N, n0 + rows_per);
  float s = 0.0f;
  for (int n = n0; n < n1; ++n) {
    const int64_t off = blk_off(n, k, Kb, b_n, b_k);
    float g = ld_any(dy, off, bf16);
    if (y != nullptr) {
      if (!(ld_any(y, off, bf16) > 0.0f)) g = 0.0f;
      if (dz_out != nullptr) st_any(dz_out, off, g, bf16);
    }
    s += g;
  }
  part[static_cast<int64_t>(blockIdx.y) * K + k] = s;
}

__global__ void colsum_final_kernel(const float* part, int splits, int K, float* db) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  float s = 0.0f;
  for (int i = 0; i < splits; ++i) s += part[static_cast<int64_t>(i) * K + k];
  db[k] = s;
}

__global__ void sgd_apply_kernel(void* w, const float* __restrict__ dw, float lr, int64_t n, int bf16) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    st_any(w, i, ld_any(w, i, bf16) - lr * dw[i], bf16);
  }
}

}  // namespace
}  // namespace brk

using namespace brk;

extern "C" {

BRK_API int brk_colsum_blocked(const void* dy, const void* y, void* dz_out, float* db, int N, int K,
                               int b_n, int b_k, int dtype, void* stream) {
  if (N <= 0 || K <= 0 || b_n <= 0 || b_k <= 0 || N % b_n || K % b_k)
    return set_error(BRK_ERR_CONTRACT, "colsum: block factors must divide N and K");
  if (dtype != BRK_F32 && dtype != BRK_BF16) return set_error(BRK_ERR_CONTRACT, "colsum: bad dtype");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int tiles = (K + 255) / 256;
  int splits = (148 * 8) / tiles;
  splits = splits < 1 ? 1 : (splits > N ? N : splits);
  const int rows_per = (N + splits - 1) / splits;
  splits = (N + rows_per - 1) / rows_per;
  float* part = nullptr;  // stream-ordered scratch
  cudaError_t err = cudaMallocAsync(reinterpret_cast<void**>(&part), static_cast<size_t>(splits) * K * sizeof(float), st);
  if (err != cudaSuccess) return set_cuda_error(err, "colsum scratch");
  g_launches.fetch_add(2);
  colsum_partial_kernel<<<dim3(tiles, splits), 256, 0, st>>>(dy, y, dz_out, part, N, K, b_n, b_k, dtype == BRK_BF16,
                                                             rows_per);
  colsum_final_kernel<<<tiles, 256, 0, st>>>(part, splits, K, db);
  err = cudaGetLastError();
  cudaError_t err2 = cudaFreeAsync(part, st);
  if (err != cudaSuccess) return set_cuda_error(err, "colsum launch");
  return err2 == cudaSuccess ? BRK_OK : set_cuda_error(err2, "colsum scratch free");
}

BRK_API int brk_round_tf32(const float* src, float* dst, int64_t n, void* stream) {
  if (n < 0) return set_error(BRK_ERR_CONTRACT, "round_tf32: n must be >= 0");
  if (n == 0) return BRK_OK;
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15)
    return set_error(BRK_ERR_CONTRACT, "round_tf32: 16-byte aligned buffers");
  g_launches.fetch_add(1);
  const int64_t vec = (n + 3) / 4;
  const int blocks = static_cast<int>(vec / 256 + 1 < 148 * 8 ? vec / 256 + 1 : 148 * 8);
  round_tf32_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(src, dst, n);
  cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? BRK_OK : set_cuda_error(err, "round_tf32 launch");
}

BRK_API int brk_sgd_apply(void* w, const float* dw, float lr, int64_t n, int w_dtype, void* stream) {
  if (n < 0) return set_error(BRK_ERR_CONTRACT, "sgd: n must be >= 0");
  if (w_dtype != BRK_F32 && w_dtype != BRK_BF16) return set_error(BRK_ERR_CONTRACT, "sgd: bad dtype");
  if (n == 0) return BRK_OK;
  g_launches.fetch_add(1);
  const int blocks = static_cast<int>((n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8);
  sgd_apply_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(w, dw, lr, n, w_dtype == BRK_BF16);
  cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? BRK_OK : set_cuda_error(err, "sgd launch");
}

}  // extern "C"
