// brk_elementwise.cu — the small bandwidth-bound kernels around the BRGEMM passes:
//   * blocked column sum (bias gradient) with optional ReLU mask, any block factors
//   * SGD apply  w -= lr * dw  (after a data-parallel allreduce of dw)
#include <cuda_bf16.h>

#include "brk_internal.h"

namespace brk {
namespace {

__device__ __forceinline__ float ld_any(const void* p, int64_t i, int bf16) {
  return bf16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]) : static_cast<const float*>(p)[i];
}
__device__ __forceinline__ void st_any(void* p, int64_t i, float v, int bf16) {
  if (bf16) static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
  else static_cast<float*>(p)[i] = v;
}

// One thread per column k; rows summed in ascending n (deterministic).
__global__ void colsum_blocked_kernel(const void* dy, const void* y, void* dz_out, float* db, int N, int K,
                                      int b_n, int b_k, int bf16) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const int Kb = K / b_k;
  const int kb = k / b_k, ki = k % b_k;
  float s = 0.0f;
  for (int n = 0; n < N; ++n) {
    const int64_t off = (static_cast<int64_t>(n / b_n) * Kb + kb) * b_n * b_k + static_cast<int64_t>(n % b_n) * b_k + ki;
    float g = ld_any(dy, off, bf16);
    if (y != nullptr) {
      if (!(ld_any(y, off, bf16) > 0.0f)) g = 0.0f;
      if (dz_out != nullptr) st_any(dz_out, off, g, bf16);
    }
    s += g;
  }
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
  g_launches.fetch_add(1);
  colsum_blocked_kernel<<<(K + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      dy, y, dz_out, db, N, K, b_n, b_k, dtype == BRK_BF16);
  cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? BRK_OK : set_cuda_error(err, "colsum launch");
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
