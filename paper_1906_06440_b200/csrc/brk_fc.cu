// brk_fc.cu — fully-connected layer passes on the blocked layouts of the
// reference (fc.py:99-163, tensor.py:143-158/237-247), each ONE launch of the
// tcgen05 BRGEMM engine whose batch list runs over the reduction blocks:
//
//   fwd : Y [Nb][Kb][bn][bk]  = act(W X + b)        batch over C_b  (Alg. 5)
//   bwd : dX[Nb][Cb][bn][bc]  = (W^T dZ) * mask     batch over K_b
//   upd : dW[Kb][Cb][bc][bk]  = dZ X^T  (+ SGD)     batch over N_b
//   bias: db[K] = sum_n dZ,  dZ = dY * (Y > 0)      (deterministic column sum)
//
// TMA engine path: bf16 storage with all block factors = 64 (one 128 B
// swizzle row per block row).  Tensor-map coordinates per k-step are the
// blocked-tensor coordinates of the batch entry.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <cuda_bf16.h>

#include "brk_engine.h"
#include "brk_internal.h"
#include "brk_tma_host.h"

namespace brk {

int launch_engine(const EngineParams& p, int bn, int tf32, int max_ctas, cudaStream_t stream);
int engine_sm_count();


namespace {

constexpr int kB = 64;  // block factor served by the TMA path (bf16)

int pick_bn(int m_tiles, int n_extent) {
  if (const char* env = std::getenv("BRK_BN")) {
    int v = std::atoi(env);
    if ((v == 64 || v == 128 || v == 256) && n_extent % v == 0) return v;
  }
  const int sms = engine_sm_count();
  int best = 0;
  long best_cost = 0;
  for (int bn : {256, 128, 64}) {
    if (n_extent % bn) continue;
    const long tiles = static_cast<long>(m_tiles) * (n_extent / bn);
    const long waves = (tiles + sms - 1) / sms;
    const long cost = waves * (bn + 64);
    if (best == 0 || cost < best_cost) { best = bn; best_cost = cost; }
  }
  return best;
}

// Blocked 2-D activation [Rb][Xb][64][64] (row-major blocks, x innermost):
// X (rows n, x = c), dZ/Y (rows n, x = k).
struct Act4 {
  uint64_t dims[4];
  uint64_t strides[4];
};
Act4 act_layout(int64_t rows, int64_t xs) {
  Act4 a;
  a.dims[0] = kB; a.dims[1] = kB; a.dims[2] = xs / kB; a.dims[3] = rows / kB;
  a.strides[0] = 1; a.strides[1] = kB; a.strides[2] = kB * kB; a.strides[3] = (xs / kB) * kB * kB;
  return a;
}
// Weights [Kb][Cb][64 c][64 k] (k innermost): dims (k_in, c_in, cb, kb)
Act4 w_layout(int64_t K, int64_t C) {
  Act4 a;
  a.dims[0] = kB; a.dims[1] = kB; a.dims[2] = C / kB; a.dims[3] = K / kB;
  a.strides[0] = 1; a.strides[1] = kB; a.strides[2] = kB * kB; a.strides[3] = (C / kB) * kB * kB;
  return a;
}

void set_coords(OperandCoords& oc, std::initializer_list<int> rc, std::initializer_list<int> kq,
                int n_loads, uint32_t load_bytes, int mn_major) {
  std::memset(&oc, 0, sizeof(oc));
  int d = 0;
  for (int v : rc) oc.rc[d++] = v;
  d = 0;
  for (int v : kq) oc.kq[d++] = v;
  oc.kdiv = 1;
  oc.n_loads = n_loads;
  oc.load_bytes = load_bytes;
  oc.mn_major = mn_major;
  oc.ndims = 4;
}

int check_fc(int N, int C, int K, int b_n, int b_c, int b_k, int dtype) {
  char buf[256];
  if (dtype != BRK_BF16)
    return set_error(BRK_ERR_CONTRACT, "fc engine path: bf16 storage only (use the generic BRGEMM path)");
  if (b_n != kB || b_c != kB || b_k != kB) {
    std::snprintf(buf, sizeof(buf), "fc engine path needs b_n=b_c=b_k=64, got (%d,%d,%d)", b_n, b_c, b_k);
    return set_error(BRK_ERR_CONTRACT, buf);
  }
  if (N <= 0 || C <= 0 || K <= 0 || N % 128 || C % 128 || K % 128) {
    std::snprintf(buf, sizeof(buf), "fc engine path needs N, C, K multiples of 128 (N=%d C=%d K=%d)", N, C, K);
    return set_error(BRK_ERR_CONTRACT, buf);
  }
  return BRK_OK;
}

int enc(CUtensorMap* map, const void* ptr, const Act4& l, uint32_t b0, uint32_t b1, uint32_t b2,
        uint32_t b3) {
  const uint32_t box[4] = {b0, b1, b2, b3};
  return encode_tmap(map, ptr, true, 4, l.dims, l.strides, box);
}

// ---------------------------------------------------------------------------
// dZ = dY * (Y > 0) (optional) and db[k] = sum_n dZ[n][k]  — deterministic:
// grid (K/64, kSplit); CTA (kb, s) sums rows of split s for 64 columns, then
// the last CTA of column block kb adds the kSplit partials in a fixed order.
// ---------------------------------------------------------------------------
constexpr int kSplit = 16;

__global__ void __launch_bounds__(256) bias_grad_kernel(const __nv_bfloat16* dy,
                                                        const __nv_bfloat16* __restrict__ y,
                                                        __nv_bfloat16* dz_out,
                                                        float* __restrict__ db, float* __restrict__ partial,
                                                        unsigned* __restrict__ counters, int N, int K,
                                                        float* __restrict__ bias, float lr) {
  const int kb = blockIdx.x, split = blockIdx.y;
  const int Kb = K / kB;
  const int tid = threadIdx.x;
  const int cgrp = tid & 7;   // 8 column groups of 8 (16 B)
  const int rlane = tid >> 3;  // 32 row lanes
  const int rows_per = N / kSplit;
  const int r0 = split * rows_per;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int r = r0 + rlane; r < r0 + rows_per; r += 32) {
    const int64_t off = static_cast<int64_t>(r / kB) * Kb * kB * kB + static_cast<int64_t>(kb) * kB * kB +
                        (r % kB) * kB + cgrp * 8;
    uint4 g = *reinterpret_cast<const uint4*>(dy + off);
    __nv_bfloat16* gh = reinterpret_cast<__nv_bfloat16*>(&g);
    if (y != nullptr) {
      uint4 m = *reinterpret_cast<const uint4*>(y + off);
      const __nv_bfloat16* mh = reinterpret_cast<const __nv_bfloat16*>(&m);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (!(__bfloat162float(mh[j]) > 0.0f)) gh[j] = __float2bfloat16_rn(0.0f);
      if (dz_out != nullptr) *reinterpret_cast<uint4*>(dz_out + off) = g;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += __bfloat162float(gh[j]);
  }
  __shared__ float red[32][65];
#pragma unroll
  for (int j = 0; j < 8; ++j) red[rlane][cgrp * 8 + j] = acc[j];
  __syncthreads();
  __shared__ bool is_last;
  if (tid < 64) {
    float s = 0.0f;
    for (int l = 0; l < 32; ++l) s += red[l][tid];
    partial[(static_cast<int64_t>(split) * Kb + kb) * kB + tid] = s;
    __threadfence();
  }
  __syncthreads();
  if (tid == 0) {
    const unsigned prev = atomicAdd(&counters[kb], 1u);
    is_last = (prev == kSplit - 1);
  }
  __syncthreads();
  if (is_last && tid < 64) {
    __threadfence();
    float s = 0.0f;
    for (int sp = 0; sp < kSplit; ++sp) s += __ldcg(&partial[(static_cast<int64_t>(sp) * Kb + kb) * kB + tid]);
    db[kb * kB + tid] = s;
    if (bias != nullptr) bias[kb * kB + tid] -= lr * s;
    if (tid == 0) counters[kb] = 0;  // self-reset for the next launch / graph replay
  }
}

}  // namespace
}  // namespace brk

using namespace brk;

extern "C" {

BRK_API int brk_fc_fwd(const void* x, const void* w, const float* bias, void* y, int N, int C, int K,
                       int b_n, int b_c, int b_k, int act, int dtype, void* stream) {
  int rc = check_fc(N, C, K, b_n, b_c, b_k, dtype);
  if (rc) return rc;
  if (act < kActNone || act > kActSigmoid) return set_error(BRK_ERR_CONTRACT, "unknown activation");
  EngineParams p;
  std::memset(&p, 0, sizeof(p));
  const int m_tiles = N / 128;
  const int bn = pick_bn(m_tiles, K);
  // A = X (rows n, red c) K-major: box (c 64, n 64, cb 1, nb 2)
  if ((rc = enc(&p.map_a, x, act_layout(N, C), 64, 64, 1, 2))) return rc;
  set_coords(p.ca, {0, 0, 0, 2}, {0, 0, 1, 0}, 1, 128 * 128, 0);
  // B = W (rows k, red c) MN-major: box (k 64, c 64, cb 1, kb bn/64)
  if ((rc = enc(&p.map_b, w, w_layout(K, C), 64, 64, 1, bn / 64))) return rc;
  set_coords(p.cb, {0, 0, 0, bn / 64}, {0, 0, 1, 0}, 1, bn * 128, 1);
  p.m_tiles = m_tiles;
  p.n_tiles = K / bn;
  p.k_steps = C / kB;
  p.rows = N;
  p.cols = K;
  p.out = y;
  p.out_bf16 = 1;
  p.om = OutMap{kB, (int64_t)(K / kB) * kB * kB, kB, kB, kB * kB, 1};
  p.alpha = 1.0f;
  p.bias = bias;
  p.act = act;
  if (const char* dbg = std::getenv("BRK_DEBUG_FLAGS")) p.debug_flags = std::atoi(dbg);
  g_launches.fetch_add(1);
  return launch_engine(p, bn, 0, 0, static_cast<cudaStream_t>(stream));
}

BRK_API int brk_fc_bwd_data(const void* dz, const void* w, const void* mask, void* dx, int N, int C,
                            int K, int b_n, int b_c, int b_k, int dtype, void* stream) {
  int rc = check_fc(N, C, K, b_n, b_c, b_k, dtype);
  if (rc) return rc;
  EngineParams p;
  std::memset(&p, 0, sizeof(p));
  const int m_tiles = N / 128;
  const int bn = pick_bn(m_tiles, C);
  // A = dZ (rows n, red k) K-major
  if ((rc = enc(&p.map_a, dz, act_layout(N, K), 64, 64, 1, 2))) return rc;
  set_coords(p.ca, {0, 0, 0, 2}, {0, 0, 1, 0}, 1, 128 * 128, 0);
  // B = W (rows c, red k) K-major: dims (k_in, c_in, cb, kb), box (64, 64, bn/64, 1)
  if ((rc = enc(&p.map_b, w, w_layout(K, C), 64, 64, bn / 64, 1))) return rc;
  set_coords(p.cb, {0, 0, bn / 64, 0}, {0, 0, 0, 1}, 1, bn * 128, 0);
  p.m_tiles = m_tiles;
  p.n_tiles = C / bn;
  p.k_steps = K / kB;
  p.rows = N;
  p.cols = C;
  p.out = dx;
  p.out_bf16 = 1;
  p.om = OutMap{kB, (int64_t)(C / kB) * kB * kB, kB, kB, kB * kB, 1};
  p.alpha = 1.0f;
  p.mask = mask;
  g_launches.fetch_add(1);
  return launch_engine(p, bn, 0, 0, static_cast<cudaStream_t>(stream));
}

BRK_API int brk_fc_upd(const void* x, const void* dz, float* dw, void* w_sgd, float lr, int N, int C,
                       int K, int b_n, int b_c, int b_k, int dtype, void* stream) {
  int rc = check_fc(N, C, K, b_n, b_c, b_k, dtype);
  if (rc) return rc;
  EngineParams p;
  std::memset(&p, 0, sizeof(p));
  const int m_tiles = C / 128;
  const int bn = pick_bn(m_tiles, K);
  // A = X^T (rows c, red n) MN-major: box (c 64, n 64, cb 2, nb 1) -> 2 atoms
  if ((rc = enc(&p.map_a, x, act_layout(N, C), 64, 64, 2, 1))) return rc;
  set_coords(p.ca, {0, 0, 2, 0}, {0, 0, 0, 1}, 1, 128 * 128, 1);
  // B = dZ^T (rows k, red n) MN-major: box (k 64, n 64, kb bn/64, nb 1)
  if ((rc = enc(&p.map_b, dz, act_layout(N, K), 64, 64, bn / 64, 1))) return rc;
  set_coords(p.cb, {0, 0, bn / 64, 0}, {0, 0, 0, 1}, 1, bn * 128, 1);
  p.m_tiles = m_tiles;
  p.n_tiles = K / bn;
  p.k_steps = N / kB;
  p.rows = C;
  p.cols = K;
  p.out = dw;
  p.out_bf16 = 0;
  // dW [Kb][Cb][64 c][64 k]: row c -> (c/64)*4096 + (c%64)*64 ; col k -> (k/64)*Cb*4096 + k%64
  p.om = OutMap{kB, kB * kB, kB, kB, (int64_t)(C / kB) * kB * kB, 1};
  p.alpha = 1.0f;
  p.sgd_w = w_sgd;
  p.sgd_lr = lr;
  g_launches.fetch_add(1);
  return launch_engine(p, bn, 0, 0, static_cast<cudaStream_t>(stream));
}

// dz_out = dy * (y > 0) when y != NULL (dz_out may alias dy), db = column sums.
// workspace: >= kSplit*K floats + K/64 unsigned counters (zero-initialised once).
BRK_API int brk_fc_bias_grad(const void* dy, const void* y, void* dz_out, float* db, void* workspace,
                             int N, int K, int b_n, int b_k, float* bias_sgd, float lr, void* stream) {
  if (b_n != kB || b_k != kB || N % (kSplit * 1) || N % kB || K % kB)
    return set_error(BRK_ERR_CONTRACT, "bias_grad needs b_n=b_k=64 and N, K multiples of 64");
  if (N % kSplit) return set_error(BRK_ERR_CONTRACT, "bias_grad needs N % 16 == 0");
  float* partial = static_cast<float*>(workspace);
  unsigned* counters = reinterpret_cast<unsigned*>(partial + static_cast<size_t>(kSplit) * K);
  dim3 grid(K / kB, kSplit);
  g_launches.fetch_add(1);
  bias_grad_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(y),
      static_cast<__nv_bfloat16*>(dz_out), db, partial, counters, N, K, bias_sgd, lr);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error(err, "bias_grad launch");
  return BRK_OK;
}

BRK_API size_t brk_fc_bias_grad_workspace(int K) {
  return static_cast<size_t>(kSplit) * K * sizeof(float) + static_cast<size_t>(K / kB + 1) * sizeof(unsigned);
}

}  // extern "C"
