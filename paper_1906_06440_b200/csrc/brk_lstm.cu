// brk_lstm.cu — fused LSTM recurrent steps on tcgen05 (reference lstm.py:217-327,
// paper Alg. 2 / Eqs. 1-6; backward is the north-star BPTT restated in oracle/).
//
// Forward step t (one launch): every CTA owns 128 minibatch rows x 64 hidden
// units and computes the recurrent batch-reduce for ALL FOUR gates at once:
//     acc[g][n][k] = sum_j h_{t-1}[n][j] R_g[k][j]         (tcgen05, TMEM)
// with the four gate accumulators side by side in TMEM columns g*64 + k, so
// one epilogue thread holds i, c, f, o of its element and fuses
//     pre_g = acc_g + gx_t[n][g][k]          (gx = W x + b, precomputed)
//     s_t = sig(f) s_{t-1} + sig(i) tanh(c) ;  h_t = sig(o) tanh(s_t)
// Backward step t: acc[n][k] = sum_{g,j} dpre_{t+1}[n][g][j] R_g[j][k] (the
// recurrent gradient) + the fused gate derivatives producing dpre_t and ds.
//
// Operands are gathered by all threads with plain loads from fp32 storage and
// converted to TF32 / BF16 (R is read in the reference's blocked layout
// [K_b][K_b][b_k][b_k] with arbitrary b_k); accumulation is fp32 in TMEM.
#include <cuda_bf16.h>

#include "brk_internal.h"
#include "brk_ptx.cuh"

namespace brk {
namespace {

constexpr int kRows = 128;
constexpr int kHid = 64;  // hidden units per CTA
constexpr int kThreads = 128;
constexpr int kStages = 2;
constexpr int kChunkBytes = 128;

enum LstmMode : int { kFwd = 0, kBwd = 1, kBwdRaw = 2 };

struct LstmStepParams {
  int mode;
  int N, K, bk;
  // forward
  const float* h_prev;  // [N][K]
  const float* s_prev;  // [N][K]
  const float* gx;      // [N][4][K]  (W x_t + b)
  float* h_out;         // [N][K]
  float* s_out;         // [N][K]
  float* gates_out;     // [N][4][K] (activated i, c, f, o) — always written (BPTT needs them)
  // backward
  const float* dpre_next;  // [N][4][K] or null (t = T-1)
  const float* dh_in;      // [N][K] gradient w.r.t. h_t from the output
  const float* gates;      // [N][4][K] of step t
  const float* s_cur;      // [N][K] s_t
  const float* ds_in;      // [N][K] ds from step t+1 (null = 0)
  float* dpre_out;         // [N][4][K]
  float* ds_out;           // [N][K]
  float* raw_out;          // kBwdRaw: [N][K] = recurrent gradient only
  const float* R;          // [4][K_b][K_b][bk][bk] blocked, fp32
};

__device__ __forceinline__ uint32_t canon_off(int row, int chunk16) {
  return static_cast<uint32_t>((row >> 3) * 1024 + chunk16 * 128 + (row & 7) * 16);
}

__device__ __forceinline__ float sigm(float x) {
  const float e = expf(-fabsf(x));
  return x >= 0.0f ? 1.0f / (1.0f + e) : e / (1.0f + e);
}

// R_g element (row a, col b) of the dense (K, K) matrix in the blocked layout
__device__ __forceinline__ float r_elem(const LstmStepParams& p, int g, int a, int b) {
  const int kb = p.K / p.bk;
  const int64_t off = static_cast<int64_t>(g) * p.K * p.K +
                      (static_cast<int64_t>(a / p.bk) * kb + b / p.bk) * p.bk * p.bk + (b % p.bk) * p.bk + a % p.bk;
  return p.R[off];
}

template <bool kTF32>
__device__ __forceinline__ uint4 pack16(const float* v) {
  uint4 r;
  if constexpr (kTF32) {
    r.x = f32_to_tf32(v[0]); r.y = f32_to_tf32(v[1]); r.z = f32_to_tf32(v[2]); r.w = f32_to_tf32(v[3]);
  } else {
    r.x = pack_bf16x2(v[0], v[1]); r.y = pack_bf16x2(v[2], v[3]);
    r.z = pack_bf16x2(v[4], v[5]); r.w = pack_bf16x2(v[6], v[7]);
  }
  return r;
}

template <bool kTF32, int kMode>
__global__ void __launch_bounds__(kThreads, 1) lstm_step_kernel(const LstmStepParams p) {
  constexpr int kE = kTF32 ? 4 : 8;                   // elements per 16 B
  constexpr int kCE = kChunkBytes / (kTF32 ? 4 : 2);  // K elements per stage
  constexpr int kMmaK = kTF32 ? 8 : 16;
  constexpr int kBRows = kMode == kFwd ? 4 * kHid : kHid;  // MMA N
  constexpr int kAOp = kRows * kChunkBytes;
  constexpr int kBOp = kBRows * kChunkBytes;
  constexpr int kStage = kAOp + kBOp;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStage);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + kStages + 1);

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int k0 = blockIdx.x * kHid;  // hidden-unit slice
  const int n0 = blockIdx.y * kRows;
  const int kdim = kMode == kFwd ? p.K : 4 * p.K;
  const bool have_rec = kMode == kFwd || p.dpre_next != nullptr;

  if (tid == 0) {
    for (int s = 0; s < kStages + 1; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int n_chunks = have_rec ? (kdim + kCE - 1) / kCE : 0;
  const uint32_t idesc = make_idesc(kTF32 ? kFmtTF32 : kFmtBF16, kRows, kBRows, 0, 0);

  for (int s = 0; s < n_chunks; ++s) {
    const int st = s % kStages;
    const int kc = s * kCE;
    if (s >= kStages) mbar_wait(&bars[st], ((s / kStages) + 1) & 1);
    uint8_t* a_op = smem + st * kStage;
    uint8_t* b_op = a_op + kAOp;
    // A: rows n, K-dim j (fwd: h_{t-1}[n][j]; bwd: dpre_{t+1}[n][(g,j)])
    for (int u = tid; u < kRows * 8; u += kThreads) {
      const int c = u & 7, r = u >> 3, n = n0 + r;
      float v[8];
#pragma unroll
      for (int t = 0; t < kE; ++t) {
        const int kk = kc + c * kE + t;
        float x = 0.0f;
        if (n < p.N && kk < kdim) x = (kMode == kFwd) ? p.h_prev[static_cast<int64_t>(n) * p.K + kk]
                                                      : p.dpre_next[static_cast<int64_t>(n) * 4 * p.K + kk];
        v[t] = x;
      }
      *reinterpret_cast<uint4*>(a_op + canon_off(r, c)) = pack16<kTF32>(v);
    }
    // B: fwd rows (g, k) -> R_g[k][j];  bwd rows k -> R_g[j][k] with kk = (g, j)
    for (int u = tid; u < kBRows * 8; u += kThreads) {
      const int i = u % kBRows, c = u / kBRows;
      float v[8];
#pragma unroll
      for (int t = 0; t < kE; ++t) {
        const int kk = kc + c * kE + t;
        float x = 0.0f;
        if (kk < kdim) {
          if (kMode == kFwd) {
            const int g = i / kHid, k = k0 + i % kHid;
            if (k < p.K) x = r_elem(p, g, k, kk);
          } else {
            const int k = k0 + i, g = kk / p.K, j = kk % p.K;
            if (k < p.K) x = r_elem(p, g, j, k);
          }
        }
        v[t] = x;
      }
      *reinterpret_cast<uint4*>(b_op + canon_off(i, c)) = pack16<kTF32>(v);
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t ab = smem_u32(a_op), bb = smem_u32(b_op);
#pragma unroll
      for (int kk = 0; kk < kCE / kMmaK; ++kk) {
        mma_ss<kTF32>(tmem, make_smem_desc(ab + kk * 256, 128, 1024, kSwizzleNone),
                      make_smem_desc(bb + kk * 256, 128, 1024, kSwizzleNone), idesc, (s > 0 || kk > 0) ? 1u : 0u);
      }
      mma_commit(&bars[st]);
      if (s == n_chunks - 1) mma_commit(&bars[kStages]);
    }
  }
  if (n_chunks > 0) {
    mbar_wait(&bars[kStages], 0);
    tc_fence_after();
  }

  // ---- fused epilogue: thread = one minibatch row, 64 hidden units ----------
  const int n = n0 + warp * 32 + lane;
  const bool ok = n < p.N;
  const uint32_t tl = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  for (int c0 = 0; c0 < kHid; c0 += 16) {
    uint32_t a[4][16];
    if (kMode == kFwd) {
#pragma unroll
      for (int g = 0; g < 4; ++g) tmem_ld16(tl + g * kHid + c0, a[g]);
      tmem_ld_wait();
    } else if (n_chunks > 0) {
      tmem_ld16(tl + c0, a[0]);
      tmem_ld_wait();
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) a[0][j] = 0u;
    }
    if (!ok) continue;
#pragma unroll 4
    for (int j = 0; j < 16; ++j) {
      const int k = k0 + c0 + j;
      if (k >= p.K) break;
      const int64_t e = static_cast<int64_t>(n) * p.K + k;            // [N][K]
      const int64_t e4 = static_cast<int64_t>(n) * 4 * p.K + k;       // [N][4][K], gate stride K
      if (kMode == kFwd) {
        const float gi = sigm(__uint_as_float(a[0][j]) + p.gx[e4]);
        const float gc = tanhf(__uint_as_float(a[1][j]) + p.gx[e4 + p.K]);
        const float gf = sigm(__uint_as_float(a[2][j]) + p.gx[e4 + 2 * p.K]);
        const float go = sigm(__uint_as_float(a[3][j]) + p.gx[e4 + 3 * p.K]);
        const float sp = p.s_prev != nullptr ? p.s_prev[e] : 0.0f;
        const float s = gf * sp + gi * gc;
        p.s_out[e] = s;
        p.h_out[e] = go * tanhf(s);
        p.gates_out[e4] = gi;
        p.gates_out[e4 + p.K] = gc;
        p.gates_out[e4 + 2 * p.K] = gf;
        p.gates_out[e4 + 3 * p.K] = go;
      } else if (kMode == kBwdRaw) {
        p.raw_out[e] = __uint_as_float(a[0][j]);
      } else {
        const float dh = p.dh_in[e] + __uint_as_float(a[0][j]);
        const float gi = p.gates[e4], gc = p.gates[e4 + p.K], gf = p.gates[e4 + 2 * p.K], go = p.gates[e4 + 3 * p.K];
        const float s = p.s_cur[e];
        const float sp = p.s_prev != nullptr ? p.s_prev[e] : 0.0f;
        const float ts = tanhf(s);
        const float ds = dh * go * (1.0f - ts * ts) + (p.ds_in != nullptr ? p.ds_in[e] : 0.0f);
        p.dpre_out[e4] = ds * gc * gi * (1.0f - gi);
        p.dpre_out[e4 + p.K] = ds * gi * (1.0f - gc * gc);
        p.dpre_out[e4 + 2 * p.K] = ds * sp * gf * (1.0f - gf);
        p.dpre_out[e4 + 3 * p.K] = dh * ts * go * (1.0f - go);
        p.ds_out[e] = ds * gf;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

template <bool kTF32, int kMode>
int launch_step(const LstmStepParams& p, cudaStream_t stream) {
  constexpr int kBRows = kMode == kFwd ? 4 * kHid : kHid;
  constexpr int kSmem = kStages * (kRows * kChunkBytes + kBRows * kChunkBytes) + 1024 + 256;
  auto kern = lstm_step_kernel<kTF32, kMode>;
  static int attr = 0;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return set_cuda_error(e, "lstm smem attribute");
    attr = 1;
  }
  dim3 grid((p.K + kHid - 1) / kHid, (p.N + kRows - 1) / kRows);
  g_launches.fetch_add(1);
  kern<<<grid, kThreads, kSmem, stream>>>(p);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BRK_OK : set_cuda_error(e, "lstm step launch");
}

int check(int N, int K, int bk, int compute) {
  if (N <= 0 || K <= 0 || bk <= 0 || K % bk) return set_error(BRK_ERR_CONTRACT, "lstm: b_k must divide K");
  if (compute != BRK_COMPUTE_TF32 && compute != BRK_COMPUTE_BF16)
    return set_error(BRK_ERR_CONTRACT, "lstm: bad compute code");
  return BRK_OK;
}

}  // namespace
}  // namespace brk

using namespace brk;

extern "C" {

BRK_API int brk_lstm_fwd_step(const float* h_prev, const float* s_prev, const float* gx, const float* R,
                              float* h_out, float* s_out, float* gates_out, int N, int K, int b_k, int compute,
                              void* stream) {
  int rc = check(N, K, b_k, compute);
  if (rc) return rc;
  if (h_prev == nullptr || gx == nullptr || R == nullptr || h_out == nullptr || s_out == nullptr ||
      gates_out == nullptr)
    return set_error(BRK_ERR_CONTRACT, "lstm_fwd_step: null pointer");
  LstmStepParams p{};
  p.mode = kFwd;
  p.N = N; p.K = K; p.bk = b_k;
  p.h_prev = h_prev; p.s_prev = s_prev; p.gx = gx; p.R = R;
  p.h_out = h_out; p.s_out = s_out; p.gates_out = gates_out;
  auto s = static_cast<cudaStream_t>(stream);
  return compute == BRK_COMPUTE_TF32 ? launch_step<true, kFwd>(p, s) : launch_step<false, kFwd>(p, s);
}

BRK_API int brk_lstm_bwd_step(const float* dpre_next, const float* R, const float* dh_in, const float* gates,
                              const float* s_cur, const float* s_prev, const float* ds_in, float* dpre_out,
                              float* ds_out, int N, int K, int b_k, int compute, void* stream) {
  int rc = check(N, K, b_k, compute);
  if (rc) return rc;
  if (R == nullptr || dh_in == nullptr || gates == nullptr || s_cur == nullptr || dpre_out == nullptr ||
      ds_out == nullptr)
    return set_error(BRK_ERR_CONTRACT, "lstm_bwd_step: null pointer");
  LstmStepParams p{};
  p.mode = kBwd;
  p.N = N; p.K = K; p.bk = b_k;
  p.dpre_next = dpre_next; p.R = R; p.dh_in = dh_in; p.gates = gates; p.s_cur = s_cur;
  p.s_prev = s_prev; p.ds_in = ds_in; p.dpre_out = dpre_out; p.ds_out = ds_out;
  auto s = static_cast<cudaStream_t>(stream);
  return compute == BRK_COMPUTE_TF32 ? launch_step<true, kBwd>(p, s) : launch_step<false, kBwd>(p, s);
}

BRK_API int brk_lstm_recurrent_grad(const float* dpre, const float* R, float* out, int N, int K, int b_k,
                                    int compute, void* stream) {
  int rc = check(N, K, b_k, compute);
  if (rc) return rc;
  if (dpre == nullptr || R == nullptr || out == nullptr)
    return set_error(BRK_ERR_CONTRACT, "lstm_recurrent_grad: null pointer");
  LstmStepParams p{};
  p.mode = kBwdRaw;
  p.N = N; p.K = K; p.bk = b_k;
  p.dpre_next = dpre; p.R = R; p.raw_out = out;
  auto s = static_cast<cudaStream_t>(stream);
  return compute == BRK_COMPUTE_TF32 ? launch_step<true, kBwdRaw>(p, s) : launch_step<false, kBwdRaw>(p, s);
}

}  // extern "C"
