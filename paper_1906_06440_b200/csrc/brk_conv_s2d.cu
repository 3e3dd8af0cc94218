// brk_conv_s2d.cu — stride-2 small-channel convolutions (the ResNet-50 stem,
// reference cnn.py:201-334 with C = 3, 7x7, stride 2, pad 3) as space-to-depth
// implicit GEMMs on the tcgen05 engine.
//
// A stride-2 conv over C <= 4 channels is rewritten exactly (same products, the
// sum reordered) as a stride-1 conv over 64 channels:
//
//   r' = r + e_h, r' = 2u + a   (e_h = 2*off_h - pad_h, off_h = ceil(pad_h / 2))
//   s' = s + e_w, s' = 2v + b
//   out(p, q) = sum_{u, v, a, b, c} x[2(p - off_h + u) + a][2(q - off_w + v) + b][c] W[k][c][r][s]
//
// The unfold kernel writes  xs[n][i][q][v*16 + (2a + b)*C + c]
//   = x[n][2(i - off_h) + a][2(q - off_w + v) + b][c]     (zero outside the image / past 4C)
// for i in [0, P + R' - 1), q in [0, Q): one 128-byte (64-channel bf16) row per pixel,
// the engine's blocked [N][1][H'][W'][64] activation.  Then
//   fwd: out = conv(xs, W'', R' x 1, stride 1, pad 0)                (brk_conv_fwd)
//   upd: dW'' = conv_upd(xs, dO, R' x 1), dW = gather(dW'')           (brk_conv_upd)
//   bwd: dxs = conv(dO, W''flip, R' x 1, pad R'-1), dX = fold(dxs)   (brk_conv_fwd)
// with W''[kb][0][u][0][v*16 + (2a+b)*C + c][k] = W[k][c][2u+a-e_h][2v+b-e_w] (0 outside).
// The explicit im2col path (brk_conv_small.cu) wrote 147-wide columns per output pixel
// (976 MB at N = 256) and a 1 ms gather col2im; the unfold writes 64 channels per output
// pixel of a 115-row image (422 MB) and the taps along H come from the engine's TMA im2col.
#include <algorithm>
#include <cstdint>
#include <cuda_bf16.h>

#include "brk_internal.h"

extern "C" {
int brk_conv_fwd(const void* in, const void* w, const float* bias, void* out, int N, int C, int K, int H, int W,
                 int R, int S, int stride, int pad_h, int pad_w, int b_c, int b_k, int act, int dtype, void* stream);
int brk_conv_upd(const void* in, const void* dout, float* dw, void* w_sgd, float lr, void* workspace,
                 size_t ws_bytes, int N, int C, int K, int H, int W, int R, int S, int stride, int pad_h, int pad_w,
                 int b_c, int b_k, int dtype, void* stream);
size_t brk_conv_upd_workspace(int N, int C, int K, int H, int W, int R, int S, int stride, int pad_h, int pad_w);
}

namespace brk {
namespace {

constexpr int kSlot = 16;  // channels per horizontal tap v (4C <= 16)

struct S2dGeom {
  int N, C, K, H, W, R, S, pad_h, pad_w;
  int P, Q;          // output extent
  int off_h, off_w;  // ceil(pad / 2)
  int e_h, e_w;      // 2 * off - pad (0 or 1)
  int Rs, Ss;        // taps of the stride-1 conv along H (R') and along W (S' <= 4)
  int Hs;            // rows of the unfolded image: P + R' - 1
};

int s2d_geom(S2dGeom& g, int N, int C, int K, int H, int W, int R, int S, int pad_h, int pad_w) {
  if (N <= 0 || C <= 0 || K <= 0 || H <= 0 || W <= 0 || R <= 0 || S <= 0 || pad_h < 0 || pad_w < 0)
    return set_error(BRK_ERR_CONTRACT, "conv s2d: bad geometry");
  g.N = N; g.C = C; g.K = K; g.H = H; g.W = W; g.R = R; g.S = S; g.pad_h = pad_h; g.pad_w = pad_w;
  g.P = (H + 2 * pad_h - R) / 2 + 1;
  g.Q = (W + 2 * pad_w - S) / 2 + 1;
  g.off_h = (pad_h + 1) / 2; g.off_w = (pad_w + 1) / 2;
  g.e_h = 2 * g.off_h - pad_h; g.e_w = 2 * g.off_w - pad_w;
  g.Rs = (R + g.e_h + 1) / 2; g.Ss = (S + g.e_w + 1) / 2;
  g.Hs = g.P + g.Rs - 1;
  if (g.P <= 0 || g.Q <= 0) return set_error(BRK_ERR_CONTRACT, "conv s2d: empty output");
  if (4 * C > kSlot || g.Ss * kSlot > 64)
    return set_error(BRK_ERR_CONTRACT, "conv s2d: needs C <= 4 and ceil((S + pad%2)/2) <= 4");
  if (g.Rs > 16 || K % 64) return set_error(BRK_ERR_CONTRACT, "conv s2d: needs R' <= 16 and K % 64 == 0");
  return BRK_OK;
}

// One CTA per unfolded row (n, i) (a non-persistent grid: many rows in flight per SM hide
// the load -> store latency of each row): the two image rows 2(i - off_h) + {0, 1} are
// staged in shared memory with 16-byte loads behind a zero margin, then every thread
// assembles 16-byte groups (8 channels) of output pixels and stores them: the CTA writes
// its Q x 128 B row with consecutive 16 B stores.
//   staged[a][margin + w*C + c] = x[n][2(i - off_h) + a][w][c]   (zero outside 0 <= w < W)
__global__ void __launch_bounds__(128) s2d_unfold_kernel(const __nv_bfloat16* __restrict__ x,
                                                         __nv_bfloat16* __restrict__ xs, S2dGeom g, int rowlen,
                                                         int margin) {
  extern __shared__ __align__(16) uint8_t sm[];
  __nv_bfloat16* rows = reinterpret_cast<__nv_bfloat16*>(sm);  // [2][rowlen]
  __shared__ int tab[kSlot];  // staged offset of channel t of a tap group (-1: zero channel)
  if (threadIdx.x < kSlot) {
    const int t = threadIdx.x;
    int off = -1;
    if (t < 4 * g.C) {
      const int ab = t / g.C, c = t - ab * g.C;
      off = (ab >> 1) * rowlen + margin - 2 * g.off_w * g.C + (ab & 1) * g.C + c;
    }
    tab[t] = off;
  }
  const int n = blockIdx.x / g.Hs, i = blockIdx.x - (blockIdx.x / g.Hs) * g.Hs;
  const int wc = g.W * g.C;
  const bool vec = (wc % 8) == 0 && (margin % 8) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  for (int a = 0; a < 2; ++a) {
    const int h = 2 * (i - g.off_h) + a;
    const bool hv = h >= 0 && h < g.H;
    __nv_bfloat16* dst = rows + a * rowlen;
    const __nv_bfloat16* src = x + (static_cast<int64_t>(n) * g.H + (hv ? h : 0)) * wc;
    if (vec) {
      uint4* d4 = reinterpret_cast<uint4*>(dst);
      const uint4* s4 = reinterpret_cast<const uint4*>(src);
      for (int e = threadIdx.x; e < rowlen / 8; e += blockDim.x) {
        const int w8 = e - margin / 8;
        d4[e] = (hv && w8 >= 0 && w8 < wc / 8) ? s4[w8] : make_uint4(0u, 0u, 0u, 0u);
      }
    } else {
      for (int e = threadIdx.x; e < rowlen; e += blockDim.x) {
        const int w1 = e - margin;
        dst[e] = (hv && w1 >= 0 && w1 < wc) ? src[w1] : __float2bfloat16_rn(0.0f);
      }
    }
  }
  __syncthreads();
  uint4* out = reinterpret_cast<uint4*>(xs + static_cast<int64_t>(blockIdx.x) * g.Q * 64);
  for (int it = threadIdx.x; it < g.Q * 8; it += blockDim.x) {
    const int q = it >> 3, grp = it & 7;
    const int v = grp >> 1, t0 = (grp & 1) * 8;
    // image column 2(q - off_w + v) + b: staged at margin + (2(q + v) - 2 off_w + b) * C
    const int base = 2 * (q + v) * g.C;
    __align__(16) __nv_bfloat16 val[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int o = tab[t0 + e];
      val[e] = (o >= 0 && v < g.Ss) ? rows[o + base] : __float2bfloat16_rn(0.0f);
    }
    out[it] = *reinterpret_cast<const uint4*>(val);
  }
}

// W''[kb][0][u][0][c''][k] (bf16, blocked [K_b][1][R'][1][64][64]) and/or the flipped,
// C<->K-swapped filter of the backward-data conv  Wf[0][kb][R'-1-u][0][k][c''].
__global__ void s2d_weight_kernel(const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ w2,
                                  __nv_bfloat16* __restrict__ wf, S2dGeom g) {
  const int kb_n = g.K / 64;
  const int64_t total = static_cast<int64_t>(kb_n) * g.Rs * 64 * 64;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int kk = static_cast<int>(idx & 63), cc = static_cast<int>((idx >> 6) & 63);
    const int64_t rest = idx >> 12;
    const int u = static_cast<int>(rest % g.Rs), kb = static_cast<int>(rest / g.Rs);
    const int v = cc / kSlot, t = cc - v * kSlot;
    __nv_bfloat16 val = __float2bfloat16_rn(0.0f);
    if (t < 4 * g.C) {
      const int ab = t / g.C, c = t - ab * g.C;
      const int r = 2 * u + (ab >> 1) - g.e_h, s = 2 * v + (ab & 1) - g.e_w;
      if (r >= 0 && r < g.R && s >= 0 && s < g.S)
        val = w[((((static_cast<int64_t>(kb) * g.R + r) * g.S + s) * g.C + c) << 6) + kk];
    }
    if (w2 != nullptr) w2[idx] = val;
    if (wf != nullptr) wf[((((static_cast<int64_t>(kb) * g.Rs + (g.Rs - 1 - u)) << 6) + kk) << 6) + cc] = val;
  }
}

// dW[kb][0][r][s][c][k] (fp32) = dW''[kb][0][u][0][c''][k] at (u, c'') of tap (r, s, c).
__global__ void s2d_dweight_kernel(const float* __restrict__ dw2, float* __restrict__ dw, S2dGeom g) {
  const int64_t total = static_cast<int64_t>(g.K / 64) * g.R * g.S * g.C * 64;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int kk = static_cast<int>(idx & 63);
    int64_t rest = idx >> 6;
    const int c = static_cast<int>(rest % g.C); rest /= g.C;
    const int s = static_cast<int>(rest % g.S); rest /= g.S;
    const int r = static_cast<int>(rest % g.R);
    const int kb = static_cast<int>(rest / g.R);
    const int rr = r + g.e_h, ss = s + g.e_w;
    const int u = rr >> 1, v = ss >> 1;
    const int cc = v * kSlot + ((rr & 1) * 2 + (ss & 1)) * g.C + c;
    dw[idx] = dw2[((((static_cast<int64_t>(kb) * g.Rs + u) << 6) + cc) << 6) + kk];
  }
}

// dX[n][0][h][w][c] = sum_v dxs[n][i + off_h][j + off_w - v][v*16 + (2a+b)*C + c]
// (h = 2i + a, w = 2j + b): one CTA per image row pair i (non-persistent grid); the
// unfolded row is staged in shared memory with 16 B loads, then each thread produces dX
// elements of image rows 2i, 2i + 1 (fp32 sum of the S' contributions in a fixed order),
// consecutive threads consecutive elements.
__global__ void __launch_bounds__(128) s2d_fold_kernel(const __nv_bfloat16* __restrict__ dxs,
                                                       __nv_bfloat16* __restrict__ dx, S2dGeom g) {
  extern __shared__ __align__(16) uint8_t sm[];
  __nv_bfloat16* row = reinterpret_cast<__nv_bfloat16*>(sm);  // [Q][64]
  const int ih = (g.H + 1) / 2;
  const int n = blockIdx.x / ih, i = blockIdx.x - (blockIdx.x / ih) * ih;
  const int is = i + g.off_h;
  const uint4* src = reinterpret_cast<const uint4*>(dxs + (static_cast<int64_t>(n) * g.Hs + is) * g.Q * 64);
  uint4* srow = reinterpret_cast<uint4*>(row);
  for (int it = threadIdx.x; it < g.Q * 8; it += blockDim.x)
    srow[it] = is < g.Hs ? src[it] : make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();
  const int wc = g.W * g.C;
  const int rows_here = 2 * i + 1 < g.H ? 2 : 1;
  for (int it = threadIdx.x; it < rows_here * wc; it += blockDim.x) {
    const int a = it >= wc ? 1 : 0;
    const int rem = it - a * wc;
    const int w = rem / g.C, c = rem - w * g.C;
    const int j = w >> 1, b = w & 1;
    float acc = 0.0f;
    for (int v = 0; v < g.Ss; ++v) {
      const int q = j + g.off_w - v;
      if (q >= 0 && q < g.Q) acc += __bfloat162float(row[q * 64 + v * kSlot + (a * 2 + b) * g.C + c]);
    }
    dx[(static_cast<int64_t>(n) * g.H + 2 * i + a) * wc + rem] = __float2bfloat16_rn(acc);
  }
}

int grid_for(int64_t items, int per_sm = 8) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t cap = static_cast<int64_t>(per_sm) * sms;
  return static_cast<int>(items < cap ? (items > 0 ? items : 1) : cap);
}

size_t align256(size_t b) { return (b + 255) / 256 * 256; }

size_t unfold_bytes(const S2dGeom& g) { return static_cast<size_t>(g.N) * g.Hs * g.Q * 64 * 2; }
size_t weight_bytes(const S2dGeom& g) { return static_cast<size_t>(g.K / 64) * g.Rs * 64 * 64 * 2; }

int run_unfold(const S2dGeom& g, const void* x, void* xs, cudaStream_t st) {
  // staged row: a zero margin of >= 2 off_w pixels (rounded to 16 B), the image row, and
  // zeros up to the last column a tap reads (2 (Q + S') + 1 pixels past the margin start)
  const int margin = (2 * g.off_w * g.C + 7) / 8 * 8;
  const int need = margin - 2 * g.off_w * g.C + (2 * (g.Q + g.Ss) + 2) * g.C;
  const int rowlen = (std::max(need, margin + g.W * g.C) + 7) / 8 * 8;
  const int smem = 2 * rowlen * 2;
  if (smem > 48 * 1024) return set_error(BRK_ERR_CONTRACT, "conv s2d: image rows too wide to stage");
  g_launches.fetch_add(1);
  s2d_unfold_kernel<<<g.N * g.Hs, 128, smem, st>>>(static_cast<const __nv_bfloat16*>(x),
                                                  static_cast<__nv_bfloat16*>(xs), g, rowlen, margin);
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? BRK_OK : set_cuda_error(err, "conv s2d unfold");
}

int run_weight(const S2dGeom& g, const void* w, void* w2, void* wf, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(g.K / 64) * g.Rs * 4096;
  g_launches.fetch_add(1);
  s2d_weight_kernel<<<grid_for((total + 255) / 256), 256, 0, st>>>(
      static_cast<const __nv_bfloat16*>(w), static_cast<__nv_bfloat16*>(w2), static_cast<__nv_bfloat16*>(wf), g);
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? BRK_OK : set_cuda_error(err, "conv s2d weight");
}

}  // namespace
}  // namespace brk

using namespace brk;

extern "C" {

BRK_API int brk_conv_s2d_shape(int N, int C, int K, int H, int W, int R, int S, int pad_h, int pad_w, int* out4) {
  S2dGeom g;
  const int rc = s2d_geom(g, N, C, K, H, W, R, S, pad_h, pad_w);
  if (rc) return rc;
  if (out4 != nullptr) { out4[0] = g.Hs; out4[1] = g.Q; out4[2] = g.Rs; out4[3] = g.P; }
  return BRK_OK;
}

BRK_API size_t brk_conv_s2d_workspace(int N, int C, int K, int H, int W, int R, int S, int pad_h, int pad_w) {
  S2dGeom g;
  if (s2d_geom(g, N, C, K, H, W, R, S, pad_h, pad_w)) return 0;
  const size_t upd = brk_conv_upd_workspace(N, 64, K, g.Hs, g.Q, g.Rs, 1, 1, 0, 0);
  const size_t dw2 = static_cast<size_t>(g.K / 64) * g.Rs * 4096 * 4;
  return align256(unfold_bytes(g)) + align256(weight_bytes(g)) + align256(dw2) + align256(upd);
}

BRK_API int brk_conv_s2d_unfold(const void* x, void* xs, int N, int C, int H, int W, int R, int S, int pad_h,
                                int pad_w, void* stream) {
  S2dGeom g;
  const int rc = s2d_geom(g, N, C, 64, H, W, R, S, pad_h, pad_w);
  if (rc) return rc;
  return run_unfold(g, x, xs, static_cast<cudaStream_t>(stream));
}

BRK_API int brk_conv_s2d_fwd(const void* x, const void* w, void* out, void* workspace, size_t ws_bytes, int N, int C,
                             int K, int H, int W, int R, int S, int pad_h, int pad_w, void* stream) {
  S2dGeom g;
  int rc = s2d_geom(g, N, C, K, H, W, R, S, pad_h, pad_w);
  if (rc) return rc;
  if (workspace == nullptr || ws_bytes < brk_conv_s2d_workspace(N, C, K, H, W, R, S, pad_h, pad_w))
    return set_error(BRK_ERR_CONTRACT, "conv s2d fwd: workspace smaller than brk_conv_s2d_workspace()");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
  void* xs = ws;
  void* w2 = ws + align256(unfold_bytes(g));
  if ((rc = run_unfold(g, x, xs, st))) return rc;
  if ((rc = run_weight(g, w, w2, nullptr, st))) return rc;
  return brk_conv_fwd(xs, w2, nullptr, out, N, 64, K, g.Hs, g.Q, g.Rs, 1, 1, 0, 0, 64, 64, 0, BRK_BF16, stream);
}

BRK_API int brk_conv_s2d_upd(const void* x, const void* dout, float* dw, void* workspace, size_t ws_bytes, int N,
                             int C, int K, int H, int W, int R, int S, int pad_h, int pad_w, void* stream) {
  S2dGeom g;
  int rc = s2d_geom(g, N, C, K, H, W, R, S, pad_h, pad_w);
  if (rc) return rc;
  if (workspace == nullptr || ws_bytes < brk_conv_s2d_workspace(N, C, K, H, W, R, S, pad_h, pad_w))
    return set_error(BRK_ERR_CONTRACT, "conv s2d upd: workspace smaller than brk_conv_s2d_workspace()");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
  void* xs = ws;
  float* dw2 = reinterpret_cast<float*>(ws + align256(unfold_bytes(g)) + align256(weight_bytes(g)));
  char* uws = reinterpret_cast<char*>(dw2) + align256(static_cast<size_t>(g.K / 64) * g.Rs * 4096 * 4);
  const size_t ubytes = brk_conv_upd_workspace(N, 64, K, g.Hs, g.Q, g.Rs, 1, 1, 0, 0);
  if ((rc = run_unfold(g, x, xs, st))) return rc;
  if ((rc = brk_conv_upd(xs, dout, dw2, nullptr, 0.0f, ubytes ? uws : nullptr, ubytes, N, 64, K, g.Hs, g.Q, g.Rs, 1,
                         1, 0, 0, 64, 64, BRK_BF16, stream)))
    return rc;
  const int64_t total = static_cast<int64_t>(g.K / 64) * g.R * g.S * g.C * 64;
  g_launches.fetch_add(1);
  s2d_dweight_kernel<<<grid_for((total + 255) / 256), 256, 0, st>>>(dw2, dw, g);
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? BRK_OK : set_cuda_error(err, "conv s2d dweight");
}

BRK_API int brk_conv_s2d_bwd_data(const void* dout, const void* w, void* dx, void* workspace, size_t ws_bytes, int N,
                                  int C, int K, int H, int W, int R, int S, int pad_h, int pad_w, void* stream) {
  S2dGeom g;
  int rc = s2d_geom(g, N, C, K, H, W, R, S, pad_h, pad_w);
  if (rc) return rc;
  if (workspace == nullptr || ws_bytes < brk_conv_s2d_workspace(N, C, K, H, W, R, S, pad_h, pad_w))
    return set_error(BRK_ERR_CONTRACT, "conv s2d bwd: workspace smaller than brk_conv_s2d_workspace()");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
  void* dxs = ws;
  void* wf = ws + align256(unfold_bytes(g));
  if ((rc = run_weight(g, w, nullptr, wf, st))) return rc;
  // dxs = conv(dO, Wf): K input channels, 64 output channels, R' x 1 taps, pad R' - 1 along H
  if ((rc = brk_conv_fwd(dout, wf, nullptr, dxs, N, K, 64, g.P, g.Q, g.Rs, 1, 1, g.Rs - 1, 0, 64, 64, 0, BRK_BF16,
                         stream)))
    return rc;
  const int ih = (g.H + 1) / 2;
  g_launches.fetch_add(1);
  if (g.Q * 128 > 48 * 1024) return set_error(BRK_ERR_CONTRACT, "conv s2d: output rows too wide to stage");
  s2d_fold_kernel<<<N * ih, 128, g.Q * 128, st>>>(
      static_cast<const __nv_bfloat16*>(dxs), static_cast<__nv_bfloat16*>(dx), g);
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? BRK_OK : set_cuda_error(err, "conv s2d fold");
}

}  // extern "C"
