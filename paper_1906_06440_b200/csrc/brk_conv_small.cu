// brk_conv_small.cu — layout kernels of the small-channel convolution path (the
// 3-channel ResNet stem, reference cnn.py:201-334 with b_c = C < 64).
//
// A 64-channel TMA im2col box would be >95 % padding for C = 3, so these convs
// run as explicit-im2col GEMMs on the tcgen05 engine (brk_gemm_dense):
//     fwd: out[pix][k]   = col[pix][(r,s,c)] . W[k][(r,s,c)]
//     upd: dW[(r,s,c)][k] = sum_pix col[pix][(r,s,c)] dO[pix][k]
//     bwd: dcol[pix][(r,s,c)] = dO[pix][k] . W[k][(r,s,c)],  dX = col2im(dcol)
// with pix = (n, p, q) and the column order (r, s, c) of the reference's
// blocked weight [K_b][C_b][R][S][b_c][b_k] (so dW rows map onto it directly).
#include <algorithm>
#include <cstdint>
#include <cuda_bf16.h>

#include "brk_internal.h"

namespace brk {
namespace {

struct SmallGeom {
  int N, C, H, W, R, S, stride, pad_h, pad_w, b_c, P, Q;
  int64_t ldcol;
};

// col[pix][j] (bf16, row stride ldcol), j = (r*S + s)*C + c; zero outside the image.
// One CTA per output row (n, p): the R input rows it reads are staged in shared memory
// with coalesced loads, then each thread assembles whole 16 B groups of a col row and
// stores them as one vector (2-byte scattered stores were L2-transaction bound).
// Columns from R*S*C up to the next multiple of 8 are written as zeros, the rest of
// the row is left untouched (the GEMMs read K = R*S*C).
__global__ void __launch_bounds__(256) im2col_kernel(const __nv_bfloat16* __restrict__ in,
                                                     __nv_bfloat16* __restrict__ col, SmallGeom g) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int cb_n = (g.C + g.b_c - 1) / g.b_c;
  const int rsc = g.R * g.S * g.C;
  const int groups = (rsc + 7) / 8;
  const int wc = g.W * g.C;
  // column j -> (s, offset of (r, c) in the staged rows): no divisions in the hot loop
  int2* tab = reinterpret_cast<int2*>(sm);
  __nv_bfloat16* rows = reinterpret_cast<__nv_bfloat16*>(sm + ((groups * 8 * sizeof(int2) + 15) / 16) * 16);
  // stored element-major (tab[e * groups + grp]): the threads of a warp read consecutive
  // entries for the same e (a group-major table put them 64 B apart: 16-way bank conflicts)
  for (int j = threadIdx.x; j < groups * 8; j += blockDim.x) {
    const int grp = j >> 3, e = j & 7;
    int2 v = make_int2(-1, 0);
    if (j < rsc) {
      const int t = j / g.C, c = j - (j / g.C) * g.C;
      const int r = t / g.S, s = t - (t / g.S) * g.S;
      v = make_int2(s, r * wc + c);
    }
    tab[e * groups + grp] = v;
  }
  const bool dense_rows = cb_n == 1 && wc % 8 == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  for (int np = blockIdx.x; np < g.N * g.P; np += gridDim.x) {
    const int n = np / g.P, p = np - (np / g.P) * g.P;
    __syncthreads();  // the table is built / the previous row's readers are done
    for (int r = 0; r < g.R; ++r) {
      const int h = p * g.stride - g.pad_h + r;
      const bool hv = h >= 0 && h < g.H;
      if (dense_rows) {  // one channel block: the input row is a contiguous [W][C] run
        const uint4* src = reinterpret_cast<const uint4*>(in + (static_cast<int64_t>(n) * g.H + h) * wc);
        uint4* dst = reinterpret_cast<uint4*>(rows + r * wc);
        for (int i = threadIdx.x; i < wc / 8; i += blockDim.x) dst[i] = hv ? src[i] : make_uint4(0u, 0u, 0u, 0u);
      } else {
        for (int i = threadIdx.x; i < wc; i += blockDim.x) {
          const int w = i / g.C, c = i - (i / g.C) * g.C;
          rows[r * wc + i] = hv ? in[((static_cast<int64_t>(n) * cb_n + c / g.b_c) * g.H + h) * g.W * g.b_c +
                                     static_cast<int64_t>(w) * g.b_c + c % g.b_c]
                                : __float2bfloat16_rn(0.0f);
        }
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < g.Q * groups; i += blockDim.x) {
      const int q = i / groups, grp = i - (i / groups) * groups;
      const int w0 = q * g.stride - g.pad_w;
      __align__(16) __nv_bfloat16 v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int2 te = tab[e * groups + grp];
        const int w = w0 + te.x;
        v[e] = (te.x >= 0 && w >= 0 && w < g.W) ? rows[te.y + w * g.C] : __float2bfloat16_rn(0.0f);
      }
      *reinterpret_cast<uint4*>(col + (static_cast<int64_t>(np) * g.Q + q) * g.ldcol + grp * 8) =
          *reinterpret_cast<const uint4*>(v);
    }
  }
}

// dX[n][c_b][h][w][c'] = sum over the taps whose output pixel lands on (h, w) of
// dcol[(n, p, q)][(r*S + s)*C + c].  Gather form: one thread per input pixel, only the
// contributing taps are visited (p from the first with stride*p + R-1 >= h + pad), fp32
// sums in a fixed tap order — deterministic, no atomics.
__global__ void __launch_bounds__(128) col2im_kernel(const __nv_bfloat16* __restrict__ dcol,
                                                     __nv_bfloat16* __restrict__ dx, SmallGeom g) {
  const int cb_n = (g.C + g.b_c - 1) / g.b_c;
  const int w = blockIdx.x * blockDim.x + threadIdx.x;  // grid.y walks input rows (n, h)
  if (w >= g.W) return;
  for (int nh = blockIdx.y; nh < g.N * g.H; nh += gridDim.y) {
    const int n = nh / g.H, h = nh - (nh / g.H) * g.H;
    const int hh = h + g.pad_h, ww = w + g.pad_w;
    const int p_lo = hh >= g.R - 1 ? (hh - (g.R - 1) + g.stride - 1) / g.stride : 0;
    const int q_lo = ww >= g.S - 1 ? (ww - (g.S - 1) + g.stride - 1) / g.stride : 0;
    // channels in groups of 8 (the C values of one tap are adjacent in a dcol row)
    for (int c0 = 0; c0 < g.C; c0 += 8) {
      const int cn = min(8, g.C - c0);
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int p = p_lo; p < g.P && p * g.stride <= hh; ++p) {
        const int r = hh - p * g.stride;
        const __nv_bfloat16* row = dcol + (static_cast<int64_t>(n) * g.P + p) * g.Q * g.ldcol;
        for (int q = q_lo; q < g.Q && q * g.stride <= ww; ++q) {
          const __nv_bfloat16* src = row + static_cast<int64_t>(q) * g.ldcol + (r * g.S + ww - q * g.stride) * g.C + c0;
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (e < cn) acc[e] += __bfloat162float(src[e]);
        }
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int c = c0 + e;
        if (e < cn)
          dx[((static_cast<int64_t>(n) * cb_n + c / g.b_c) * g.H + h) * g.W * g.b_c + static_cast<int64_t>(w) * g.b_c +
             c % g.b_c] = __float2bfloat16_rn(acc[e]);
      }
    }
  }
}

int small_geom(SmallGeom& g, int N, int C, int H, int W, int R, int S, int stride, int pad_h, int pad_w, int b_c,
               int64_t ldcol) {
  if (N <= 0 || C <= 0 || H <= 0 || W <= 0 || R <= 0 || S <= 0 || stride <= 0 || pad_h < 0 || pad_w < 0 ||
      b_c <= 0 || b_c > C)
    return set_error(BRK_ERR_CONTRACT, "conv im2col: bad geometry");
  g = SmallGeom{N, C, H, W, R, S, stride, pad_h, pad_w, b_c, (H + 2 * pad_h - R) / stride + 1,
                (W + 2 * pad_w - S) / stride + 1, ldcol};
  if (g.P <= 0 || g.Q <= 0) return set_error(BRK_ERR_CONTRACT, "conv im2col: empty output");
  if (ldcol % 8 || ldcol < static_cast<int64_t>(R) * S * C)
    return set_error(BRK_ERR_CONTRACT, "conv im2col: ldcol must be a multiple of 8 and >= R*S*C");
  return BRK_OK;
}

}  // namespace
}  // namespace brk

using namespace brk;

extern "C" {

BRK_API int brk_conv_im2col(const void* in, void* col, int N, int C, int H, int W, int R, int S, int stride,
                            int pad_h, int pad_w, int b_c, int64_t ldcol, void* stream) {
  SmallGeom g;
  int rc = small_geom(g, N, C, H, W, R, S, stride, pad_h, pad_w, b_c, ldcol);
  if (rc) return rc;
  const int groups = (R * S * C + 7) / 8;
  const int smem = ((groups * 8 * 8 + 15) / 16) * 16 + R * W * C * 2;
  if (smem > 200 * 1024) return set_error(BRK_ERR_CONTRACT, "conv im2col: R*W*C too large to stage");
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(im2col_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_cuda_error(e, "conv im2col smem");
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = std::min(N * g.P, 8 * sms);
  g_launches.fetch_add(1);
  im2col_kernel<<<grid, 256, smem, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(in), static_cast<__nv_bfloat16*>(col), g);
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? BRK_OK : set_cuda_error(err, "conv im2col");
}

BRK_API int brk_conv_col2im(const void* dcol, void* dx, int N, int C, int H, int W, int R, int S, int stride,
                            int pad_h, int pad_w, int b_c, int64_t ldcol, void* stream) {
  SmallGeom g;
  int rc = small_geom(g, N, C, H, W, R, S, stride, pad_h, pad_w, b_c, ldcol);
  if (rc) return rc;
  const dim3 grid((W + 127) / 128, std::min(N * H, 65535));
  g_launches.fetch_add(1);
  col2im_kernel<<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(dcol), static_cast<__nv_bfloat16*>(dx), g);
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? BRK_OK : set_cuda_error(err, "conv col2im");
}

}  // extern "C"
