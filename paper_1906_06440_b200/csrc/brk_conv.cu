// brk_conv.cu — direct convolution on the reference's blocked layouts
// (cnn.py:201-334; tensor.py:160-235) as implicit-GEMM launches of the tcgen05
// BRGEMM engine, each pass ONE launch whose per-tile batch list is the
// reference's (c_b, r, s) list (Alg. 4):
//
//   fwd : O [N][K_b][P][Q][64]  rows = output pixels, batch over (c_b, r, s)
//   bwd : dI[N][C_b][H][W][64]  "dual convolution": stride 1 is
//         a convolution of dO (padding R-1-pad) with the flipped, C<->K
//         swapped filter; 1x1 stride 2 scatters the 1x1 GEMM to the even input
//         positions and zero-fills the rest in the same epilogue
//   upd : dW[K_b][C_b][R][S][64 c][64 k] (fp32)  rows = (r, s, c), batch over
//         pixel chunks of 64, split across CTAs into fp32 slices that a
//         deterministic reduction sums in split order
//
// The activation side of every pass is fetched by TMA in im2col mode: the
// blocked tensor [N][X_b][H][W][64] is a 5-d map (64 ch, W, H, N, X_b) whose
// pixel walk (W, H, then N) is the GEMM row / reduction order; padding comes
// from the map's bounding box (zero fill), so no padded copy is materialised
// (the reference pads by copy, cnn.py:234-237).  Filter taps are im2col
// offsets; channel blocks are the outermost coordinate.  Weights are tiled
// 5-d maps (64 k, 64 c, RS, C_b, K_b); the backward pass reads them K-major
// at the flipped tap (no transposed copy).
//
// Engine path contract: bf16 storage, b_c = b_k = 64, C, K multiples of 64;
// stride 1 (any odd R = S with same padding) or 1x1 stride 2 (even H, W).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_bf16.h>

#include "brk_engine.h"
#include "brk_internal.h"
#include "brk_ptx.cuh"
#include "brk_tma_host.h"

namespace brk {

int launch_engine(const EngineParams& p, int bn, int tf32, int pair, int max_units, cudaStream_t stream);
int engine_sm_count();

namespace {

constexpr int kB = 64;

struct ConvGeom {
  int N, C, K, H, W, R, S, stride, pad_h, pad_w, P, Q;
};

int check_conv(const ConvGeom& g, int b_c, int b_k, int dtype, bool f32_ok = false) {
  char buf[256];
  if (dtype != BRK_BF16 && !(f32_ok && dtype == BRK_F32))
    return set_error(BRK_ERR_CONTRACT, f32_ok ? "conv engine path: bf16 or fp32 (TF32) storage"
                                              : "conv engine path: bf16 storage only");
  if (b_c != kB || b_k != kB) {
    std::snprintf(buf, sizeof(buf), "conv engine path needs b_c=b_k=64, got (%d,%d)", b_c, b_k);
    return set_error(BRK_ERR_CONTRACT, buf);
  }
  if (g.N <= 0 || g.C <= 0 || g.K <= 0 || g.C % kB || g.K % kB || g.H <= 0 || g.W <= 0 || g.R <= 0 ||
      g.S <= 0) {
    std::snprintf(buf, sizeof(buf), "conv engine path needs C, K multiples of 64 (C=%d K=%d)", g.C, g.K);
    return set_error(BRK_ERR_CONTRACT, buf);
  }
  if (g.P <= 0 || g.Q <= 0) return set_error(BRK_ERR_CONTRACT, "conv: empty output");
  if (g.stride != 1 && !(g.stride == 2 && g.R == 1 && g.S == 1 && g.pad_h == 0 && g.pad_w == 0))
    return set_error(BRK_ERR_CONTRACT, "conv engine path: stride 1, or 1x1 stride 2 without padding");
  if (g.pad_h > 15 || g.pad_w > 15 || g.R > 16 || g.S > 16)
    return set_error(BRK_ERR_CONTRACT, "conv engine path: filter / padding too large for im2col corners");
  if (static_cast<int64_t>(g.N) * g.H * g.W >= (int64_t(1) << 31))
    return set_error(BRK_ERR_CONTRACT, "conv engine path: N*H*W must fit int32");
  return BRK_OK;
}

struct ConvPlan {
  int pair, bn, splits;
  int64_t tiles;
};

// Tile choice for rows x cols outputs (rows need not divide the tile: the
// pixel walk is clamped and the epilogue masks).  Cost = max(MMA time, memory
// time).  MMA: per-SM tensor-pipe efficiency in SS mode (measured): CTA pair
// N=256 ~1, N=128 ~2/3; single CTA N=256 ~2/3, N=128 ~1/2, N=64 ~0.4.
// Memory: each operand is read once from HBM, and again once per tile along
// the other dimension (from L2 when it fits, else HBM); split-K slices are
// written and read back by the reduction.
ConvPlan choose(int64_t rows, int cols, int k_steps, bool split_ok, double a_bytes = 0, double b_bytes = 0,
                double out_bytes = 0, double slice_bytes = 0) {
  int forced_pair = -1, forced_bn = 0, forced_splits = 0;
  if (const char* env = std::getenv("BRK_CONV_TILE")) std::sscanf(env, "%d,%d", &forced_pair, &forced_bn);
  if (const char* env = std::getenv("BRK_CONV_SPLITS")) forced_splits = std::atoi(env);
  struct Opt { int pair, bn; double eff; };
  const Opt opts[] = {{1, 256, 1.0}, {1, 128, 0.67}, {0, 256, 0.67}, {0, 128, 0.5}, {0, 64, 0.4}};
  const int sms = engine_sm_count();
  constexpr double kHbm = 6.5e12, kL2 = 18e12, kL2Fit = 60e6;
  constexpr double kSmFlops = 8192.0 * 1.9e9;  // dense bf16 per SM per second
  ConvPlan best{0, 0, 1, 0};
  double best_cost = 0;
  for (const Opt& o : opts) {
    if (cols % o.bn) continue;
    if (forced_pair >= 0 && (o.pair != forced_pair || o.bn != forced_bn)) continue;
    const int tr = o.pair ? 256 : 128;
    const int64_t m_t = (rows + tr - 1) / tr, n_t = cols / o.bn;
    const int64_t tiles = m_t * n_t;
    const int64_t units = o.pair ? sms / 2 : sms;
    // one work unit (tile x k-steps) on one SM (pair: each SM does half the rows)
    const double unit_s = 128.0 * o.bn * 64 * 2 * k_steps / (kSmFlops * o.eff);
    const double reread = a_bytes * (n_t - 1) / (a_bytes < kL2Fit ? kL2 : kHbm) +
                          b_bytes * (m_t - 1) / (b_bytes < kL2Fit ? kL2 : kHbm);
    const double base_mem = (a_bytes + b_bytes + out_bytes) / kHbm;
    int max_split = 1;
    // (at most one wave of work units: a second wave of split units measured slower than
    // fewer, longer splits — each unit pays its pipeline fill and a partial-tile epilogue)
    if (split_ok) max_split = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(k_steps / 8, units / std::max<int64_t>(1, tiles))));
    if (forced_splits > 0) max_split = std::min(forced_splits, std::max(1, k_steps));
    for (int sp = forced_splits > 0 ? max_split : 1; sp <= max_split; ++sp) {
      const int64_t work = tiles * sp;
      const int64_t waves = (work + units - 1) / units;
      const double t_mma = waves * unit_s / sp;
      // weight updates (split_ok): the memory term over-penalised splits in measurement
      // (slices mostly stay in L2); they keep the MMA-time model
      const double t_mem = split_ok ? 0.0 : base_mem + reread;
      const double cost = std::max(t_mma, t_mem) + (sp > 1 ? 0.05 * unit_s : 0.0) + 2.0e-6;
      if (best.bn == 0 || cost < best_cost) {
        // every split must own >= 1 k-step: ceil(k / ceil(k / sp)) splits
        const int per = (k_steps + sp - 1) / sp;
        best = ConvPlan{o.pair, o.bn, (k_steps + per - 1) / per, tiles};
        best_cost = cost;
      }
    }
  }
  return best;
}

// 5-d im2col map over a blocked activation [N][X_b][Hh][Ww][64]:
// dims (64, Ww, Hh, N, X_b).  The filter window of output pixel (p, q) starts
// at (p*stride - pad_h, q*stride - pad_w); the last pixel's window ends at
// (P-1)*stride - pad + R-1, expressed as the bounding-box upper corner.
int im2col_map(CUtensorMap* map, const void* ptr, int N, int X, int Hh, int Ww, int R, int S, int stride,
               int pad_h, int pad_w, uint32_t pixels) {
  const uint64_t dims[5] = {kB, (uint64_t)Ww, (uint64_t)Hh, (uint64_t)N, (uint64_t)(X / kB)};
  const uint64_t hw = (uint64_t)Hh * Ww * kB;
  const uint64_t strides[5] = {1, kB, (uint64_t)Ww * kB, (uint64_t)(X / kB) * hw, hw};
  const int lower[3] = {-pad_w, -pad_h, 0};
  // 2 extra images of zero fill past N: a K-side pixel walk that runs off the
  // end reads zeros instead of wrapping into the next channel block.
  const int upper[3] = {pad_w - (S - 1), pad_h - (R - 1), 2};
  const uint32_t es[5] = {1, (uint32_t)stride, (uint32_t)stride, 1, 1};
  return encode_tmap_im2col(map, ptr, dims, strides, lower, upper, kB, pixels, es);
}

// fp32 activations for TF32 (same dims; boxes of 32 channels = one 128-byte row per pixel)
int im2col_map_f32(CUtensorMap* map, const void* ptr, int N, int X, int Hh, int Ww, int R, int S, int stride,
                   int pad_h, int pad_w, uint32_t pixels) {
  const uint64_t dims[5] = {kB, (uint64_t)Ww, (uint64_t)Hh, (uint64_t)N, (uint64_t)(X / kB)};
  const uint64_t hw = (uint64_t)Hh * Ww * kB;
  const uint64_t strides[5] = {1, kB, (uint64_t)Ww * kB, (uint64_t)(X / kB) * hw, hw};
  const int lower[3] = {-pad_w, -pad_h, 0};
  const int upper[3] = {pad_w - (S - 1), pad_h - (R - 1), 2};
  const uint32_t es[5] = {1, (uint32_t)stride, (uint32_t)stride, 1, 1};
  return encode_tmap_im2col(map, ptr, dims, strides, lower, upper, 32, pixels, es, /*f32=*/true);
}

// Weights [K_b][C_b][R][S][64 c][64 k]: dims (64 k, 64 c, RS, C_b, K_b)
int weight_map(CUtensorMap* map, const void* w, int C, int K, int RS, uint32_t box_cb, uint32_t box_kb) {
  const uint64_t dims[5] = {kB, kB, (uint64_t)RS, (uint64_t)(C / kB), (uint64_t)(K / kB)};
  const uint64_t strides[5] = {1, kB, kB * kB, (uint64_t)RS * kB * kB, (uint64_t)(C / kB) * RS * kB * kB};
  const uint32_t box[5] = {kB, kB, 1, box_cb, box_kb};
  return encode_tmap(map, w, true, 5, dims, strides, box);
}

void init_params(EngineParams& p) {
  std::memset(&p, 0, sizeof(p));
  p.ca.kdiv0 = p.cb.kdiv0 = 1 << 30;
  p.ca.kdiv1 = p.cb.kdiv1 = 1;
  p.alpha = 1.0f;
  p.om.rb2 = int64_t(0x7fffffff);
  const char* dbg = std::getenv("BRK_DEBUG_FLAGS");
  p.debug_flags = dbg ? std::atoi(dbg) : 0;
  p.debug_ts = g_debug_ts;
}

void pixel_walk(OperandCoords& oc, int kind, int P, int Q, int stride, int pad_h, int pad_w, int64_t total) {
  oc.kind = kind;
  oc.P = P;
  oc.Q = Q;
  oc.cstride = stride;
  oc.pad_h = pad_h;
  oc.pad_w = pad_w;
  oc.total_pix = static_cast<int32_t>(total);
  oc.ndims = 5;
}

// dW[i] = sum_s ws[s * n + i] in split order (deterministic), optional SGD on
// bf16 weights in the same layout.
__global__ void __launch_bounds__(256) split_reduce_kernel(const float4* __restrict__ ws, int splits, int64_t n4,
                                                           float4* __restrict__ dw, __nv_bfloat16* w_sgd, float lr) {
  pdl_launch_dependents();
  pdl_wait();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    // the slices' loads are issued eight at a time (independent), the adds stay in split order
    float4 a = __ldcs(ws + i);
    int s = 1;
    for (; s + 8 <= splits; s += 8) {
      float4 b[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = __ldcs(ws + (s + j) * n4 + i);
#pragma unroll
      for (int j = 0; j < 8; ++j) { a.x += b[j].x; a.y += b[j].y; a.z += b[j].z; a.w += b[j].w; }
    }
    for (; s < splits; ++s) {
      const float4 b = __ldcs(ws + s * n4 + i);
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    }
    dw[i] = a;
    if (w_sgd != nullptr) {
      __nv_bfloat162* w2 = reinterpret_cast<__nv_bfloat162*>(w_sgd) + 2 * i;
      const float2 w0 = __bfloat1622float2(w2[0]), w1 = __bfloat1622float2(w2[1]);
      w2[0] = __floats2bfloat162_rn(w0.x - lr * a.x, w0.y - lr * a.y);
      w2[1] = __floats2bfloat162_rn(w1.x - lr * a.z, w1.y - lr * a.w);
    }
  }
}

}  // namespace

// shared with brk_gemm.cu
int split_reduce(const float* ws, int splits, int64_t n, float* dw, void* w_sgd, float lr, cudaStream_t stream) {
  const int64_t n4 = n / 4;
  int blocks = static_cast<int>(std::min<int64_t>((n4 + 255) / 256, 4 * engine_sm_count()));
  if (blocks < 1) blocks = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  g_launches.fetch_add(1);
  cudaError_t err = cudaLaunchKernelEx(&cfg, split_reduce_kernel, reinterpret_cast<const float4*>(ws), splits, n4,
                                       reinterpret_cast<float4*>(dw), static_cast<__nv_bfloat16*>(w_sgd), lr);
  if (err != cudaSuccess) return set_cuda_error(err, "conv split reduce launch");
  return BRK_OK;
}

namespace {

ConvGeom geom(int N, int C, int K, int H, int W, int R, int S, int stride, int pad_h, int pad_w) {
  ConvGeom g{N, C, K, H, W, R, S, stride, pad_h, pad_w, 0, 0};
  if (stride > 0) {
    g.P = (H + 2 * pad_h - R) / stride + 1;
    g.Q = (W + 2 * pad_w - S) / stride + 1;
  }
  return g;
}

ConvPlan upd_plan(const ConvGeom& g) {
  const int64_t atoms = static_cast<int64_t>(g.C / kB) * g.R * g.S;
  const int64_t pix = static_cast<int64_t>(g.N) * g.P * g.Q;
  const int k_steps = static_cast<int>((pix + 63) / 64);
  const double in_b = 2.0 * g.N * g.C * g.H * g.W, out_b = 2.0 * g.N * g.K * g.P * g.Q;
  return choose(atoms * kB, g.K, k_steps, true, in_b, out_b, 0.0, 4.0 * g.C * g.K * g.R * g.S);
}

}  // namespace
}  // namespace brk

using namespace brk;

extern "C" {

BRK_API int brk_conv_fwd(const void* in, const void* w, const float* bias, void* out, int N, int C, int K, int H,
                         int W, int R, int S, int stride, int pad_h, int pad_w, int b_c, int b_k, int act, int dtype,
                         void* stream) {
  const ConvGeom g = geom(N, C, K, H, W, R, S, stride, pad_h, pad_w);
  int rc = check_conv(g, b_c, b_k, dtype, /*f32_ok=*/true);
  if (rc) return rc;
  if (act < kActNone || act > kActSigmoid) return set_error(BRK_ERR_CONTRACT, "unknown activation");
  const int64_t rows = static_cast<int64_t>(N) * g.P * g.Q;
  if (dtype == BRK_F32) {
    // TF32: k-steps of 32 channels, digits (channel half, s, r, c_b); A = fp32 im2col boxes of
    // 128 pixels x 32 channels (K-major), B = the weights' MN-major 32-element atoms (the
    // 32 B-chunk 128B swizzle), two per 64 output channels; one 64-channel K block per CTA row
    // block (CTA pairs of BN = 128, or single CTAs of BN = 64)
    const bool pair = K % 128 == 0;
    const int bn = pair ? 128 : 64;
    EngineParams p;
    init_params(p);
    if ((rc = im2col_map_f32(&p.map_a, in, N, C, H, W, R, S, stride, pad_h, pad_w, 128))) return rc;
    p.ca.kdiv0 = 2;
    p.ca.kdiv1 = S;
    p.ca.kdiv2 = R;
    p.ca.kc[0][0] = 32;  // channel half
    p.ca.kc[3][4] = 1;   // channel block c_b = d3
    p.ca.ok[0][1] = 1;   // w tap = s
    p.ca.ok[1][2] = 1;   // h tap = r
    p.ca.n_loads = 1;
    p.ca.load_bytes = 128 * 128;
    p.ca.mn_major = 0;
    pixel_walk(p.ca, 1, g.P, g.Q, stride, pad_h, pad_w, rows);
    {  // W[kb][c_b][rs][64 c][64 k] fp32 as (32 k_lo, 2 k_hi, 64 c, RS * C_b * K_b)
      const uint64_t dims[4] = {32, 2, kB, static_cast<uint64_t>(R) * S * (C / kB) * (K / kB)};
      const uint64_t strides[4] = {1, 32, kB, kB * kB};
      const uint32_t box[4] = {32, 1, 32, 1};
      if ((rc = encode_tmap(&p.map_b, w, false, 4, dims, strides, box, /*atom32=*/true))) return rc;
    }
    p.cb.kdiv0 = 2;
    p.cb.kdiv1 = S;
    p.cb.kdiv2 = R;
    p.cb.kc[0][2] = 32;               // c rows of the half
    p.cb.kc[1][3] = 1;                // s
    p.cb.kc[2][3] = S;                // r
    p.cb.kc[3][3] = R * S;            // c_b
    p.cb.rc[3] = R * S * (C / kB);    // k_b = the CTA's row block
    p.cb.lc[1] = 1;                   // load l = k_hi atom
    p.cb.n_loads = 2;
    p.cb.load_bytes = 32 * 128;
    p.cb.mn_major = 1;
    p.cb.ndims = 4;
    p.m_tiles = static_cast<int>((rows + (pair ? 255 : 127)) / (pair ? 256 : 128));
    p.n_tiles = K / bn;
    p.k_steps = 2 * (C / kB) * R * S;
    p.rows = static_cast<int>(rows);
    p.cols = K;
    p.out = out;
    p.out_bf16 = 0;
    const int64_t pq = static_cast<int64_t>(g.P) * g.Q;
    p.om = OutMap{pq, 0, kB, kB, pq * kB, 1, pq, (int64_t)(K / kB) * pq * kB};
    p.bias = bias;
    p.act = act;
    g_launches.fetch_add(1);
    return launch_engine(p, bn, 1, pair ? 1 : 0, 0, static_cast<cudaStream_t>(stream));
  }
  const int k_steps = (C / kB) * R * S;
  const ConvPlan pl = choose(rows, K, k_steps, false, 2.0 * N * C * H * W, 2.0 * K * C * R * S,
                             2.0 * N * K * g.P * g.Q);
  if (pl.bn == 0) return set_error(BRK_ERR_CONTRACT, "conv fwd: no engine tile fits K");
  const int brows = pl.pair ? pl.bn / 2 : pl.bn;
  EngineParams p;
  init_params(p);
  // A: input pixels (K-major rows of 64 channels), taps (s, r) as im2col offsets
  if ((rc = im2col_map(&p.map_a, in, N, C, H, W, R, S, stride, pad_h, pad_w, 128))) return rc;
  p.ca.kdiv0 = S;
  p.ca.kdiv1 = R;
  p.ca.kc[2][4] = 1;  // channel block c_b = d2
  p.ca.ok[0][0] = 1;  // w tap = s
  p.ca.ok[1][1] = 1;  // h tap = r
  p.ca.n_loads = 1;
  p.ca.load_bytes = 128 * 128;
  p.ca.mn_major = 0;
  pixel_walk(p.ca, 1, g.P, g.Q, stride, pad_h, pad_w, rows);
  // B: W[kb][c_b][r][s] (64 c x 64 k, k contiguous = MN-major), brows/64 K blocks
  if ((rc = weight_map(&p.map_b, w, C, K, R * S, 1, brows / kB))) return rc;
  p.cb.kdiv0 = S;
  p.cb.kdiv1 = R;
  p.cb.kc[0][2] = 1;
  p.cb.kc[1][2] = S;
  p.cb.kc[2][3] = 1;
  p.cb.rc[4] = brows / kB;
  p.cb.n_loads = 1;
  p.cb.load_bytes = brows * 128;
  p.cb.mn_major = 1;
  p.cb.ndims = 5;
  p.m_tiles = static_cast<int>((rows + (pl.pair ? 255 : 127)) / (pl.pair ? 256 : 128));
  p.n_tiles = K / pl.bn;
  p.k_steps = k_steps;
  p.rows = static_cast<int>(rows);
  p.cols = K;
  p.out = out;
  p.out_bf16 = 1;
  const int64_t pq = static_cast<int64_t>(g.P) * g.Q;
  p.om = OutMap{pq, 0, kB, kB, pq * kB, 1, pq, (int64_t)(K / kB) * pq * kB};
  p.bias = bias;
  p.act = act;
  g_launches.fetch_add(1);
  return launch_engine(p, pl.bn, 0, pl.pair, 0, static_cast<cudaStream_t>(stream));
}

BRK_API int brk_conv_bwd_data(const void* dout, const void* w, void* din, int N, int C, int K, int H, int W, int R,
                              int S, int stride, int pad_h, int pad_w, int b_c, int b_k, int dtype, void* stream) {
  const ConvGeom g = geom(N, C, K, H, W, R, S, stride, pad_h, pad_w);
  int rc = check_conv(g, b_c, b_k, dtype, /*f32_ok=*/true);
  if (rc) return rc;
  if (stride == 1 && (g.P != H || g.Q != W))
    return set_error(BRK_ERR_CONTRACT, "conv bwd engine path: stride 1 needs same padding");
  if (stride == 2 && (H != 2 * g.P || W != 2 * g.Q))
    return set_error(BRK_ERR_CONTRACT, "conv bwd engine path: 1x1 stride 2 needs even H, W");
  EngineParams p;
  init_params(p);
  if (dtype == BRK_F32) {
    // TF32: the dual convolution with k-steps of 32 output channels, digits (channel half, s',
    // r', k_b); A = fp32 im2col boxes of dO, B = the flipped weights read K-major (rows c, 32
    // contiguous k = one 128-byte row), one 64-channel C block per CTA row block.  1x1 stride 2:
    // rows are output pixels scattered to (2p, 2q), the other input pixels zeroed first.
    const bool pair = C % 128 == 0;
    const int bn = pair ? 128 : 64;
    const int64_t rows = stride == 1 ? static_cast<int64_t>(N) * H * W : static_cast<int64_t>(N) * g.P * g.Q;
    const int dph = stride == 1 ? R - 1 - pad_h : 0, dpw = stride == 1 ? S - 1 - pad_w : 0;
    if ((rc = im2col_map_f32(&p.map_a, dout, N, K, g.P, g.Q, R, S, 1, dph, dpw, 128))) return rc;
    p.ca.kdiv0 = 2;
    p.ca.kdiv1 = S;
    p.ca.kdiv2 = R;
    p.ca.kc[0][0] = 32;  // channel half
    p.ca.kc[3][4] = 1;   // output-channel block k_b = d3
    p.ca.ok[0][1] = 1;   // w tap = s'
    p.ca.ok[1][2] = 1;   // h tap = r'
    p.ca.n_loads = 1;
    p.ca.load_bytes = 128 * 128;
    p.ca.mn_major = 0;
    if (stride == 1) pixel_walk(p.ca, 1, H, W, 1, dph, dpw, rows);
    else pixel_walk(p.ca, 1, g.P, g.Q, 1, 0, 0, rows);
    {  // W[kb][c_b][rs][64 c][64 k] fp32 as (32 k_lo, 2 k_hi, 64 c, RS * C_b * K_b)
      const uint64_t dims[4] = {32, 2, kB, static_cast<uint64_t>(R) * S * (C / kB) * (K / kB)};
      const uint64_t strides[4] = {1, 32, kB, kB * kB};
      const uint32_t box[4] = {32, 1, kB, 1};
      if ((rc = encode_tmap(&p.map_b, w, false, 4, dims, strides, box))) return rc;
    }
    p.cb.kdiv0 = 2;
    p.cb.kdiv1 = S;
    p.cb.kdiv2 = R;
    p.cb.kc[0][1] = 1;                 // k_hi = the channel half
    p.cb.base[3] = R * S - 1;          // flipped tap (R-1-r')*S + (S-1-s')
    p.cb.kc[1][3] = -1;
    p.cb.kc[2][3] = -S;
    p.cb.rc[3] = R * S;                // c_b = the CTA's row block
    p.cb.kc[3][3] = R * S * (C / kB);  // k_b
    p.cb.n_loads = 1;
    p.cb.load_bytes = kB * 128;
    p.cb.mn_major = 0;
    p.cb.ndims = 4;
    p.m_tiles = static_cast<int>((rows + (pair ? 255 : 127)) / (pair ? 256 : 128));
    p.n_tiles = C / bn;
    p.k_steps = 2 * (K / kB) * R * S;
    p.rows = static_cast<int>(rows);
    p.cols = C;
    p.out = din;
    p.out_bf16 = 0;
    const int64_t hw = static_cast<int64_t>(H) * W;
    if (stride == 1) {
      p.om = OutMap{hw, 0, kB, kB, hw * kB, 1, hw, (int64_t)(C / kB) * hw * kB};
    } else {
      const int64_t pq = static_cast<int64_t>(g.P) * g.Q;
      p.om = OutMap{g.Q, 2 * (int64_t)W * kB, 2 * kB, kB, hw * kB, 1, pq, (int64_t)(C / kB) * hw * kB};
      const cudaError_t err =
          cudaMemsetAsync(din, 0, static_cast<size_t>(N) * C * H * W * sizeof(float), static_cast<cudaStream_t>(stream));
      if (err != cudaSuccess) return set_cuda_error(err, "conv bwd: zeroing dX");
    }
    g_launches.fetch_add(1);
    return launch_engine(p, bn, 1, pair ? 1 : 0, 0, static_cast<cudaStream_t>(stream));
  }
  // rows: input pixels (stride 1) or output pixels scattered to (2p, 2q) (stride 2)
  const int64_t rows = stride == 1 ? static_cast<int64_t>(N) * H * W : static_cast<int64_t>(N) * g.P * g.Q;
  const int k_steps = (K / kB) * R * S;
  const ConvPlan pl = choose(rows, C, k_steps, false, 2.0 * N * K * g.P * g.Q, 2.0 * K * C * R * S,
                             2.0 * N * C * H * W);
  if (pl.bn == 0) return set_error(BRK_ERR_CONTRACT, "conv bwd: no engine tile fits C");
  const int brows = pl.pair ? pl.bn / 2 : pl.bn;
  // A: dO pixels; the dual convolution pads by R-1-pad and walks taps (s', r')
  const int dph = stride == 1 ? R - 1 - pad_h : 0, dpw = stride == 1 ? S - 1 - pad_w : 0;
  if ((rc = im2col_map(&p.map_a, dout, N, K, g.P, g.Q, R, S, 1, dph, dpw, 128))) return rc;
  p.ca.kdiv0 = S;
  p.ca.kdiv1 = R;
  p.ca.kc[2][4] = 1;  // output-channel block k_b = d2
  p.ca.ok[0][0] = 1;
  p.ca.ok[1][1] = 1;
  p.ca.n_loads = 1;
  p.ca.load_bytes = 128 * 128;
  p.ca.mn_major = 0;
  if (stride == 1) pixel_walk(p.ca, 1, H, W, 1, dph, dpw, rows);
  else pixel_walk(p.ca, 1, g.P, g.Q, 1, 0, 0, rows);
  // B: W[kb][cb][R-1-r'][S-1-s'] read K-major (rows c, 64 k contiguous)
  if ((rc = weight_map(&p.map_b, w, C, K, R * S, brows / kB, 1))) return rc;
  p.cb.kdiv0 = S;
  p.cb.kdiv1 = R;
  p.cb.base[2] = R * S - 1;
  p.cb.kc[0][2] = -1;
  p.cb.kc[1][2] = -S;
  p.cb.kc[2][4] = 1;
  p.cb.rc[3] = brows / kB;
  p.cb.n_loads = 1;
  p.cb.load_bytes = brows * 128;
  p.cb.mn_major = 0;
  p.cb.ndims = 5;
  p.m_tiles = static_cast<int>((rows + (pl.pair ? 255 : 127)) / (pl.pair ? 256 : 128));
  p.n_tiles = C / pl.bn;
  p.k_steps = k_steps;
  p.rows = static_cast<int>(rows);
  p.cols = C;
  p.out = din;
  p.out_bf16 = 1;
  const int64_t hw = static_cast<int64_t>(H) * W;
  if (stride == 1) {
    p.om = OutMap{hw, 0, kB, kB, hw * kB, 1, hw, (int64_t)(C / kB) * hw * kB};
  } else {
    const int64_t pq = static_cast<int64_t>(g.P) * g.Q;
    p.om = OutMap{g.Q, 2 * (int64_t)W * kB, 2 * kB, kB, hw * kB, 1, pq, (int64_t)(C / kB) * hw * kB};
    p.zf_w = kB;
    p.zf_h = static_cast<int64_t>(W) * kB;
  }
  g_launches.fetch_add(1);
  return launch_engine(p, pl.bn, 0, pl.pair, 0, static_cast<cudaStream_t>(stream));
}

BRK_API size_t brk_conv_upd_workspace(int N, int C, int K, int H, int W, int R, int S, int stride, int pad_h,
                                      int pad_w) {
  const ConvGeom g = geom(N, C, K, H, W, R, S, stride, pad_h, pad_w);
  if (check_conv(g, kB, kB, BRK_BF16)) return 0;
  const ConvPlan pl = upd_plan(g);
  if (pl.splits <= 1) return 0;
  return static_cast<size_t>(pl.splits) * C * K * R * S * sizeof(float);
}

BRK_API int brk_conv_upd(const void* in, const void* dout, float* dw, void* w_sgd, float lr, void* workspace,
                         size_t ws_bytes, int N, int C, int K, int H, int W, int R, int S, int stride, int pad_h,
                         int pad_w, int b_c, int b_k, int dtype, void* stream) {
  const ConvGeom g = geom(N, C, K, H, W, R, S, stride, pad_h, pad_w);
  int rc = check_conv(g, b_c, b_k, dtype, /*f32_ok=*/true);
  if (rc) return rc;
  ConvPlan pl = upd_plan(g);
  if (pl.bn == 0) return set_error(BRK_ERR_CONTRACT, "conv upd: no engine tile fits K");
  const int64_t dw_elems = static_cast<int64_t>(C) * K * R * S;
  if (pl.splits > 1 && (workspace == nullptr || ws_bytes < static_cast<size_t>(pl.splits) * dw_elems * 4))
    return set_error(BRK_ERR_CONTRACT, "conv upd: workspace too small (see brk_conv_upd_workspace)");
  const int brows = pl.pair ? pl.bn / 2 : pl.bn;
  const int64_t pix = static_cast<int64_t>(N) * g.P * g.Q;
  const int64_t atoms = static_cast<int64_t>(C / kB) * R * S;
  EngineParams p;
  init_params(p);
  if (dtype == BRK_F32) {
    // TF32, tile mode: a k-step is a block of 32 output pixels (bw x bh, bw >= Q when Q <= 32,
    // else row pieces of 32) of one image; A = 32-channel atoms of the input block shifted by each
    // atom's tap (padding and slots past Q / P read as out-of-bounds zeros; the latter meet dO
    // zeros) — for 1x1 stride 2 every other input pixel (TMA traversal strides of 2), B = dO's
    // block as two 32-channel atoms of the CTA's 64 output channels; both MN-major TF32 atoms
    // (32 B-chunk swizzle).  CTA pairs of BN = 128 or single CTAs of BN = 64.
    if (w_sgd != nullptr) return set_error(BRK_ERR_CONTRACT, "conv upd: fused SGD needs bf16 weights");
    const bool pair = K % 128 == 0;
    const int bn = pair ? 128 : 64;
    int bw = 1;
    while (bw < g.Q && bw < 32) bw *= 2;
    const int bh = 32 / bw, qb = (g.Q + bw - 1) / bw, pg = (g.P + bh - 1) / bh;
    auto map4 = [&](CUtensorMap* m, const void* ptr, int X, int hh, int ww, uint32_t st) {
      const uint64_t dims[4] = {kB, static_cast<uint64_t>(ww), static_cast<uint64_t>(hh),
                                static_cast<uint64_t>(N) * (X / kB)};
      const uint64_t strides[4] = {1, kB, static_cast<uint64_t>(ww) * kB, static_cast<uint64_t>(hh) * ww * kB};
      const uint32_t box[4] = {32, static_cast<uint32_t>(bw) * st, static_cast<uint32_t>(bh) * st, 1};
      const uint32_t es[4] = {1, st, st, 1};
      return encode_tmap(m, ptr, false, 4, dims, strides, box, /*atom32=*/true, es);
    };
    if ((rc = map4(&p.map_a, in, C, H, W, static_cast<uint32_t>(stride))) ||
        (rc = map4(&p.map_b, dout, K, g.P, g.Q, 1)))
      return rc;
    for (OperandCoords* oc : {&p.ca, &p.cb}) {  // k-step s = ((n * pg + row group) * qb + column block)
      oc->kdiv0 = qb;
      oc->kdiv1 = pg;
      oc->kc[0][1] = bw;
      oc->kc[1][2] = bh;
      oc->load_bytes = 32 * 128;
      oc->mn_major = 1;
      oc->ndims = 4;
    }
    p.ca.base[1] = -pad_w;
    p.ca.base[2] = -pad_h;
    p.ca.kc[0][1] = bw * stride;
    p.ca.kc[1][2] = bh * stride;
    p.ca.kc[2][3] = C / kB;
    p.ca.n_loads = 4;
    p.ca.atom_cb = C / kB;
    p.ca.atom_s = S;
    p.ca.kind = 5;
    p.cb.kc[2][3] = K / kB;
    p.cb.rc[3] = 1;   // k_b = the CTA's row block
    p.cb.lc[0] = 32;  // load l = channel half
    p.cb.n_loads = 2;
    p.k_steps = N * pg * qb;
    if (pl.splits > 1) {  // the workspace holds upd_plan's splits; re-plan them for these k-steps
      const int per = (p.k_steps + pl.splits - 1) / pl.splits;
      pl.splits = (p.k_steps + per - 1) / per;
    }
    p.m_tiles = static_cast<int>((atoms * kB + (pair ? 255 : 127)) / (pair ? 256 : 128));
    p.n_tiles = K / bn;
    p.rows = static_cast<int>(atoms * kB);
    p.cols = K;
    p.out_bf16 = 0;
    const int64_t rs_n = static_cast<int64_t>(R) * S;
    p.om = OutMap{kB, rs_n * kB * kB, kB, kB, (int64_t)(C / kB) * rs_n * kB * kB, 1, (int64_t)(C / kB) * kB,
                  kB * kB};
    if (pl.splits > 1) {
      p.k_splits = pl.splits;
      p.split_slice = dw_elems;
      p.out = workspace;
    } else {
      p.out = dw;
    }
    g_launches.fetch_add(1);
    rc = launch_engine(p, bn, 1, pair ? 1 : 0, 0, static_cast<cudaStream_t>(stream));
    if (rc || pl.splits <= 1) return rc;
    return split_reduce(static_cast<const float*>(workspace), pl.splits, dw_elems, dw, nullptr, 0.0f,
                        static_cast<cudaStream_t>(stream));
  }
  // 1x1 stride-1 convolutions: tile-mode boxes of 64 pixels x 64 channels per image (k-steps
  // aligned to images, the tail of an image's last box zero-filled out of bounds) instead of the
  // im2col pixel walk: im2col-mode boxes streamed at ~28 B/clk per SM (tools/probes/
  // engine_waits.py), tile-mode boxes at the ~70 B/clk chip limit (brk_diag_tma_lanes)
  static const char* tile_env = std::getenv("BRK_CONV_UPD_TILE");
  const bool tile_upd = R == 1 && S == 1 && stride == 1 && pad_h == 0 && pad_w == 0 &&
                        !(tile_env != nullptr && std::atoi(tile_env) == 0);
  if (tile_upd) {
    const int64_t hw = static_cast<int64_t>(H) * W;
    const int kpi = static_cast<int>((hw + 63) / 64);  // k-steps per image
    auto map3 = [&](CUtensorMap* m, const void* ptr, int X) {
      const uint64_t dims[3] = {kB, static_cast<uint64_t>(hw), static_cast<uint64_t>(N) * (X / kB)};
      const uint64_t strides[3] = {1, kB, static_cast<uint64_t>(hw) * kB};
      const uint32_t box[3] = {kB, 64, 1};
      return encode_tmap(m, ptr, true, 3, dims, strides, box);
    };
    if ((rc = map3(&p.map_a, in, C)) || (rc = map3(&p.map_b, dout, K))) return rc;
    // k-step s = (image n = s / kpi, pixel block j = s % kpi): coordinate (0, 64 j, n * X_b + block)
    for (OperandCoords* oc : {&p.ca, &p.cb}) {
      oc->kdiv0 = kpi;
      oc->kdiv1 = 1 << 30;
      oc->kc[0][1] = 64;
      oc->lc[2] = 1;
      oc->load_bytes = 64 * 128;
      oc->mn_major = 1;
      oc->ndims = 3;
      oc->kind = 0;
    }
    p.ca.kc[1][2] = C / kB;
    p.ca.rc[2] = 2;  // the CTA's 128 rows: 2 channel blocks (1 when C = 64: rows 64.. are masked)
    p.ca.n_loads = std::min(2, C / kB);
    p.cb.kc[1][2] = K / kB;
    p.cb.rc[2] = brows / kB;
    p.cb.n_loads = brows / kB;
    p.k_steps = N * kpi;
    if (pl.splits > 1) {  // re-plan the split count for the image-aligned k-steps
      const int per = (p.k_steps + pl.splits - 1) / pl.splits;
      pl.splits = (p.k_steps + per - 1) / per;
    }
  } else {
  // A: input pixels (K side, 64 per step) as 2 MN-major atoms (c_b, rs) of 64 channels
  if ((rc = im2col_map(&p.map_a, in, N, C, H, W, R, S, stride, pad_h, pad_w, 64))) return rc;
  p.ca.n_loads = 2;
  p.ca.load_bytes = 64 * 128;
  p.ca.mn_major = 1;
  p.ca.atom_cb = C / kB;
  p.ca.atom_s = S;
  pixel_walk(p.ca, 2, g.P, g.Q, stride, pad_h, pad_w, pix);
  // B: dO pixels (K side) as brows/64 MN-major atoms of 64 output channels
  if ((rc = im2col_map(&p.map_b, dout, N, K, g.P, g.Q, 1, 1, 1, 0, 0, 64))) return rc;
  p.cb.rc[4] = brows / kB;
  p.cb.lc[4] = 1;
  p.cb.n_loads = brows / kB;
  p.cb.load_bytes = 64 * 128;
  p.cb.mn_major = 1;
  pixel_walk(p.cb, 3, g.P, g.Q, 1, 0, 0, pix);
  p.k_steps = static_cast<int>((pix + 63) / 64);
  }
  p.m_tiles = static_cast<int>((atoms * kB + (pl.pair ? 255 : 127)) / (pl.pair ? 256 : 128));
  p.n_tiles = K / pl.bn;
  p.rows = static_cast<int>(atoms * kB);
  p.cols = K;
  p.out_bf16 = 0;
  // row = (rs * C_b + c_b) * 64 + c  ->  ((kb*C_b + c_b)*RS + rs)*4096 + c*64 + k
  const int64_t rs_n = static_cast<int64_t>(R) * S;
  p.om = OutMap{kB, rs_n * kB * kB, kB, kB, (int64_t)(C / kB) * rs_n * kB * kB, 1, (int64_t)(C / kB) * kB,
                kB * kB};
  if (pl.splits > 1) {
    p.k_splits = pl.splits;
    p.split_slice = dw_elems;
    p.out = workspace;
  } else {
    p.out = dw;
    p.sgd_w = w_sgd;
    p.sgd_lr = lr;
  }
  g_launches.fetch_add(1);
  rc = launch_engine(p, pl.bn, 0, pl.pair, 0, static_cast<cudaStream_t>(stream));
  if (rc || pl.splits <= 1) return rc;
  return split_reduce(static_cast<const float*>(workspace), pl.splits, dw_elems, dw, w_sgd, lr,
                             static_cast<cudaStream_t>(stream));
}

// Diagnostic: the engine plan the conv passes would use ("pair,bn,splits").
BRK_API int brk_conv_plan(int pass, int N, int C, int K, int H, int W, int R, int S, int stride, int pad_h,
                          int pad_w, int* out3) {
  const ConvGeom g = geom(N, C, K, H, W, R, S, stride, pad_h, pad_w);
  int rc = check_conv(g, kB, kB, BRK_BF16);
  if (rc) return rc;
  ConvPlan pl;
  if (pass == 0)
    pl = choose(static_cast<int64_t>(N) * g.P * g.Q, K, (C / kB) * R * S, false, 2.0 * N * C * H * W,
                2.0 * K * C * R * S, 2.0 * N * K * g.P * g.Q);
  else if (pass == 1)
    pl = choose(stride == 1 ? static_cast<int64_t>(N) * H * W : static_cast<int64_t>(N) * g.P * g.Q, C,
                (K / kB) * R * S, false, 2.0 * N * K * g.P * g.Q, 2.0 * K * C * R * S, 2.0 * N * C * H * W);
  else pl = upd_plan(g);
  out3[0] = pl.pair;
  out3[1] = pl.bn;
  out3[2] = pl.splits;
  return BRK_OK;
}

}  // extern "C"
