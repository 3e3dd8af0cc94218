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
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_bf16.h>

#include "brk_engine.h"
#include "brk_mlp.h"
#include "brk_internal.h"
#include "brk_ptx.cuh"
#include "brk_tma_host.h"

namespace brk {

int launch_engine(const EngineParams& p, int bn, int tf32, int pair, int max_units, cudaStream_t stream);
int engine_sm_count();
size_t engine_split_ws_bytes(int tiles, int splits, int bn, int pair);
unsigned long long* g_debug_ts = nullptr;  // set by brk_diag_set_timestamps (diagnostics build stamps)

namespace {

constexpr int kB = 64;  // block factor served by the TMA path (bf16)

struct Plan {
  int pair;    // 1: CTA pair, 256-row tiles
  int bn;      // tile columns
  int splits;  // split-K factor (1 = none)
  int tiles;
};

// Pick (pair, BN, split-K) for a rows x cols output with k_steps batch
// entries: minimise waves x per-work-unit time.  Per-SM tensor-pipe
// efficiency in SS mode (measured): 1-CTA N=128 ~1/2, N=256 ~2/3, CTA pair
// N=128 ~2/3 (L2-fed), N=256 ~1.  Split-K only when tiles cannot fill the
// machine; each chunk keeps >= 4 k-steps.
// Grouped (whole-step) launches build every problem with one tile shape and
// collect the parameter blocks instead of launching them.
thread_local const Plan* g_force_plan = nullptr;
thread_local EngineParams* g_capture = nullptr;

Plan choose_plan(int rows, int cols, int k_steps, bool allow_split) {
  if (g_force_plan != nullptr) {
    Plan f = *g_force_plan;
    f.tiles = (rows / (f.pair ? 256 : 128)) * (cols / f.bn);
    return f;
  }
  Plan forced{-1, 0, 0, 0};
  if (const char* env = std::getenv("BRK_TILE")) {  // "pair,bn" e.g. "1,256"
    int a = 0, b = 0;
    if (std::sscanf(env, "%d,%d", &a, &b) == 2) forced = Plan{a, b, 0, 0};
  }
  int forced_splits = 0;
  if (const char* env = std::getenv("BRK_SPLITS")) forced_splits = std::atoi(env);
  // Split-K is opt-in: measured slower than the unsplit tile for the MLP shapes
  // (profiles/r01_engine_notes.md); kept for deep-K / few-tile problems.
  if (forced_splits <= 0) allow_split = false;
  const int sms = engine_sm_count();
  struct Opt { int pair, bn; double eff; };
  const Opt opts[] = {{1, 256, 1.0}, {1, 128, 0.67}, {0, 256, 0.67}, {0, 128, 0.5}, {0, 64, 0.33}};
  Plan best{0, 0, 1, 0};
  double best_cost = 0;
  for (const Opt& o : opts) {
    const int tile_rows = o.pair ? 256 : 128;
    if (rows % tile_rows || cols % o.bn) continue;
    if (forced.pair >= 0 && (forced.pair != o.pair || forced.bn != o.bn)) continue;
    const long tiles = static_cast<long>(rows / tile_rows) * (cols / o.bn);
    const long units = o.pair ? sms / 2 : sms;
    const double per_tile = static_cast<double>(tile_rows) * o.bn * k_steps / ((o.pair ? 2.0 : 1.0) * o.eff);
    int max_split = allow_split ? (int)std::max(1L, std::min<long>(k_steps / 4, units / std::max(1L, tiles))) : 1;
    if (forced_splits > 0) max_split = allow_split ? std::min(forced_splits, k_steps) : 1;
    for (int sp = (forced_splits > 0 ? max_split : 1); sp <= max_split; ++sp) {
      const long work = tiles * sp;
      const long waves = (work + units - 1) / units;
      const double cost = waves * per_tile / sp * (sp > 1 ? 1.1 : 1.0) + 2.0e5;  // + fixed launch cost
      if (best.bn == 0 || cost < best_cost) {
        const int per = (k_steps + sp - 1) / sp;
        best = Plan{o.pair, o.bn, (k_steps + per - 1) / per, static_cast<int>(tiles)};
        best_cost = cost;
      }
    }
  }
  return best;
}

// Blocked 2-D activation [Rb][Xb][64][64] (row-major blocks, x innermost):
// X (rows n, x = c), dZ/Y (rows n, x = k).  dims (x_in, r_in, xb, rb)
struct Map4 {
  uint64_t dims[4];
  uint64_t strides[4];
};
Map4 act_layout(int64_t rows, int64_t xs) {
  Map4 a;
  a.dims[0] = kB; a.dims[1] = kB; a.dims[2] = xs / kB; a.dims[3] = rows / kB;
  a.strides[0] = 1; a.strides[1] = kB; a.strides[2] = kB * kB; a.strides[3] = (xs / kB) * kB * kB;
  return a;
}
// Weights [Kb][Cb][64 c][64 k] (k innermost): dims (k_in, c_in, cb, kb)
Map4 w_layout(int64_t K, int64_t C) {
  Map4 a;
  a.dims[0] = kB; a.dims[1] = kB; a.dims[2] = C / kB; a.dims[3] = K / kB;
  a.strides[0] = 1; a.strides[1] = kB; a.strides[2] = kB * kB; a.strides[3] = (C / kB) * kB * kB;
  return a;
}

void set_coords(OperandCoords& oc, std::initializer_list<int> rc, std::initializer_list<int> kq,
                uint32_t load_bytes, int mn_major) {
  std::memset(&oc, 0, sizeof(oc));
  int d = 0;
  for (int v : rc) oc.rc[d++] = v;
  d = 0;
  for (int v : kq) oc.kc[0][d++] = v;
  oc.kdiv0 = 1 << 30;
  oc.kdiv1 = 1;
  oc.n_loads = 1;
  oc.load_bytes = load_bytes;
  oc.mn_major = mn_major;
  oc.ndims = 4;
}

// fp32 storage (TF32 tensor cores): a 64-wide block row is 256 B, two 128 B swizzle
// atoms.  The maps view every blocked tensor with the 64-wide inner dimension split
// into (32 elements, half) — the half as its own dimension with a 32-element
// stride — so one TMA box is one 32-wide (128 B) atom column, a k-step covers 32
// elements of the reduction (k-step s: half s % 2, block s / 2) and an MN-major
// box lists its 32 x 32 atoms in MN order.  Dims: (x32, r_in, xhalf, xb, rb) for
// [Rb][Xb][64 r][64 x] (x innermost), strides (1, 64, 32, 4096, Xb*4096).
struct Map5 {
  uint64_t dims[5];
  uint64_t strides[5];
};
Map5 split_layout(int64_t rows, int64_t xs) {
  Map5 a;
  a.dims[0] = 32; a.dims[1] = kB; a.dims[2] = 2; a.dims[3] = xs / kB; a.dims[4] = rows / kB;
  a.strides[0] = 1; a.strides[1] = kB; a.strides[2] = 32; a.strides[3] = kB * kB; a.strides[4] = (xs / kB) * kB * kB;
  return a;
}
// mn_major: the 32 B-chunk swizzle UMMA reads MN-major TF32 operands in
int enc5(CUtensorMap* map, const void* ptr, const Map5& l, std::initializer_list<uint32_t> box,
         bool mn_major = false) {
  uint32_t b[5];
  int d = 0;
  for (uint32_t v : box) b[d++] = v;
  return encode_tmap(map, ptr, false, 5, l.dims, l.strides, b, mn_major);
}
// f32 coordinates: rowblk advances dim rdim by rstep; k-step s: dim hdim += hstep * (s % 2),
// dim bdim += s / 2
void set_coords_f32(OperandCoords& oc, int rdim, int rstep, int hdim, int hstep, int bdim, uint32_t load_bytes,
                    int n_loads, int mn_major) {
  std::memset(&oc, 0, sizeof(oc));
  oc.rc[rdim] = rstep;
  oc.kc[0][hdim] = hstep;
  oc.kc[1][bdim] = 1;
  oc.kdiv0 = 2;
  oc.kdiv1 = 1 << 30;
  oc.n_loads = n_loads;
  oc.load_bytes = load_bytes;
  oc.mn_major = mn_major;
  oc.ndims = 5;
}

int check_fc(int N, int C, int K, int b_n, int b_c, int b_k, int dtype) {
  char buf[256];
  if (dtype != BRK_BF16 && dtype != BRK_F32)
    return set_error(BRK_ERR_CONTRACT, "fc engine path: bf16 (kind::f16) or fp32 (kind::tf32) storage");
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

int enc(CUtensorMap* map, const void* ptr, const Map4& l, uint32_t b0, uint32_t b1, uint32_t b2,
        uint32_t b3) {
  const uint32_t box[4] = {b0, b1, b2, b3};
  return encode_tmap(map, ptr, true, 4, l.dims, l.strides, box);
}

int debug_flags() {
  const char* dbg = std::getenv("BRK_DEBUG_FLAGS");
  return dbg ? std::atoi(dbg) : 0;
}


int finish(const EngineParams& p, const Plan& pl, void* stream, int tf32 = 0) {
  if (g_capture != nullptr) {
    *g_capture = p;
    return BRK_OK;
  }
  g_launches.fetch_add(1);
  return launch_engine(p, pl.bn, tf32, pl.pair, 0, static_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------------------
// dZ = dY * (Y > 0) (optional) and db[k] = sum_n dZ[n][k]  — deterministic:
// grid (K/64, kSplit); CTA (kb, s) sums rows of split s for 64 columns, then
// the last CTA of column block kb adds the kSplit partials in a fixed order.
// ---------------------------------------------------------------------------
constexpr int kSplit = 16;

// 8 consecutive elements of a bf16 or fp32 row segment, as floats
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float* v) {
  const uint4 g = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&g);
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = __bfloat162float(h[j]);
}
__device__ __forceinline__ void load8(const float* p, float* v) {
  const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float* v) {
  uint4 g;
  __nv_bfloat16* h = reinterpret_cast<__nv_bfloat16*>(&g);
#pragma unroll
  for (int j = 0; j < 8; ++j) h[j] = __float2bfloat16_rn(v[j]);  // exact: v[j] is a bf16 value or 0
  *reinterpret_cast<uint4*>(p) = g;
}
__device__ __forceinline__ void store8(float* p, const float* v) {
  reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}

template <typename T>
__global__ void __launch_bounds__(256) bias_grad_kernel(const T* dy, const T* __restrict__ y, T* dz_out,
                                                        float* __restrict__ db, float* __restrict__ partial,
                                                        unsigned* __restrict__ counters, int N, int K,
                                                        float* __restrict__ bias, float lr) {
  pdl_launch_dependents();
  pdl_wait();
  const int kb = blockIdx.x, split = blockIdx.y;
  const int Kb = K / kB;
  const int tid = threadIdx.x;
  const int cgrp = tid & 7;    // 8 column groups of 8
  const int rlane = tid >> 3;  // 32 row lanes
  const int rows_per = N / kSplit;
  const int r0 = split * rows_per;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int r = r0 + rlane; r < r0 + rows_per; r += 32) {
    const int64_t off = static_cast<int64_t>(r / kB) * Kb * kB * kB + static_cast<int64_t>(kb) * kB * kB +
                        (r % kB) * kB + cgrp * 8;
    float g[8];
    load8(dy + off, g);
    if (y != nullptr) {
      float m[8];
      load8(y + off, m);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (!(m[j] > 0.0f)) g[j] = 0.0f;
      if (dz_out != nullptr) store8(dz_out + off, g);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += g[j];
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
  const bool f32 = dtype == BRK_F32;
  const Plan pl = choose_plan(N, K, C / kB, false);
  const int brows = pl.pair ? pl.bn / 2 : pl.bn;
  if (!f32) {
    // A = X (rows n, red c) K-major: box (c 64, n 64, cb 1, nb 2) = 128 rows
    if ((rc = enc(&p.map_a, x, act_layout(N, C), 64, 64, 1, 2))) return rc;
    set_coords(p.ca, {0, 0, 0, 2}, {0, 0, 1, 0}, 128 * 128, 0);
    // B = W (rows k, red c) MN-major: box (k 64, c 64, cb 1, kb brows/64)
    if ((rc = enc(&p.map_b, w, w_layout(K, C), 64, 64, 1, brows / 64))) return rc;
    set_coords(p.cb, {0, 0, 0, brows / 64}, {0, 0, 1, 0}, brows * 128, 1);
  } else {
    // A = X K-major: box (c 32, n 64, half 1, cb 1, nb 2) = 128 rows x 128 B
    if ((rc = enc5(&p.map_a, x, split_layout(N, C), {32, 64, 1, 1, 2}))) return rc;
    set_coords_f32(p.ca, 4, 2, 2, 1, 3, 128 * 128, 1, 0);
    // B = W MN-major (x = k, r = c): box (k 32, c 32, khalf 2, cb 1, kb brows/64): brows/32 atoms
    if ((rc = enc5(&p.map_b, w, split_layout(K, C), {32, 32, 2, 1, (uint32_t)(brows / 64)}, true))) return rc;
    // (W's blocked layout [Kb][Cb][64 c][64 k] is split_layout(rows = K, xs = C) with the roles
    //  of its inner dims read as (k32, c_in, khalf, cb, kb): strides (1, 64, 32, 4096, Cb*4096))
    set_coords_f32(p.cb, 4, brows / 64, 1, 32, 3, brows * 128, 1, 1);
  }
  p.m_tiles = N / (pl.pair ? 256 : 128);
  p.n_tiles = K / pl.bn;
  p.k_steps = f32 ? C / 32 : C / kB;
  p.rows = N;
  p.cols = K;
  p.out = y;
  p.out_bf16 = f32 ? 0 : 1;
  p.om = OutMap{kB, (int64_t)(K / kB) * kB * kB, kB, kB, kB * kB, 1, int64_t(0x7fffffff), 0};
  p.alpha = 1.0f;
  p.bias = bias;
  p.act = act;
  p.debug_flags = debug_flags();
  p.debug_ts = g_debug_ts;
  return finish(p, pl, stream, f32);
}

BRK_API int brk_fc_bwd_data(const void* dz, const void* w, const void* mask, void* dx, float* colsum_ws,
                            int N, int C, int K, int b_n, int b_c, int b_k, int dtype, void* stream) {
  int rc = check_fc(N, C, K, b_n, b_c, b_k, dtype);
  if (rc) return rc;
  EngineParams p;
  std::memset(&p, 0, sizeof(p));
  p.colsum_ws = colsum_ws;
  const bool f32 = dtype == BRK_F32;
  const Plan pl = choose_plan(N, C, K / kB, false);
  const int brows = pl.pair ? pl.bn / 2 : pl.bn;
  if (!f32) {
    // A = dZ (rows n, red k) K-major
    if ((rc = enc(&p.map_a, dz, act_layout(N, K), 64, 64, 1, 2))) return rc;
    set_coords(p.ca, {0, 0, 0, 2}, {0, 0, 1, 0}, 128 * 128, 0);
    // B = W (rows c, red k) K-major: dims (k_in, c_in, cb, kb), box (64, 64, brows/64, 1)
    if ((rc = enc(&p.map_b, w, w_layout(K, C), 64, 64, brows / 64, 1))) return rc;
    set_coords(p.cb, {0, 0, brows / 64, 0}, {0, 0, 0, 1}, brows * 128, 0);
  } else {
    // A = dZ K-major: box (k 32, n 64, half 1, kb 1, nb 2)
    if ((rc = enc5(&p.map_a, dz, split_layout(N, K), {32, 64, 1, 1, 2}))) return rc;
    set_coords_f32(p.ca, 4, 2, 2, 1, 3, 128 * 128, 1, 0);
    // B = W (rows c, red k) K-major on (k32, c_in, khalf, cb, kb): box (32, 64, 1, brows/64, 1)
    if ((rc = enc5(&p.map_b, w, split_layout(K, C), {32, 64, 1, (uint32_t)(brows / 64), 1}))) return rc;
    set_coords_f32(p.cb, 3, brows / 64, 2, 1, 4, brows * 128, 1, 0);
  }
  p.m_tiles = N / (pl.pair ? 256 : 128);
  p.n_tiles = C / pl.bn;
  p.k_steps = f32 ? K / 32 : K / kB;
  p.rows = N;
  p.cols = C;
  p.out = dx;
  p.out_bf16 = f32 ? 0 : 1;
  p.om = OutMap{kB, (int64_t)(C / kB) * kB * kB, kB, kB, kB * kB, 1, int64_t(0x7fffffff), 0};
  p.alpha = 1.0f;
  p.mask = mask;
  p.debug_flags = debug_flags();
  p.debug_ts = g_debug_ts;
  return finish(p, pl, stream, f32);
}

// Split-K workspace of brk_fc_upd: [counters: 4 KiB][fp32 partial tiles].
static constexpr size_t kCounterBytes = 4096;

BRK_API size_t brk_fc_upd_workspace(int N, int C, int K) {
  if (N <= 0 || C <= 0 || K <= 0 || N % 128 || C % 128 || K % 128) return 0;
  const Plan pl = choose_plan(C, K, N / kB, true);
  if (pl.splits <= 1) return kCounterBytes;
  return kCounterBytes + engine_split_ws_bytes(pl.tiles, pl.splits, pl.bn, pl.pair);
}

BRK_API int brk_fc_upd(const void* x, const void* dz, float* dw, void* w_sgd, float lr,
                       const float* db_partials, int db_parts, float* db_out, float* bias_sgd, float bias_lr,
                       void* workspace, size_t ws_bytes, int N, int C, int K, int b_n, int b_c, int b_k,
                       int dtype, void* stream) {
  int rc = check_fc(N, C, K, b_n, b_c, b_k, dtype);
  if (rc) return rc;
  EngineParams p;
  std::memset(&p, 0, sizeof(p));
  const Plan pl = choose_plan(C, K, N / kB, workspace != nullptr);
  if (pl.splits > 1) {
    if (ws_bytes < kCounterBytes + engine_split_ws_bytes(pl.tiles, pl.splits, pl.bn, pl.pair) ||
        static_cast<size_t>(pl.tiles) * 2 * sizeof(unsigned) > kCounterBytes)
      return set_error(BRK_ERR_CONTRACT, "fc_upd: workspace too small (see brk_fc_upd_workspace)");
    p.k_splits = pl.splits;
    p.split_counters = static_cast<unsigned*>(workspace);
    p.split_ws = reinterpret_cast<float*>(static_cast<char*>(workspace) + kCounterBytes);
  }
  if (db_partials != nullptr) {
    if (db_out == nullptr || db_parts <= 0) return set_error(BRK_ERR_CONTRACT, "fc_upd: db_partials needs db_out");
    p.db_partials = db_partials;
    p.db_parts = db_parts;
    p.db_out = db_out;
    p.bias_sgd = bias_sgd;
    p.bias_lr = bias_lr;
  }
  const int brows = pl.pair ? pl.bn / 2 : pl.bn;
  const bool f32 = dtype == BRK_F32;
  if (f32 && w_sgd != nullptr)
    return set_error(BRK_ERR_CONTRACT, "fc_upd: the fused SGD updates bf16 weights (fp32: use brk_sgd_apply)");
  if (!f32) {
    // A = X^T (rows c, red n) MN-major: box (c 64, n 64, cb 2, nb 1) -> 2 atoms of 64 rows
    if ((rc = enc(&p.map_a, x, act_layout(N, C), 64, 64, 2, 1))) return rc;
    set_coords(p.ca, {0, 0, 2, 0}, {0, 0, 0, 1}, 128 * 128, 1);
    // B = dZ^T (rows k, red n) MN-major: box (k 64, n 64, kb brows/64, nb 1)
    if ((rc = enc(&p.map_b, dz, act_layout(N, K), 64, 64, brows / 64, 1))) return rc;
    set_coords(p.cb, {0, 0, brows / 64, 0}, {0, 0, 0, 1}, brows * 128, 1);
  } else {
    // A = X^T MN-major on (c32, n_in, chalf, cb, nb): box (32, 32, 2, 2, 1) = 4 atoms (128 rows)
    if ((rc = enc5(&p.map_a, x, split_layout(N, C), {32, 32, 2, 2, 1}, true))) return rc;
    set_coords_f32(p.ca, 3, 2, 1, 32, 4, 128 * 128, 1, 1);
    // B = dZ^T MN-major: box (32, 32, 2, brows/64, 1)
    if ((rc = enc5(&p.map_b, dz, split_layout(N, K), {32, 32, 2, (uint32_t)(brows / 64), 1}, true))) return rc;
    set_coords_f32(p.cb, 3, brows / 64, 1, 32, 4, brows * 128, 1, 1);
  }
  p.m_tiles = C / (pl.pair ? 256 : 128);
  p.n_tiles = K / pl.bn;
  p.k_steps = f32 ? N / 32 : N / kB;
  p.rows = C;
  p.cols = K;
  p.out = dw;
  p.out_bf16 = 0;
  // dW [Kb][Cb][64 c][64 k]: row c -> (c/64)*4096 + (c%64)*64 ; col k -> (k/64)*Cb*4096 + k%64
  p.om = OutMap{kB, kB * kB, kB, kB, (int64_t)(C / kB) * kB * kB, 1, int64_t(0x7fffffff), 0};
  p.alpha = 1.0f;
  p.sgd_w = w_sgd;
  p.sgd_lr = lr;
  p.debug_flags = debug_flags();
  p.debug_ts = g_debug_ts;
  return finish(p, pl, stream, f32);
}

// dz_out = dy * (y > 0) when y != NULL (dz_out may alias dy), db = column sums,
// bias_sgd -= lr * db when bias_sgd != NULL.
// workspace: brk_fc_bias_grad_workspace(K) bytes (zero-initialised once).
BRK_API int brk_fc_bias_grad(const void* dy, const void* y, void* dz_out, float* db, void* workspace,
                             int N, int K, int b_n, int b_k, float* bias_sgd, float lr, void* stream) {
  return brk_fc_bias_grad_dt(dy, y, dz_out, db, workspace, N, K, b_n, b_k, bias_sgd, lr, BRK_BF16, stream);
}

BRK_API int brk_fc_bias_grad_dt(const void* dy, const void* y, void* dz_out, float* db, void* workspace,
                                int N, int K, int b_n, int b_k, float* bias_sgd, float lr, int dtype, void* stream) {
  if (dtype != BRK_BF16 && dtype != BRK_F32) return set_error(BRK_ERR_CONTRACT, "bias_grad: dtype bf16 or f32");
  if (b_n != kB || b_k != kB || N % kB || K % kB || N % kSplit)
    return set_error(BRK_ERR_CONTRACT, "bias_grad needs b_n=b_k=64, N and K multiples of 64");
  float* partial = static_cast<float*>(workspace);
  unsigned* counters = reinterpret_cast<unsigned*>(partial + static_cast<size_t>(kSplit) * K);
  dim3 grid(K / kB, kSplit);
  g_launches.fetch_add(1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(256);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  cudaError_t err =
      dtype == BRK_F32
          ? cudaLaunchKernelEx(&cfg, bias_grad_kernel<float>, static_cast<const float*>(dy),
                               static_cast<const float*>(y), static_cast<float*>(dz_out), db, partial, counters, N, K,
                               bias_sgd, lr)
          : cudaLaunchKernelEx(&cfg, bias_grad_kernel<__nv_bfloat16>, static_cast<const __nv_bfloat16*>(dy),
                               static_cast<const __nv_bfloat16*>(y), static_cast<__nv_bfloat16*>(dz_out), db,
                               partial, counters, N, K, bias_sgd, lr);
  if (err != cudaSuccess) return set_cuda_error(err, "bias_grad launch");
  return BRK_OK;
}

// Diagnostic: subsequent engine launches record per-CTA phase timestamps into
// ts (device, >= 8 * grid entries); NULL disables.
BRK_API void brk_diag_set_timestamps(unsigned long long* ts) { g_debug_ts = ts; }

BRK_API size_t brk_fc_bias_grad_workspace(int K) {
  return static_cast<size_t>(kSplit) * K * sizeof(float) + static_cast<size_t>(K / kB + 1) * sizeof(unsigned);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// The whole MLP training step (BASELINE config 2) as ONE persistent grouped
// launch of the engine: 3L dependent problems (L forward, then per layer from
// the top bwd-data and weight update), tile-level dependency counters instead
// of kernel boundaries, so the tail of one GEMM overlaps the head of the next.
// ---------------------------------------------------------------------------
namespace brk {
int launch_engine_group(const EngineGroup& G, int bn, int pair, cudaStream_t stream);
}

extern "C" {

}  // extern "C"

namespace {
// MLP step workspace: the dependency counters (zeroed by every call)
size_t mlp_counter_bytes(int L) { return (static_cast<size_t>(3 * L) * kCounterStride + 1) * sizeof(unsigned); }
// 64-column chunk counters of the chained passes: [3L][N/256][2][C/64]
size_t mlp_chunk_counters(int L, int N, int C) { return static_cast<size_t>(3 * L) * (N / 256) * 2 * (C / 64); }
}  // namespace

// The captured engine problems of the step -> the lean MLP kernel's problem table (brk_mlp.h):
// the same operand maps and schedule, plus TMA maps for the epilogue's stores and side operands.
// The captured engine problems of the step -> the lean MLP kernel's problem table (brk_mlp.h):
// the same operand maps and schedule, plus TMA maps for the epilogue's stores and side operands
// (bf16: 64-column boxes; fp32 storage / TF32: 32-column boxes).
static int to_mlp_group(const EngineGroup& G, const int* kinds, int N, int C, int dtype, MlpGroup& M) {
  std::memset(&M, 0, sizeof(M));
  M.sched = G.sched;
  const bool f32 = dtype == BRK_F32;
  M.tf32 = f32 ? 1 : 0;
  const Map4 act = act_layout(N, C), wl = w_layout(C, C);
  const uint32_t bx = f32 ? 32 : 64;  // side / output box width (128 B of elements)
  auto enc_act = [&](CUtensorMap* m, const void* ptr) {
    const uint32_t box[4] = {bx, 32, 1, 1};
    return encode_tmap(m, ptr, !f32, 4, act.dims, act.strides, box);
  };
  auto enc_w = [&](CUtensorMap* m, const void* ptr) {
    const uint32_t box[4] = {bx, 32, 1, 1};
    return encode_tmap(m, ptr, !f32, 4, wl.dims, wl.strides, box);
  };
  int rc = 0;
  for (int q = 0; q < G.sched.n_probs && !rc; ++q) {
    const EngineParams& e = G.probs[q];
    MlpProb& m = M.probs[q];
    m.map_a = e.map_a;
    m.map_b = e.map_b;
    m.m_tiles = e.m_tiles;
    m.n_tiles = e.n_tiles;
    m.k_steps = e.k_steps;
    for (int d = 0; d < 5; ++d) {
      if (e.ca.base[d] != 0 || e.cb.base[d] != 0) return set_error(BRK_ERR_CONTRACT, "mlp step: operand base offset");
      m.a_rc[d] = e.ca.rc[d]; m.a_k0[d] = e.ca.kc[0][d]; m.a_k1[d] = e.ca.kc[1][d];
      m.b_rc[d] = e.cb.rc[d]; m.b_k0[d] = e.cb.kc[0][d]; m.b_k1[d] = e.cb.kc[1][d];
    }
    m.a_mn = e.ca.mn_major;
    m.b_mn = e.cb.mn_major;
    m.cols = e.cols;
    m.b_first = e.b_first;
    m.bias = e.bias;
    m.colsum_ws = e.colsum_ws;
    m.db_partials = e.db_partials;
    m.db_parts = e.db_parts;
    m.db_out = e.db_out;
    m.bias_sgd = e.bias_sgd;
    m.lr = e.sgd_lr != 0.0f ? e.sgd_lr : e.bias_lr;
    m.kind = kinds[q];
    if (m.kind != kMlpUpd) {
      if ((rc = enc_act(&m.map_out, e.out))) break;
      const void* in = m.kind == kMlpFwdTop ? e.aux_in : (m.kind == kMlpBwd ? e.mask : nullptr);
      if (in != nullptr) {
        m.has_in = 1;
        if ((rc = enc_act(&m.map_in, in))) break;
      }
      if (m.kind == kMlpFwdTop) {
        m.has_aux = 1;
        if ((rc = enc_act(&m.map_aux, e.aux_out))) break;
      }
    } else {
      const uint32_t box[4] = {32, 32, 1, 1};
      if ((rc = encode_tmap(&m.map_out, e.out, false, 4, wl.dims, wl.strides, box))) break;  // dW fp32
      if (e.sgd_w != nullptr) {
        m.has_in = m.has_aux = 1;
        if ((rc = enc_w(&m.map_in, e.sgd_src != nullptr ? e.sgd_src : e.sgd_w))) break;
        if ((rc = enc_w(&m.map_aux, e.sgd_w))) break;
      }
    }
  }
  return rc;
}

extern "C" {

BRK_API size_t brk_mlp_step_workspace_bytes(int L, int N, int C) {
  if (L < 1 || N < 256 || C < 64) return 0;
  return mlp_counter_bytes(L) + mlp_chunk_counters(L, N, C) * sizeof(unsigned);
}

BRK_API int brk_mlp_step(int L, int N, int C, const void* const* y, void* const* dz, const void* dy,
                         void* const* w, void* const* w_next, float* const* bias, float* const* dw, float* const* db,
                         float* const* colsum, float lr, void* workspace, size_t ws_bytes, void* stream) {
  return brk_mlp_step_dt(L, N, C, y, dz, dy, w, w_next, bias, dw, db, colsum, lr, workspace, ws_bytes, BRK_BF16,
                         stream);
}

BRK_API int brk_mlp_step_dt(int L, int N, int C, const void* const* y, void* const* dz, const void* dy,
                            void* const* w, void* const* w_next, float* const* bias, float* const* dw,
                            float* const* db, float* const* colsum, float lr, void* workspace, size_t ws_bytes,
                            int dtype, void* stream) {
  if (L < 1 || 3 * L > kMaxProbs) return set_error(BRK_ERR_CONTRACT, "mlp_step: 1 <= layers <= 4");
  int rc = check_fc(N, C, C, kB, kB, kB, dtype);
  if (rc) return rc;
  if (N % 256 || C % 256 || N / 256 > kCounterStride - 1)
    return set_error(BRK_ERR_CONTRACT, "mlp_step: N, C multiples of 256, N <= 16384");
  if (workspace == nullptr || ws_bytes < brk_mlp_step_workspace_bytes(L, N, C))
    return set_error(BRK_ERR_CONTRACT, "mlp_step: workspace smaller than brk_mlp_step_workspace_bytes(L, N, C)");
  unsigned* counters = static_cast<unsigned*>(workspace);
  // chained passes (fwd l <- fwd l-1, bwd-data l <- bwd-data l+1) wait per 64-column chunk of
  // the rows they read (dep_mode 2) instead of for the whole 256-row block (mode 0);
  // BRK_MLP_CHUNK=0 (diagnostics) restores the row-block dependencies
  const char* chunk_env = std::getenv("BRK_MLP_CHUNK");
  const int chunk_mode = (chunk_env != nullptr && std::atoi(chunk_env) == 0) ? 0 : 2;
  // BRK_MLP_BFIRST=0 (diagnostics): producers wait for a tile's dependencies before loading
  // the weight operand too
  const char* bfirst_env = std::getenv("BRK_MLP_BFIRST");
  const int b_first = bfirst_env ? std::atoi(bfirst_env) : 1;
  static EngineGroup G;  // large: keep off the stack (host-side staging of the kernel parameter block)
  std::memset(&G, 0, sizeof(G));
  GroupSched& gs = G.sched;
  const Plan force{1, 128, 1, 0};
  g_force_plan = &force;
  int q = 0;
  auto capture = [&](auto&& build) -> int {
    g_capture = &G.probs[q];
    const int r = build();
    g_capture = nullptr;
    for (int d = 0; d < kMaxDeps; ++d) gs.dep_prob[q][d] = -1;
    return r;
  };
  int fwd_of[8], bwd_of[8], upd_of[8];
  int kinds[kMaxProbs];
  for (int i = 0; i < 8; ++i) fwd_of[i] = bwd_of[i] = upd_of[i] = -1;
  for (int l = 0; l < L && !rc; ++l) {  // forward: y[l+1] = relu(W_l y[l] + b_l)
    rc = capture([&] {
      return brk_fc_fwd(y[l], w[l], bias[l], const_cast<void*>(y[l + 1]), N, C, C, kB, kB, kB, kActRelu, dtype,
                        stream);
    });
    kinds[q] = l == L - 1 ? kMlpFwdTop : kMlpFwd;
    if (l > 0) { gs.dep_prob[q][0] = fwd_of[l - 1]; gs.dep_mode[q][0] = chunk_mode; }
    G.probs[q].b_first = b_first;  // B = W_l, not written in this launch before the weight updates
    if (l == L - 1) {  // top layer also emits dz_L = dy * (y_L > 0) and its column sums
      const char* de = std::getenv("BRK_MLP_DIAG");  // diagnostics only: drop parts of the top epilogue
      const int diag = de ? std::atoi(de) : 0;
      if (!(diag & 1)) {
        G.probs[q].aux_in = dy;
        G.probs[q].aux_out = dz[L];
      }
      if (!(diag & 2)) G.probs[q].colsum_ws = colsum[L];
    }
    fwd_of[l] = q++;
  }
  auto add_bwd = [&](int l) {  // layer l (weights w[l-1]): bwd-data
    const int dz_src = l == L ? fwd_of[L - 1] : bwd_of[l + 1];
    if (dz_src < 0 || bwd_of[l] >= 0) { rc = set_error(BRK_ERR_CONTRACT, "mlp_step: unit order breaks a dependency"); return; }
    rc = capture([&] {
      return brk_fc_bwd_data(dz[l], w[l - 1], l > 1 ? y[l - 1] : nullptr, dz[l - 1], l > 1 ? colsum[l - 1] : nullptr,
                             N, C, C, kB, kB, kB, dtype, stream);
    });
    kinds[q] = l > 1 ? kMlpBwd : kMlpBwdPlain;
    gs.dep_prob[q][0] = dz_src; gs.dep_mode[q][0] = chunk_mode;  // the same rows of dz_l
    // B = W_{l-1}: with in-place SGD it is rewritten only after this pass completes (dependency below)
    G.probs[q].b_first = b_first;
    bwd_of[l] = q++;
  };
  auto add_upd = [&](int l) {  // layer l: weight update (+ fused SGD)
    const int dz_src = l == L ? fwd_of[L - 1] : bwd_of[l + 1];
    if (dz_src < 0 || upd_of[l] >= 0 || (lr != 0.0f && w_next == nullptr && bwd_of[l] < 0)) {
      rc = set_error(BRK_ERR_CONTRACT, "mlp_step: unit order breaks a dependency");
      return;
    }
    // lr == 0: gradients only (data parallel: all-reduce, then SGD outside the step)
    const bool sgd = lr != 0.0f;
    void* w_out = !sgd ? nullptr : (w_next != nullptr ? w_next[l - 1] : w[l - 1]);
    // (fp32 weights: brk_fc_upd rejects a fused fp32 SGD for its own epilogue; the lean kernel
    //  does it, so the SGD operands are set on the captured problem)
    const bool f32 = dtype == BRK_F32;
    rc = capture([&] {
      return brk_fc_upd(y[l - 1], dz[l], dw[l - 1], f32 ? nullptr : w_out, lr, colsum[l], N / 32, db[l - 1],
                        sgd ? bias[l - 1] : nullptr, lr, nullptr, 0, N, C, C, kB, kB, kB, dtype, stream);
    });
    if (f32 && w_out != nullptr) {
      G.probs[q].sgd_w = w_out;
      G.probs[q].sgd_lr = lr;
    }
    kinds[q] = kMlpUpd;
    gs.dep_prob[q][0] = dz_src; gs.dep_mode[q][0] = 1;  // all of dz_l (reduction over N)
    if (!sgd) {
      // no weight write: no ordering against the bwd-data pass
    } else if (w_next != nullptr) {
      G.probs[q].sgd_src = w[l - 1];  // double-buffered weights: no write-after-read on W_{l-1}
    } else {
      gs.dep_prob[q][1] = bwd_of[l]; gs.dep_mode[q][1] = 1;  // W_{l-1} read by bwd-data before the SGD rewrites it
    }
    upd_of[l] = q++;
  };
  // Work-unit order (the global tile order; CTA pairs run their units in it).  Default with
  // double-buffered weights (or no SGD): the bwd-data chain of layers L..2 first, then the
  // weight updates of layers L..1, then the bwd-data of layer 1 (dx: nothing in the step reads
  // it), scheduled over the pairs by the host list scheduler (brk_mlp.cu mlp_list_schedule),
  // which places the long weight-update units where the chain leaves pairs idle: 64.1 ->
  // 60.9 us per step.  In-place SGD (the update of W_{l-1} must follow the bwd-data pass that
  // reads it): the weight update of layer l after the bwd-data pass of layer l - lag, round
  // robin.  BRK_MLP_ORDER (tuning): the backward units as (kind, layer) pairs, e.g.
  // "b4b3u4b2u3u2u1b1"; every bwd-data (b) and weight update (u) exactly once, each after the
  // units it reads.
  const char* lag_env = std::getenv("BRK_MLP_UPD_LAG");
  const char* order_env = std::getenv("BRK_MLP_ORDER");
  const bool chain_first = order_env == nullptr && lag_env == nullptr && (w_next != nullptr || lr == 0.0f);
  if (chain_first) {
    for (int l = L; l >= 2 && !rc; --l) add_bwd(l);
    for (int l = L; l >= 1 && !rc; --l) add_upd(l);
    if (!rc) add_bwd(1);
  } else if (order_env != nullptr) {
    int n = 0;
    for (const char* c = order_env; c[0] && c[1] && !rc; c += 2, ++n) {
      const int l = c[1] - '0';
      if (l < 1 || l > L || (c[0] != 'b' && c[0] != 'u')) rc = set_error(BRK_ERR_CONTRACT, "mlp_step: bad BRK_MLP_ORDER");
      else if (c[0] == 'b') add_bwd(l);
      else add_upd(l);
    }
    if (!rc && n != 2 * L) rc = set_error(BRK_ERR_CONTRACT, "mlp_step: BRK_MLP_ORDER must list 2L units");
  } else {
    const int lag = lag_env ? std::max(0, std::atoi(lag_env)) : 1;
    for (int l = L; l >= 1 - lag && !rc; --l) {
      if (l >= 1) add_bwd(l);
      if (!rc && l + lag <= L && l + lag >= 1) add_upd(l + lag);
    }
  }
  g_force_plan = nullptr;
  (void)upd_of;
  if (rc) return rc;
  gs.n_probs = q;
  gs.tile_begin[0] = 0;
  for (int i = 0; i < q; ++i)
    gs.tile_begin[i + 1] = gs.tile_begin[i] + G.probs[i].m_tiles * G.probs[i].n_tiles;
  gs.counters = counters;
  gs.chunk_counters = counters + (mlp_counter_bytes(L) / sizeof(unsigned));
  gs.chunk_mb = N / 256;
  gs.chunk_n = C / 64;
  gs.chunk_target = 4;  // BN=128 pairs: the 4 epilogue warps (TMEM lane quarters) of a column half
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // the counters are zero: zero-initialised once by the caller, re-zeroed by every launch's
  // last CTA (no memset between back-to-back steps)
  g_launches.fetch_add(1);
  const char* lean_env = std::getenv("BRK_MLP_LEAN");  // 0 (diagnostics): the generic grouped engine
  if (lean_env != nullptr && std::atoi(lean_env) == 0 && dtype == BRK_BF16) return launch_engine_group(G, 128, 1, st);
  static MlpGroup M;
  if ((rc = to_mlp_group(G, kinds, N, C, dtype, M))) return rc;
  M.debug_ts = g_debug_ts;
  const char* fl = std::getenv("BRK_MLP_FLAGS");
  M.flags = fl ? std::atoi(fl) : 0;
  const char* cse = std::getenv("BRK_MLP_CS");
  M.cluster = cse ? std::atoi(cse) : 2;
  // host list schedule (BRK_MLP_LIST=1/0 forces it on/off): the default with the chain-first
  // order (round robin with it: 66.0 us; the lag order is equal either way, 63.1 us)
  const char* lse = std::getenv("BRK_MLP_LIST");
  M.list_len = lse != nullptr ? (std::atoi(lse) != 0 ? 1 : 0) : (chain_first ? 1 : 0);
  return launch_mlp_group(M, st);
}

}  // extern "C"
