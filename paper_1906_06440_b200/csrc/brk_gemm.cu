// brk_gemm.cu — dense row-major GEMM on the tcgen05 engine:
//     C[M][N] (fp32 or bf16, row stride ldc) = act(alpha * op(A) op(B) + bias) (+ beta C)
// A is M x K, stored K-contiguous ("K-major", a_kmajor = 1: A[m][k] at m*lda + k)
// or M-contiguous (a_kmajor = 0: A[m][k] at k*lda + m); B is N x K likewise
// (b_kmajor = 1: B[n][k] at n*ldb + k; 0: at k*ldb + n).  bf16 operands.
//
// This is the batch-reduce GEMM with a batch list of K/64 entries whose
// blocks are consecutive 64-wide slices of dense operands: the LSTM drivers
// use it for the input projection W x over all steps, the backward-data
// product dpre W, and the weight gradients dpre^T x / dpre^T h over T*N rows
// (the reduction of the weight update runs over all steps in TMEM).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "brk_engine.h"
#include "brk_internal.h"
#include "brk_tma_host.h"

namespace brk {

int launch_engine(const EngineParams& p, int bn, int tf32, int pair, int max_units, cudaStream_t stream);
int engine_sm_count();
size_t engine_split_ws_bytes(int tiles, int splits, int bn, int pair);

namespace {

// A operand map: rows = the GEMM's M (or N for B) side, 128 (or brows) per tile.
//   K-major : 2-d (K, rows), box (64, box_rows)            -> one load
//   MN-major: 2-d (rows, K), box (64, 64), box_rows/64 loads (64-wide atoms)
int operand_map(CUtensorMap* map, OperandCoords& oc, const void* ptr, int64_t rows, int64_t K, int64_t ld,
                int kmajor, int box_rows, bool f32 = false) {
  std::memset(&oc, 0, sizeof(oc));
  oc.kdiv0 = 1 << 30;
  oc.kdiv1 = 1;
  oc.ndims = 2;
  if (f32) {
    // fp32 (TF32): one k-step = 32 elements of K (a 128 B swizzle atom column)
    if (kmajor) {
      const uint64_t dims[2] = {(uint64_t)K, (uint64_t)rows};
      const uint64_t strides[2] = {1, (uint64_t)ld};
      const uint32_t box[2] = {32, (uint32_t)box_rows};
      oc.rc[1] = box_rows;
      oc.kc[0][0] = 32;
      oc.n_loads = 1;
      oc.load_bytes = box_rows * 128;
      oc.mn_major = 0;
      return encode_tmap(map, ptr, false, 2, dims, strides, box);
    }
    const uint64_t dims[2] = {(uint64_t)rows, (uint64_t)K};
    const uint64_t strides[2] = {1, (uint64_t)ld};
    const uint32_t box[2] = {32, 32};
    oc.rc[0] = box_rows;
    oc.lc[0] = 32;
    oc.kc[0][1] = 32;
    oc.n_loads = box_rows / 32;
    oc.load_bytes = 32 * 128;
    oc.mn_major = 1;
    return encode_tmap(map, ptr, false, 2, dims, strides, box, true);
  }
  if (kmajor) {
    const uint64_t dims[2] = {(uint64_t)K, (uint64_t)rows};
    const uint64_t strides[2] = {1, (uint64_t)ld};
    const uint32_t box[2] = {64, (uint32_t)box_rows};
    oc.rc[1] = box_rows;   // row block
    oc.kc[0][0] = 64;      // k-step -> K offset
    oc.n_loads = 1;
    oc.load_bytes = box_rows * 128;
    oc.mn_major = 0;
    return encode_tmap(map, ptr, true, 2, dims, strides, box);
  }
  const uint64_t dims[2] = {(uint64_t)rows, (uint64_t)K};
  const uint64_t strides[2] = {1, (uint64_t)ld};
  const uint32_t box[2] = {64, 64};
  oc.rc[0] = box_rows;
  oc.lc[0] = 64;
  oc.kc[0][1] = 64;
  oc.n_loads = box_rows / 64;
  oc.load_bytes = 64 * 128;
  oc.mn_major = 1;
  return encode_tmap(map, ptr, true, 2, dims, strides, box);
}

struct GemmPlan {
  int pair, bn, splits;
  int64_t tiles;
};

GemmPlan gemm_plan(int64_t M, int N, int k_steps, bool split_ok) {
  const int sms = engine_sm_count();
  struct Opt { int pair, bn; double eff; };
  const Opt opts[] = {{1, 256, 1.0}, {1, 128, 0.67}, {0, 128, 0.5}, {0, 64, 0.4}};
  GemmPlan best{0, 0, 1, 0};
  double best_cost = 0;
  for (const Opt& o : opts) {
    if (N % o.bn) continue;
    const int tr = o.pair ? 256 : 128;
    const int64_t tiles = ((M + tr - 1) / tr) * (N / o.bn);
    const int64_t units = o.pair ? sms / 2 : sms;
    const double per_tile = static_cast<double>(tr) * o.bn * k_steps / ((o.pair ? 2.0 : 1.0) * o.eff);
    int max_split = 1;
    if (split_ok)
      max_split = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(k_steps / 8, units / std::max<int64_t>(1, tiles))));
    for (int sp = 1; sp <= max_split; ++sp) {
      const int64_t waves = (tiles * sp + units - 1) / units;
      const double cost = waves * per_tile / sp + (sp > 1 ? 0.05 * per_tile : 0.0) + 2.0e5;
      if (best.bn == 0 || cost < best_cost) {
        const int per = (k_steps + sp - 1) / sp;
        best = GemmPlan{o.pair, o.bn, (k_steps + per - 1) / per, tiles};
        best_cost = cost;
      }
    }
  }
  return best;
}

}  // namespace

// split-K workspace: splits * M * N fp32 slices (0 = no split needed)
size_t gemm_dense_workspace(int64_t M, int N, int K) {
  if (M <= 0 || N <= 0 || K <= 0 || N % 64) return 0;
  const GemmPlan pl = gemm_plan(M, N, (K + 63) / 64, true);
  return pl.splits > 1 ? static_cast<size_t>(pl.splits) * M * N * sizeof(float) : 0;
}

int split_reduce(const float* ws, int splits, int64_t n, float* dst, void* w_sgd, float lr, cudaStream_t stream);

}  // namespace brk

using namespace brk;

extern "C" {

BRK_API size_t brk_gemm_dense_workspace(int64_t M, int N, int K) { return gemm_dense_workspace(M, N, K); }

static int gemm_dense_impl(const void* a, int64_t lda, int a_kmajor, const void* b, int64_t ldb, int b_kmajor,
                           void* c, int64_t ldc, int c_bf16, int64_t M, int N, int K, float alpha, float beta,
                           const float* bias, int act, void* workspace, size_t ws_bytes, void* stream, bool f32) {
  char buf[256];
  // K need not be a multiple of the k-step: the operand maps zero-fill the tail of the last k-step
  if (M <= 0 || N <= 0 || K <= 0 || N % 64 || lda % (f32 ? 4 : 8) || ldb % (f32 ? 4 : 8) || ldc % 4) {
    std::snprintf(buf, sizeof(buf),
                  "gemm_dense: need M, N, K > 0, N a multiple of 64, 16-byte aligned rows (M=%lld N=%d K=%d)",
                  (long long)M, N, K);
    return set_error(BRK_ERR_CONTRACT, buf);
  }
  if (M >= (int64_t(1) << 31)) return set_error(BRK_ERR_CONTRACT, "gemm_dense: M must fit int32");
  if (act < kActNone || act > kActSigmoid) return set_error(BRK_ERR_CONTRACT, "unknown activation");
  const int k_steps = f32 ? (K + 31) / 32 : (K + 63) / 64;
  const bool split_ok = workspace != nullptr && beta == 0.0f && bias == nullptr && act == kActNone && !c_bf16 &&
                        alpha == 1.0f;
  // planned in 64-element k-steps for both storage types (matches brk_gemm_dense_workspace)
  const GemmPlan pl = gemm_plan(M, N, (K + 63) / 64, split_ok);
  if (pl.bn == 0) return set_error(BRK_ERR_CONTRACT, "gemm_dense: no engine tile fits N");
  if (pl.splits > 1 && ws_bytes < static_cast<size_t>(pl.splits) * M * N * sizeof(float))
    return set_error(BRK_ERR_CONTRACT, "gemm_dense: workspace too small (see brk_gemm_dense_workspace)");
  if (pl.splits > 1 && ldc != N) return set_error(BRK_ERR_CONTRACT, "gemm_dense: split-K needs ldc == N");
  const int brows = pl.pair ? pl.bn / 2 : pl.bn;
  EngineParams p;
  std::memset(&p, 0, sizeof(p));
  int rc;
  if ((rc = operand_map(&p.map_a, p.ca, a, M, K, lda, a_kmajor, 128, f32))) return rc;
  if ((rc = operand_map(&p.map_b, p.cb, b, N, K, ldb, b_kmajor, brows, f32))) return rc;
  p.m_tiles = static_cast<int>((M + (pl.pair ? 255 : 127)) / (pl.pair ? 256 : 128));
  p.n_tiles = N / pl.bn;
  p.k_steps = k_steps;
  p.rows = static_cast<int>(M);
  p.cols = N;
  p.out_bf16 = c_bf16;
  // row-major C: off(r, c) = r * ldc + c
  p.om = OutMap{int64_t(0x7fffffff), 0, ldc, 64, 64, 1, int64_t(0x7fffffff), 0};
  p.alpha = alpha;
  p.beta = beta;
  p.bias = bias;
  p.act = act;
  const char* dbg = std::getenv("BRK_DEBUG_FLAGS");
  p.debug_flags = dbg ? std::atoi(dbg) : 0;
  if (pl.splits > 1) {
    p.k_splits = pl.splits;
    p.split_slice = M * static_cast<int64_t>(N);
    p.out = workspace;
    p.om.rl = N;  // slices are dense M x N
  } else {
    p.out = c;
  }
  g_launches.fetch_add(1);
  rc = launch_engine(p, pl.bn, f32 ? 1 : 0, pl.pair, 0, static_cast<cudaStream_t>(stream));
  if (rc || pl.splits <= 1) return rc;
  return split_reduce(static_cast<const float*>(workspace), pl.splits, M * static_cast<int64_t>(N),
                      static_cast<float*>(c), nullptr, 0.0f, static_cast<cudaStream_t>(stream));
}

BRK_API int brk_gemm_dense(const void* a, int64_t lda, int a_kmajor, const void* b, int64_t ldb, int b_kmajor,
                           void* c, int64_t ldc, int c_bf16, int64_t M, int N, int K, float alpha, float beta,
                           const float* bias, int act, void* workspace, size_t ws_bytes, void* stream) {
  return gemm_dense_impl(a, lda, a_kmajor, b, ldb, b_kmajor, c, ldc, c_bf16, M, N, K, alpha, beta, bias, act,
                         workspace, ws_bytes, stream, false);
}

BRK_API int brk_gemm_dense_f32(const float* a, int64_t lda, int a_kmajor, const float* b, int64_t ldb,
                               int b_kmajor, void* c, int64_t ldc, int c_bf16, int64_t M, int N, int K, float alpha,
                               float beta, const float* bias, int act, void* workspace, size_t ws_bytes,
                               void* stream) {
  return gemm_dense_impl(a, lda, a_kmajor, b, ldb, b_kmajor, c, ldc, c_bf16, M, N, K, alpha, beta, bias, act,
                         workspace, ws_bytes, stream, true);
}

}  // extern "C"
