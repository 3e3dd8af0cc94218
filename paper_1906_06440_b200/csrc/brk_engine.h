// brk_engine.h — the TMA-fed, warp-specialised tcgen05 BRGEMM engine.
//
// One launch computes a set of output tiles (128 x BN per CTA, or 256 x BN
// per CTA pair).  Every tile is the batch-reduce  D = sum_s A_s * B_s^T  over
// "k-steps" s; each k-step is one (A block, B block) pair of the paper's
// batch list, fetched by TMA from a tensor map at coordinates that are an
// affine function of (tile row block, k-step).  This is the stride/offset
// BRGEMM of the paper expressed as TMA coordinates: the blocked layouts of
// the reference (tensor.py:143-247) become <=5-d tensor maps whose boxes land
// directly in the canonical UMMA shared-memory layout (128B swizzle).
#pragma once
#include <cstdint>
#include <cuda.h>

namespace brk {

constexpr int kEngineBM = 128;  // tile rows per CTA = TMEM lanes

// How one operand's k-step box(es) are located.
//   coord[d] = rc[d]*rowblk + kq[d]*(s / kdiv) + kr[d]*(s % kdiv) + lc[d]*load
// for load in [0, n_loads); each load writes load_bytes to consecutive smem.
struct OperandCoords {
  int32_t rc[5];
  int32_t kq[5];
  int32_t kr[5];
  int32_t lc[5];
  int32_t kdiv;
  int32_t n_loads;
  uint32_t load_bytes;
  int32_t mn_major;  // 0: K-major rows of 128 B; 1: MN-major 64-wide atoms
  int32_t ndims;
};

// Output addressing: off(r, c) = (r/rb)*rh + (r%rb)*rl + (c/cb)*ch + (c%cb)*cl
struct OutMap {
  int64_t rb, rh, rl;
  int64_t cb, ch, cl;
};

enum EpiAct : int { kActNone = 0, kActRelu = 1, kActSigmoid = 2 };

struct EngineParams {
  CUtensorMap map_a;  // 64-byte aligned inside the param block
  CUtensorMap map_b;
  OperandCoords ca;
  OperandCoords cb;
  int32_t m_tiles, n_tiles, k_steps;
  int32_t rows, cols;  // valid output extent (M, N)
  // split-K: the batch list of a tile is cut into k_splits contiguous chunks;
  // partial tiles go to split_ws, the last-arriving split sums them in split
  // order (deterministic) and runs the epilogue.  counters self-reset.
  int32_t k_splits;
  float* split_ws;
  unsigned* split_counters;
  // epilogue
  void* out;
  int32_t out_bf16;
  OutMap om;
  float alpha;
  float beta;            // beta != 0 reads out (same dtype) before writing
  const float* bias;     // per output column, may be null
  int32_t act;           // EpiAct
  const void* mask;      // bf16 tensor in the OUTPUT layout; out *= (mask > 0)
  void* sgd_w;           // bf16 weights in the OUTPUT layout: w -= lr * out
  float sgd_lr;
  // fused column sums of the final output (bias gradient of the next pass):
  // colsum_ws[(row / 32) * cols + col] = sum of the 32 rows' values
  float* colsum_ws;
  // reduction of column-sum partials written by a previous pass (rows of
  // that pass / 32 of them): tiles of row block 0 write
  // db[col] = sum_p db_partials[p * cols + col]; bias_sgd[col] -= lr * db[col]
  const float* db_partials;
  int32_t db_parts;
  float* db_out;
  float* bias_sgd;
  float bias_lr;
  int32_t debug_flags;  // bit0: skip MMA, bit1: skip TMA, bit2: no k rotation (diagnostics)
  // diagnostics: per-CTA %globaltimer stamps [blockIdx.x][8]:
  // 0 entry, 1 setup done, 2 first TMA issued, 3 first full-barrier passed (MMA),
  // 4 last MMA committed, 5 epilogue got accumulator, 6 epilogue done, 7 exit
  unsigned long long* debug_ts;
};

}  // namespace brk
