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

// How one operand's k-step box(es) are located.  The k-step s is split into
// mixed-radix digits d0 = s % kdiv0, d1 = (s / kdiv0) % kdiv1,
// d2 = s / (kdiv0 * kdiv1) (e.g. conv: (s, r, c_b)) — or, with kdiv2 set, d2 = that % kdiv2
// and d3 = that / kdiv2 (TF32 conv: (channel half, s, r, c_b)); then for load l:
//   coord[d] = base[d] + rc[d]*rowblk + sum_j kc[j][d]*d_j + lc[d]*l
// and each load writes load_bytes to consecutive smem.
//
// kind != 0 selects TMA im2col mode on a 5-d map (64 channels, W, H, N, X)
// of a blocked activation [N][X_b][H][W][64] (X = channel blocks), whose
// pixel walk (W fastest, then H, then N) is the implicit-GEMM row/K order:
//   kind 1: rows are output pixels, pix = rowblk * 128 (clamped to the last
//           pixel; rows past the end are masked in the epilogue); the filter
//           tap offsets (w, h) = (ok[0] . d, ok[1] . d)
//   kind 2: the reduction runs over pixels, pix = s * 64; atom a = rowblk *
//           n_loads + l is (c_b, rs) = (a % atom_cb, a / atom_cb) with the
//           tap (rs % atom_s, rs / atom_s)  (conv weight update, input side)
//   kind 3: the reduction runs over pixels, pix = s * 64, no tap offsets
//           (conv weight update, output-gradient side)
//   kind 5: tile mode (not im2col), TF32 weight update: atom a = rowblk * n_loads + l is
//           ((rs * atom_cb + c_b) * 2 + half) and adds (32 half, rs % atom_s, rs / atom_s, c_b)
//           to coords 0..3
// pixel -> (n, p, q) adds (q*cstride - pad_w, p*cstride - pad_h, n) to coords
// 1..3.  The maps' bounding boxes extend two images past N (zero fill), so a
// pixel walk that runs off the end reads zeros (K-side kinds rely on it).
struct OperandCoords {
  int32_t base[5];
  int32_t rc[5];
  int32_t kc[4][5];
  int32_t lc[5];
  int32_t kdiv0, kdiv1;
  int32_t kdiv2;  // 0: no fourth digit (d2 = s / (kdiv0 * kdiv1)); else d2 = that % kdiv2, d3 = that / kdiv2
  int32_t n_loads;
  uint32_t load_bytes;
  int32_t mn_major;  // 0: K-major rows of 128 B; 1: MN-major 64-wide atoms
  int32_t ndims;
  int32_t kind;
  int32_t P, Q, cstride, pad_h, pad_w, total_pix;
  int32_t ok[2][3];
  int32_t atom_cb, atom_s;
};

// Output addressing:
//   off(r, c) = (r / rb2)*rh2 + ((r % rb2) / rb)*rh + (r % rb)*rl
//             + (c / cb)*ch + (c % cb)*cl
struct OutMap {
  int64_t rb, rh, rl;
  int64_t cb, ch, cl;
  int64_t rb2, rh2;
};

enum EpiAct : int { kActNone = 0, kActRelu = 1, kActSigmoid = 2 };

struct EngineParams {
  CUtensorMap map_a;  // 64-byte aligned inside the param block
  CUtensorMap map_b;
  // compact-epilogue TMA stores (set by launch_engine when the output is a blocked
  // [outer][cols / 64][out_rb][64] bf16 layout): 3-d map (64, out_rb, outer * cols / 64),
  // box (64, 32, 1); a warp's 32 x 64 staging tile leaves in one store (the generic flush
  // where its rows cross an outer block)
  CUtensorMap map_out;
  int32_t tma_out;
  int32_t out_rb;
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
  const void* sgd_src;   // if set: sgd_w = sgd_src - lr * out (double-buffered weights, staged path)
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
  // split-K into slices: when k_splits > 1 and split_ws == null, split sp
  // writes its partial result (plain store, no epilogue ops) to out + sp *
  // split_slice elements; a separate deterministic reduction sums them.
  int64_t split_slice;
  // stride-2 1x1 backward-data scatter: besides out[off], zero
  // out[off + zf_w], out[off + zf_h], out[off + zf_w + zf_h] (bf16 output)
  int64_t zf_w, zf_h;
  // aux gradient output (fused top-layer ReLU mask): aux_out = aux_in * (out > 0),
  // bf16 in the output layout; column sums (colsum_ws) then see aux_out
  const void* aux_in;
  void* aux_out;
  int32_t debug_flags;  // bit0: skip MMA, bit1: skip TMA, bit2: no k rotation (diagnostics)
  // grouped launches: the B operand does not depend on this problem's dependencies
  // (e.g. layer weights): each producer issues its first B block before waiting for them
  int32_t b_first;
  // diagnostics: per-CTA %globaltimer stamps [blockIdx.x][8]:
  // 0 entry, 1 setup done, 2 first TMA issued, 3 first full-barrier passed (MMA),
  // 4 last MMA committed, 5 epilogue got accumulator, 6 epilogue done, 7 exit
  unsigned long long* debug_ts;
};


constexpr int kMaxProbs = 12;
constexpr int kMaxDeps = 3;
constexpr int kCounterStride = 65;  // per problem: 64 row-block counters + 1 whole-problem counter

// Tile schedule of a grouped launch: problem q owns work units
// [tile_begin[q], tile_begin[q+1]); a tile of q waits until, for every
// dependency d, counters[dep_prob][mb] (dep_mode 0: the same 256-row block)
// or counters[dep_prob][64] (dep_mode 1: the whole problem) shows all tiles done,
// or (dep_mode 2) each k-step only for the 64-column chunk it reads (chunk_counters).
struct GroupSched {
  int32_t n_probs;
  int32_t tile_begin[kMaxProbs + 1];
  int32_t dep_prob[kMaxProbs][kMaxDeps];  // -1: none
  int32_t dep_mode[kMaxProbs][kMaxDeps];
  // [n_probs][kCounterStride] + 1 exit counter, all zero at launch; the last CTA to finish
  // zeroes them again, so back-to-back launches need no memset
  unsigned* counters;
  // dep_mode 2 (64-column chunks): k-step s of a tile in row block mb, CTA rank r, waits only
  // for the 64 columns [64 s, 64 s + 64) of the same 128 rows of the dependency, i.e. for
  //   chunk_counters[((dep_prob * chunk_mb + mb) * 2 + r) * chunk_n + s] == chunk_target
  // (the epilogue warps that store those rows x columns each add one after their stores).  Zero at launch, re-zeroed by the last CTA like `counters`; null: no chunk deps.
  unsigned* chunk_counters;
  int32_t chunk_mb, chunk_n;
  int32_t chunk_target;  // epilogue-warp arrivals per chunk: 8 for BN=128 pairs (both column quarters)
};

struct EngineGroup {
  EngineParams probs[kMaxProbs];
  GroupSched sched;
};

}  // namespace brk
