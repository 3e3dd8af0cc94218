// brk_mlp.h — the fused MLP training step (BASELINE config 2) as one lean
// persistent tcgen05 launch (brk_mlp.cu).
//
// Same schedule as the grouped engine (brk_engine.h: GroupSched, one CTA pair
// per 256 x 128 output tile, tile-level / 64-column-chunk dependency counters),
// but every problem is one of five fixed MLP passes, so the kernel carries only
// their epilogues: each is a short, fully specialised code path (the grouped
// engine's general epilogue executed ~63 KB of code per step, twice the SM's
// instruction cache) whose outputs leave through TMA stores from a per-warp
// staging tile and whose side operands (output gradient, ReLU mask, old
// weights) arrive by TMA before the accumulator does.
#pragma once
#include <cstdint>
#include <cuda.h>

#include "brk_engine.h"

namespace brk {

enum MlpKind : int32_t {
  kMlpFwd = 0,      // y = relu(acc + bias)                                  -> out (bf16)
  kMlpFwdTop = 1,   // y = relu(acc + bias) -> out; dz = dy * (y > 0) -> aux, column sums of dz
  kMlpBwd = 2,      // dz = acc * (mask > 0) -> out (bf16), column sums of dz
  kMlpBwdPlain = 3, // dx = acc -> out (bf16)
  kMlpUpd = 4,      // dW = acc -> out (fp32); w_next = w - lr dW -> aux; db = sum of partials
};

// One problem of the step (A: the CTA's 128-row block, B: its 64-row block, in the blocked FC
// layouts of brk_fc.cu).  fp32 storage (TF32 step): every map is fp32 and every side / output
// box is 32 columns (128 B) wide, two per warp.
struct MlpProb {
  CUtensorMap map_a;
  CUtensorMap map_b;
  CUtensorMap map_out;  // bf16 activations: box (64, 32, 1, 1); fp32 (dW, TF32 step): box (32, 32, 1, 1)
  CUtensorMap map_in;   // dy (top) / ReLU mask (bwd) / old weights (upd): box (64, 32, 1, 1)
  CUtensorMap map_aux;  // dz_L (top) / new weights (upd): box (64, 32, 1, 1)
  int32_t kind;         // MlpKind
  int32_t m_tiles, n_tiles, k_steps;
  // operand box of k-step s for row block `row`: coordinate d = rc[d] * row + k0[d] * d0 +
  // k1[d] * d1 with (d0, d1) = (s, 0) for bf16 (4-d maps) and (s % 2, s / 2) for TF32 (5-d
  // maps of 32-element halves, brk_fc.cu split_layout)
  int32_t a_rc[5], a_k0[5], a_k1[5];
  int32_t b_rc[5], b_k0[5], b_k1[5];
  int32_t a_mn, b_mn;   // MN-major operand (UMMA descriptor / idesc)
  int32_t cols;         // output columns (row length of colsum_ws)
  int32_t has_in;       // the epilogue loads map_in
  int32_t has_aux;      // the epilogue stores map_aux
  int32_t b_first;      // B does not depend on this problem's dependencies
  const float* bias;
  float* colsum_ws;     // [rows / 32][cols] column sums of the stored gradient
  const float* db_partials;  // upd: [db_parts][cols] partials to reduce into db_out
  int32_t db_parts;
  float* db_out;
  float* bias_sgd;      // upd: bias -= lr * db (may be null)
  float lr;
};

constexpr int kMaxListPairs = 80;
constexpr int kMaxListUnits = 2048;

struct MlpGroup {
  MlpProb probs[kMaxProbs];
  GroupSched sched;
  // diagnostics build only (BRK_DIAG): per-CTA, per-local-tile %globaltimer stamps
  // [blockIdx.x][16][8], slots as in the grouped engine (brk_engine.cu BRK_TT)
  unsigned long long* debug_ts;
  // tuning (BRK_MLP_FLAGS): bit0 per-tile k-step rotation, bit1 no writer-side proxy fence,
  // bit2 relaxed dependency polling + one acquire fence, bit3 release (not relaxed) chunk counters
  int32_t flags;
  // CTAs per cluster: 2 (one pair) or 4 (two pairs sharing the A operand by TMA multicast)
  int32_t cluster;
  int32_t tf32;  // fp32 storage, kind::tf32 MMAs (k-steps of 32 elements)
  // list schedule (cluster == 2): CTA pair c runs units list[list_off[c] .. list_off[c+1]) in
  // that order (each list increasing: every unit waits only on units of lower index, so the
  // lists cannot deadlock); list_len == 0: round robin (pair c runs c, c + pairs, ...)
  int32_t list_len;
  int16_t list_off[kMaxListPairs + 1];
  int16_t list[kMaxListUnits];
};

int launch_mlp_group(const MlpGroup& G, cudaStream_t stream);
// list-schedule the group's work units over `pairs` CTA pairs (fills list / list_off / list_len;
// leaves list_len = 0 when the units do not fit the table)
void mlp_list_schedule(MlpGroup& G, int pairs);

}  // namespace brk
