// brk_engine.cu — persistent, warp-specialised tcgen05 BRGEMM engine (see brk_engine.h).
//
// Roles:
//   warps 0..7  epilogue: tcgen05.ld the accumulator (TMEM lane = output row),
//               fuse alpha/beta, bias, activation, ReLU-mask, the SGD update
//               and bias-gradient column sums, and store.  Warp e drains TMEM
//               lane quarter e%4, column half e/4 (two warps per SM
//               sub-partition: the epilogue is issue-bound, not TMEM-bound).
//               Two TMEM accumulators let the epilogue of one tile overlap the
//               MMAs of the next.
//   warp 8      MMA issuer: one elected thread issues tcgen05.mma into a TMEM
//               accumulator that stays resident for the whole batch reduce;
//               tcgen05.commit frees ring stages and publishes finished tiles.
//   warps 9..   kProducers TMA producers: producer j streams the (A_s, B_s)
//               boxes of every k-step g = j (mod kProducers) of the batch list
//               into the kStages ring.  Several issuing warps are required:
//               one warp keeps only ~one box in flight (measured with
//               brk_diag_tma_bw: 1 warp 12 B/clk/SM, 4 warps 44 B/clk/SM).
//               kStages % kProducers == 0, so a slot is always refilled by the
//               warp that filled it last and the parity waits cannot alias.
//
// kPair = true runs a CTA pair (cluster of 2, tcgen05 cta_group::2): the tile
// is 256 x BN, each CTA stages its own 128 rows of A and BN/2 rows of B, the
// leader CTA issues M=256 MMAs that read both CTAs' shared memory, and each
// CTA drains its own 128-lane half of the accumulator.  Per-SM shared-memory
// operand traffic per MMA halves versus the single-CTA 128 x BN tile, which is
// what lets the tensor pipe run at full rate in SS mode.
//
// Split-K (k_splits > 1) cuts each tile's batch list into contiguous chunks
// run by different CTAs; partial accumulators go through an fp32 workspace
// and the last-arriving chunk sums them in chunk order (deterministic).
//
// Launched with programmatic stream serialisation (PDL): the prologue
// (barrier init, TMEM alloc, tensor-map prefetch) overlaps the previous
// kernel; griddepcontrol.wait precedes every global-memory access.
#include <cstdio>
#include <cstdlib>

#include "brk_engine.h"
#include "brk_internal.h"
#include "brk_ptx.cuh"
#include "brk_sched.cuh"
#include "brk_tma_host.h"

namespace brk {
namespace {

constexpr int kTileABytes = kEngineBM * 128;  // 128 rows x 128 B per CTA
constexpr int kEpiWarps = 8;
constexpr int kEpiThreads = kEpiWarps * 32;

template <int BN, bool kPair>
struct EngineCfg {
  static constexpr int kBRows = kPair ? BN / 2 : BN;  // B rows staged per CTA
  static constexpr int kTileBBytes = kBRows * 128;
  static constexpr int kStageBytes = kTileABytes + kTileBBytes;
  // epilogue staging: one 32-row x 128 B tile per epilogue warp (coalesced stores)
  static constexpr int kEpiStageBytes = kEpiWarps * 4096;  // one staging tile per epilogue warp
  static constexpr int kAvail = 232448 - 1024 - 256 - kEpiStageBytes;  // 227 KB opt-in max
  // ring depth: as many stages as fit (<= 7), one producer warp each
  static constexpr int kFit = kAvail / kStageBytes > 7 ? 7 : kAvail / kStageBytes;
  static constexpr int kStages = kFit;
  // accumulator buffers in TMEM: four when they fit the 512 columns (BN <= 128), so the MMA can
  // run up to three tiles ahead of the epilogue (short tiles: 1x1 convs with one or two k-steps)
  static constexpr int kAcc = 4 * BN <= 512 ? 4 : 2;
  static constexpr int kTmemCols = kAcc * BN;
  static constexpr int kSmem = kStages * kStageBytes + kEpiStageBytes + 1024 + 256;
  // 7 producer warps: a TMA-issuing warp keeps about one box in flight (~1 box
  // per ~930 clk of latency, profiles/r01_tma_sweep.txt), so the per-SM operand
  // rate scales with the number of issuing warps.  8 epilogue + 1 MMA + 7
  // producer warps = 4 warpgroups; setmaxnreg moves registers from the
  // producer/MMA warpgroups (56) to the epilogue warpgroups (192).
  // one producer per stage (a producer refills only its own stage, so the
  // mbarrier parity waits cannot alias); warps beyond 8 + 1 + kStages idle
  static constexpr int kProducers = kStages;
  static constexpr int kMmaWarp = kEpiWarps;
  static constexpr int kThreads = 16 * 32;  // 4 warpgroups (setmaxnreg is per warpgroup)
  static constexpr int kColsPerWarp = BN >= 64 ? BN / 2 : BN;  // column half per epilogue warp
};

template <bool kPair>
__device__ __forceinline__ void issue_operand(const CUtensorMap* map, const OperandCoords& oc, int rowblk, int s,
                                              uint8_t* dst, uint64_t* bar) {
  const int d0 = s % oc.kdiv0, t = s / oc.kdiv0;
  const int d1 = t % oc.kdiv1, t2 = t / oc.kdiv1;
  const int d2 = oc.kdiv2 > 0 ? t2 % oc.kdiv2 : t2, d3 = oc.kdiv2 > 0 ? t2 / oc.kdiv2 : 0;
  int32_t cs[5];
#pragma unroll
  for (int d = 0; d < 5; ++d)
    cs[d] = oc.base[d] + oc.rc[d] * rowblk + oc.kc[0][d] * d0 + oc.kc[1][d] * d1 + oc.kc[2][d] * d2 + oc.kc[3][d] * d3;
  uint16_t off[3] = {0, 0, 0};
  if (oc.kind != 0 && oc.kind != 5) {
    // implicit-GEMM pixel walk: first pixel of this box -> (n, p, q)
    int pix = oc.kind == 1 ? rowblk * kEngineBM : s * 64;
    if (pix >= oc.total_pix) pix = oc.total_pix - 1;  // rows-side only (masked rows)
    const int pq = oc.P * oc.Q;
    const int n = pix / pq, rem = pix - n * pq;
    const int pp = rem / oc.Q, q = rem - pp * oc.Q;
    cs[1] += q * oc.cstride - oc.pad_w;
    cs[2] += pp * oc.cstride - oc.pad_h;
    cs[3] += n;
    if (oc.kind == 1) {
      off[0] = static_cast<uint16_t>(oc.ok[0][0] * d0 + oc.ok[0][1] * d1 + oc.ok[0][2] * d2);
      off[1] = static_cast<uint16_t>(oc.ok[1][0] * d0 + oc.ok[1][1] * d1 + oc.ok[1][2] * d2);
    }
  }
  for (int l = 0; l < oc.n_loads; ++l) {
    int32_t c[5];
#pragma unroll
    for (int d = 0; d < 5; ++d) c[d] = cs[d] + oc.lc[d] * l;
    uint8_t* p = dst + l * oc.load_bytes;
    if (oc.kind == 5) {
      // TF32 weight update in tile mode: load l of the row block is the 32-channel atom
      // a = ((rs * atom_cb + c_b) * 2 + half); its box is the k-step's pixel block shifted by the
      // tap (r, s), in plane n * C_b + c_b, at channel offset 32 * half
      const int a = rowblk * oc.n_loads + l, a2 = a >> 1;
      const int rs = a2 / oc.atom_cb, r = rs / oc.atom_s;
      c[0] += (a & 1) * 32;
      c[1] += rs - r * oc.atom_s;
      c[2] += r;
      c[3] += a2 - rs * oc.atom_cb;
    } else if (oc.kind != 0) {
      if (oc.kind == 2) {
        const int atom = rowblk * oc.n_loads + l;
        const int rs = atom / oc.atom_cb;
        c[4] += atom - rs * oc.atom_cb;
        const int r = rs / oc.atom_s;
        off[0] = static_cast<uint16_t>(rs - r * oc.atom_s);
        off[1] = static_cast<uint16_t>(r);
      }
      tma_load_im2col5<kPair>(p, map, bar, c, off);
      continue;
    }
    if constexpr (kPair) {
      switch (oc.ndims) {
        case 2: { const int32_t cc[2] = {c[0], c[1]}; tma_load_pair<2>(p, map, bar, cc); break; }
        case 3: { const int32_t cc[3] = {c[0], c[1], c[2]}; tma_load_pair<3>(p, map, bar, cc); break; }
        case 4: { const int32_t cc[4] = {c[0], c[1], c[2], c[3]}; tma_load_pair<4>(p, map, bar, cc); break; }
        default: { tma_load_pair<5>(p, map, bar, c); break; }
      }
    } else {
      switch (oc.ndims) {
        case 2: { const int32_t cc[2] = {c[0], c[1]}; tma_load<2>(p, map, bar, cc); break; }
        case 3: { const int32_t cc[3] = {c[0], c[1], c[2]}; tma_load<3>(p, map, bar, cc); break; }
        case 4: { const int32_t cc[4] = {c[0], c[1], c[2], c[3]}; tma_load<4>(p, map, bar, cc); break; }
        default: { tma_load<5>(p, map, bar, c); break; }
      }
    }
  }
}

// smem descriptor for the MMA sub-step kk (32 bytes of K) of one operand tile
template <bool kTF32>
__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int mn_major, int kk) {
  if (!mn_major) {
    // K-major, 128B swizzle: 8-row groups 1024 B apart; K advance = 32 B.
    return make_smem_desc(base + kk * 32, 16, 1024, kSwizzle128B);
  }
  // MN-major: atom = 128 B of MN x BK rows (BK = 64 bf16 / 32 TF32 K-rows).  bf16: 128B
  // swizzle, 8 K-rows = 1024 B (SBO).  TF32 requires the 32 B-chunk 128B swizzle
  // (SWIZZLE_128B_BASE32B, TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) whose K groups are
  // 4 rows = 512 B; one MMA (K = 8) spans two of them.
  constexpr uint32_t kRowsPerMma = kTF32 ? 8 : 16;
  constexpr uint32_t kAtomBytes = (kTF32 ? 32 : 64) * 128;  // BK rows x 128 B
  if constexpr (kTF32) return make_smem_desc(base + kk * kRowsPerMma * 128, kAtomBytes, 512, kSwizzle128B32);
  return make_smem_desc(base + kk * kRowsPerMma * 128, kAtomBytes, 1024, kSwizzle128B);
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// grouped launches: per-CTA, per-local-tile stamps [blockIdx.x][16 tiles][4]:
// 0 producer 0 dependencies satisfied, 1 MMA first stage full, 2 MMA last commit, 3 epilogue released,
// 4 epilogue got the accumulator, 5 stores issued, 6 proxy fence + barrier passed
// (compiled only into the diagnostics build, `make diag` -> libbrk_sm100_diag.so, selected
//  with BRK_LIB: the stamps cost ~50 instructions per epilogue tile)
#ifdef BRK_DIAG
#define BRK_TT(tile, slot)                                                                      \
  do {                                                                                          \
    if (gs != nullptr && P[0].debug_ts != nullptr && (tile) < 16)                               \
      P[0].debug_ts[(blockIdx.x * 16 + (tile)) * 8 + (slot)] = gtimer();                         \
  } while (0)
#define BRK_TS(slot)                                                              \
  do {                                                                            \
    if (gs == nullptr && P[0].debug_ts != nullptr) P[0].debug_ts[blockIdx.x * 16 + (slot)] = gtimer();   \
  } while (0)
#else
#define BRK_TT(tile, slot) \
  do {                     \
  } while (0)
#define BRK_TS(slot) \
  do {               \
  } while (0)
#endif

// diagnostics (BRK_DIAG, single-problem launches): per-CTA sums of clock64 spent waiting,
// written after the stamps at debug_ts[gridDim.x * 16 + blockIdx.x * 8 + slot]:
// 0 MMA waits for a free accumulator, 1 MMA waits for operands, 2 epilogue waits for the
// accumulator, 3 epilogue busy (accumulator -> tile done), 4 producer 0 waits for a free stage
#ifdef BRK_DIAG
#define BRK_CLK(var) const long long var = clock64()
#define BRK_ACC(slot, t0)                                                                          \
  do {                                                                                             \
    if (gs == nullptr && P[0].debug_ts != nullptr)                                                 \
      atomicAdd(&P[0].debug_ts[gridDim.x * 16 + blockIdx.x * 8 + (slot)],                          \
                static_cast<unsigned long long>(clock64() - (t0)));                                \
  } while (0)
#else
#define BRK_CLK(var) \
  do {               \
  } while (0)
#define BRK_ACC(slot, t0) \
  do {                    \
  } while (0)
#endif

__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Warp reduce-scatter: lane l ends with f[0] = sum over the 32 lanes of column l.
__device__ __forceinline__ float warp_column_sum(float (&f)[32], int lane) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int j = 0; j < off; ++j) {
      const float send = upper ? f[j] : f[j + off];
      const float keep = upper ? f[j + off] : f[j];
      f[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return f[0];
}

// Fused epilogue of one 32-column chunk of one row.  `f` holds alpha*acc;
// `bias_lane` is bias[col0 + lane] (broadcast by shuffle).  All 32 lanes of
// the warp must call it (shuffles).
__device__ __forceinline__ void epilogue_finish(const EngineParams& p, float (&f)[32], bool valid, int64_t off,
                                                int col0, int warp_row0, int lane, float bias_lane) {
  if (p.bias != nullptr && !(p.debug_flags & 16)) {
#pragma unroll
    for (int j = 0; j < 32; ++j) f[j] += __shfl_sync(0xffffffffu, bias_lane, j);
  }
  if (valid) {
    if (p.beta != 0.0f) {
      if (p.out_bf16) {
        const __nv_bfloat16* src = static_cast<const __nv_bfloat16*>(p.out) + off;
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] += p.beta * __bfloat162float(src[j]);
      } else {
        const float* src = static_cast<const float*>(p.out) + off;
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] += p.beta * src[j];
      }
    }
    if (p.act == kActRelu) {
#pragma unroll
      for (int j = 0; j < 32; ++j) f[j] = fmaxf(f[j], 0.0f);
    } else if (p.act == kActSigmoid) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float e = __expf(-fabsf(f[j]));
        const float r = __fdividef(1.0f, 1.0f + e);
        f[j] = f[j] >= 0.0f ? r : e * r;
      }
    }
    if (p.mask != nullptr) {
      const uint4* mk = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.mask) + off);
      uint4 w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = mk[q];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w[q]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 m2 = __bfloat1622float2(h[j]);
          f[q * 8 + 2 * j] = m2.x > 0.0f ? f[q * 8 + 2 * j] : 0.0f;
          f[q * 8 + 2 * j + 1] = m2.y > 0.0f ? f[q * 8 + 2 * j + 1] : 0.0f;
        }
      }
    }
    if (p.debug_flags & 8) {
      // diagnostic: skip the output stores (keep the values live)
      float acc = 0.0f;
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += f[j];
      if (acc == 1234.5f) static_cast<float*>(p.out)[off] = acc;
    } else if (p.out_bf16) {
      uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + off);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 w;
        w.x = pack_bf16x2(f[q * 8 + 0], f[q * 8 + 1]);
        w.y = pack_bf16x2(f[q * 8 + 2], f[q * 8 + 3]);
        w.z = pack_bf16x2(f[q * 8 + 4], f[q * 8 + 5]);
        w.w = pack_bf16x2(f[q * 8 + 6], f[q * 8 + 7]);
        dst[q] = w;
      }
      if (p.zf_w != 0) {  // stride-2 scatter: the three skipped input positions get zeros
        const uint4 z = make_uint4(0u, 0u, 0u, 0u);
        uint4* d1 = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + off + p.zf_w);
        uint4* d2 = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + off + p.zf_h);
        uint4* d3 = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + off + p.zf_w + p.zf_h);
#pragma unroll
        for (int q = 0; q < 4; ++q) { d1[q] = z; d2[q] = z; d3[q] = z; }
      }
      if (p.aux_in != nullptr) {
        // fused output-gradient mask: aux_out = aux_in * (out > 0); the column
        // sums (bias gradient of the next pass) then see aux_out
        const uint4* ai = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.aux_in) + off);
        uint4* ao = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.aux_out) + off);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 w = ai[q];
          __nv_bfloat16* h = reinterpret_cast<__nv_bfloat16*>(&w);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float y = __bfloat162float(__float2bfloat16_rn(f[q * 8 + j]));
            const float a = y > 0.0f ? __bfloat162float(h[j]) : 0.0f;
            h[j] = __float2bfloat16_rn(a);
            f[q * 8 + j] = a;
          }
          ao[q] = w;
        }
      } else if (p.colsum_ws != nullptr) {  // column sums see the stored (rounded) values
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] = __bfloat162float(__float2bfloat16_rn(f[j]));
      }
    } else {
      float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.out) + off);
#pragma unroll
      for (int q = 0; q < 8; ++q) dst[q] = make_float4(f[q * 4], f[q * 4 + 1], f[q * 4 + 2], f[q * 4 + 3]);
    }
    if (p.sgd_w != nullptr) {
      uint4* wp = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.sgd_w) + off);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 w = wp[q];
        __nv_bfloat16* h = reinterpret_cast<__nv_bfloat16*>(&w);
#pragma unroll
        for (int j = 0; j < 8; ++j) h[j] = __float2bfloat16_rn(__bfloat162float(h[j]) - p.sgd_lr * f[q * 8 + j]);
        wp[q] = w;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) f[j] = 0.0f;
  }
  if (p.colsum_ws != nullptr) {
    const float s = warp_column_sum(f, lane);
    if (col0 < p.cols && warp_row0 < p.rows)
      p.colsum_ws[static_cast<int64_t>(warp_row0 / 32) * p.cols + col0 + lane] = s;
  }
}

// The epilogue's view of a problem, loaded into registers once per tile: in
// grouped launches every EngineParams field access is an indexed constant-bank
// load, which serialises the epilogue if repeated per element group.
struct EpiView {
  void* out;
  const float* bias;
  const void* mask;
  const void* aux_in;
  void* aux_out;
  float* colsum_ws;
  void* sgd_w;
  const void* sgd_src;
  int64_t zf_w, zf_h;
  float sgd_lr;
  int out_bf16, act, rows, cols;
  __device__ __forceinline__ explicit EpiView(const EngineParams& p)
      : out(p.out), bias(p.bias), mask(p.mask), aux_in(p.aux_in), aux_out(p.aux_out), colsum_ws(p.colsum_ws),
        sgd_w(p.sgd_w), sgd_src(p.sgd_src != nullptr ? p.sgd_src : p.sgd_w), zf_w(p.zf_w), zf_h(p.zf_h), sgd_lr(p.sgd_lr), out_bf16(p.out_bf16), act(p.act),
        rows(p.rows), cols(p.cols) {}
};

__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr)
               : "memory");
  return v;
}

// a[c] for a loop-variant c without dynamic register indexing (rolled epilogue loops)
template <int N>
__device__ __forceinline__ float pick(const float (&a)[N], int c) {
  float v = a[0];
#pragma unroll
  for (int i = 1; i < N; ++i) v = c == i ? a[i] : v;
  return v;
}

// Staged epilogue, part 1: bias, activation on one 32-column chunk of this
// lane's row, written into the warp's staging tile (32 rows x 128 B at the
// shared address `row`; 16 B slot j of row r at slot j ^ (r % 8): conflict-free
// for the row-wise writes here and the segment-wise reads of epilogue_flush).
// bf16: chunk = 4 slots (two chunks fill a 128 B row segment); fp32: 8 slots.
__device__ __forceinline__ void epilogue_stage(const EpiView& p, float (&f)[32], float bias_lane, uint32_t row,
                                               int lane, int slot0) {
  if (p.bias != nullptr) {  // the chunk's 32 bias values: lane j holds column j's (loaded before the accumulator wait)
#pragma unroll
    for (int j = 0; j < 32; ++j) f[j] += __shfl_sync(0xffffffffu, bias_lane, j);
  }
  if (p.act == kActRelu) {
#pragma unroll
    for (int j = 0; j < 32; ++j) f[j] = fmaxf(f[j], 0.0f);
  } else if (p.act == kActSigmoid) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float e = __expf(-fabsf(f[j]));
      const float r = __fdividef(1.0f, 1.0f + e);
      f[j] = f[j] >= 0.0f ? r : e * r;
    }
  }
  if (p.out_bf16) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      sts128(row + (((slot0 + q) ^ (lane & 7)) << 4),
             make_uint4(pack_bf16x2(f[q * 8 + 0], f[q * 8 + 1]), pack_bf16x2(f[q * 8 + 2], f[q * 8 + 3]),
                        pack_bf16x2(f[q * 8 + 4], f[q * 8 + 5]), pack_bf16x2(f[q * 8 + 6], f[q * 8 + 7])));
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      sts128(row + ((q ^ (lane & 7)) << 4),
             make_uint4(__float_as_uint(f[q * 4]), __float_as_uint(f[q * 4 + 1]), __float_as_uint(f[q * 4 + 2]),
                        __float_as_uint(f[q * 4 + 3])));
  }
}

// Staged epilogue, part 2: write the staged 32 x 128 B tile as coalesced 16 B
// stores (kLanes lanes per row segment: 8 for 128 B, 4 for 64 B) instead of one
// 16 B store per row per lane.  roff is this lane's row offset (element), ok
// the row validity bits, coff the segment's column offset.  kFull adds, per
// 16 B element group and still coalesced: the ReLU-derivative mask (bf16
// outputs), the fused output-gradient mask (aux), the SGD update of bf16
// weights (fp32 outputs) and the 32-row column sums (colsum_ws row
// warp_row0 / 32, columns col_seg ..).  All global loads of the segment are
// issued before any is consumed (one latency per flush, not per row).
// Global operands the full flush reads (ReLU mask / aux gradient for bf16
// outputs, SGD weights for fp32 outputs) do not depend on the accumulator:
// they are fetched for the first segments before the epilogue waits for it.
__device__ __forceinline__ const void* flush_src(const EpiView& p) {
  if (p.out_bf16) return p.mask != nullptr ? p.mask : p.aux_in;
  // fp32 outputs: the fp32 ReLU mask (TF32 backward-data) or the bf16 weights of the fused SGD
  return p.mask != nullptr ? p.mask : (p.sgd_w != nullptr ? p.sgd_src : nullptr);
}
// The 16 B flush operand of destination element e: 8 bf16 (bf16 outputs), 4 fp32 (fp32 mask),
// or 4 bf16 widened into the low half (bf16 SGD weights of an fp32 weight gradient).
__device__ __forceinline__ uint4 flush_load(const EpiView& p, const void* src, int64_t e, bool streaming) {
  if (p.out_bf16) {
    const uint4* q = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(src) + e);
    return streaming ? __ldcs(q) : *q;
  }
  if (p.mask != nullptr) return *reinterpret_cast<const uint4*>(static_cast<const float*>(src) + e);
  const uint2 w2 = *reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(src) + e);
  return make_uint4(w2.x, w2.y, 0u, 0u);
}
template <int kLanes>
__device__ __forceinline__ void epilogue_prefetch(const EpiView& p, int64_t roff, uint32_t ok, int64_t coff,
                                                  int lane, uint4 (&pre)[8]) {
  const void* src = flush_src(p);
  if (src == nullptr) return;
  constexpr int kRowsPer = 32 / kLanes;
  const int s = lane & (kLanes - 1);
  const int esz = p.out_bf16 ? 2 : 4;
#pragma unroll
  for (int i = 0; i < kLanes; ++i) {
    const int r = kRowsPer * i + lane / kLanes;
    const int64_t ro = __shfl_sync(0xffffffffu, roff, r);
    if (!((ok >> r) & 1u)) continue;
    const int64_t e = ro + coff + s * (16 / esz);
    pre[i] = flush_load(p, src, e, true);
  }
}

template <int kLanes, bool kFull>
__device__ __forceinline__ void epilogue_flush(const EpiView& p, uint32_t stage, int64_t roff, uint32_t ok,
                                               int64_t coff, int lane, int warp_row0 = 0, int col_seg = 0,
                                               const uint4* pre = nullptr) {
  __syncwarp();
  constexpr int kRowsPer = 32 / kLanes;
  const int s = lane & (kLanes - 1);
  const int esz = p.out_bf16 ? 2 : 4;
  uint8_t* out = static_cast<uint8_t*>(p.out);
  int64_t eo[kLanes];
  uint4 v[kLanes];
  uint4 ld[kLanes];
  bool okr[kLanes];
#pragma unroll
  for (int i = 0; i < kLanes; ++i) {
    const int r = kRowsPer * i + lane / kLanes;
    eo[i] = __shfl_sync(0xffffffffu, roff, r) + coff + s * (16 / esz);
    v[i] = lds128(stage + r * 128 + ((s ^ (r & 7)) << 4));
    okr[i] = (ok >> r) & 1u;
  }
  if (kFull && pre != nullptr) {
#pragma unroll
    for (int i = 0; i < kLanes; ++i) ld[i] = pre[i];
  } else if (kFull) {
    const void* src = flush_src(p);
    if (src != nullptr) {
#pragma unroll
      for (int i = 0; i < kLanes; ++i) {
        if (!okr[i]) continue;
        ld[i] = flush_load(p, src, eo[i], false);
      }
    }
  }
  // One short loop per feature (branch outside, rows inside): the code size is
  // the sum of the features, not their product, so the epilogue stays in the
  // instruction cache.
  float cs[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  // masks as packed bf16x2 ops (v * (m > 0): exact, one compare + one multiply per pair —
  // a quarter of the unpack / select / repack code, which is fetched cold once per SM)
  const __nv_bfloat162 zero2 = __float2bfloat162_rn(0.0f);
  if (kFull && p.out_bf16 && p.mask != nullptr) {
#pragma unroll
    for (int i = 0; i < kLanes; ++i) {
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v[i]);
      const __nv_bfloat162* mh = reinterpret_cast<const __nv_bfloat162*>(&ld[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) h[j] = __hmul2(h[j], __hgt2(mh[j], zero2));
    }
  }
  if (kFull && !p.out_bf16 && p.mask != nullptr) {  // fp32 outputs (TF32 path): v * (mask > 0)
#pragma unroll
    for (int i = 0; i < kLanes; ++i) {
      float* f4 = reinterpret_cast<float*>(&v[i]);
      const float* m4 = reinterpret_cast<const float*>(&ld[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) f4[j] = m4[j] > 0.0f ? f4[j] : 0.0f;
    }
  }
#pragma unroll
  for (int i = 0; i < kLanes; ++i)
    if (okr[i]) *reinterpret_cast<uint4*>(out + eo[i] * esz) = v[i];
  if (kFull && p.out_bf16 && p.aux_in != nullptr) {  // (aux only on forward outputs, never with mask)
#pragma unroll
    for (int i = 0; i < kLanes; ++i) {
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v[i]);
      __nv_bfloat162* ah = reinterpret_cast<__nv_bfloat162*>(&ld[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) ah[j] = __hmul2(ah[j], __hgt2(h[j], zero2));
      if (okr[i]) *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.aux_out) + eo[i]) = ld[i];
      v[i] = ld[i];  // column sums of the gradient
    }
  }
  if (kFull && !p.out_bf16 && p.sgd_w != nullptr) {
#pragma unroll
    for (int i = 0; i < kLanes; ++i) {
      const float4 f4 = *reinterpret_cast<const float4*>(&v[i]);
      const __nv_bfloat162* wo = reinterpret_cast<const __nv_bfloat162*>(&ld[i]);
      const float2 w0 = __bfloat1622float2(wo[0]), w1 = __bfloat1622float2(wo[1]);
      const __nv_bfloat162 n0 = __floats2bfloat162_rn(w0.x - p.sgd_lr * f4.x, w0.y - p.sgd_lr * f4.y);
      const __nv_bfloat162 n1 = __floats2bfloat162_rn(w1.x - p.sgd_lr * f4.z, w1.y - p.sgd_lr * f4.w);
      if (okr[i])
        *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(p.sgd_w) + eo[i]) =
            make_uint2(*reinterpret_cast<const uint32_t*>(&n0), *reinterpret_cast<const uint32_t*>(&n1));
    }
  }
  if (kFull && p.colsum_ws != nullptr) {
#pragma unroll
    for (int i = 0; i < kLanes; ++i) {
      if (!okr[i]) continue;
      if (p.out_bf16) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 c2 = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(&v[i])[j]);
          cs[2 * j] += c2.x;
          cs[2 * j + 1] += c2.y;
        }
      } else {
        const float4 f4 = *reinterpret_cast<const float4*>(&v[i]);
        cs[0] += f4.x; cs[1] += f4.y; cs[2] += f4.z; cs[3] += f4.w;
      }
    }
  }
  if (p.zf_w != 0) {
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int i = 0; i < kLanes; ++i) {
      if (!okr[i]) continue;
      uint8_t* dst = out + eo[i] * esz;
      *reinterpret_cast<uint4*>(dst + p.zf_w * 2) = z;
      *reinterpret_cast<uint4*>(dst + p.zf_h * 2) = z;
      *reinterpret_cast<uint4*>(dst + (p.zf_w + p.zf_h) * 2) = z;
    }
  }
  if (kFull && p.colsum_ws != nullptr) {
#pragma unroll
    for (int off = kLanes; off < 32; off <<= 1)
#pragma unroll
      for (int j = 0; j < 8; ++j) cs[j] += __shfl_xor_sync(0xffffffffu, cs[j], off);
    const int per = p.out_bf16 ? 8 : 4;  // columns per 16 B group
    if (lane < kLanes && warp_row0 < p.rows) {
      float* dst = p.colsum_ws + static_cast<int64_t>(warp_row0 / 32) * p.cols + col_seg + s * per;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < per) dst[j] = cs[j];
    }
  }
  __syncwarp();
}

// Work unit u of a launch -> (problem, tile index t, split sp).  Single-problem
// launches (gs == null) order tiles column-block-major (mb fastest); grouped
// launches order each problem row-major (nb fastest) so that the tiles of one
// row block finish together and release the dependent problem's row block early.
// nsp = the batch-list splits of the unit's problem (grouped problems are not split).
__device__ __forceinline__ void locate(const EngineParams* P, const GroupSched* gs, int u, int splits, int& prob,
                                       int& mb, int& nb, int& t, int& sp, int& nsp) {
  if (gs == nullptr) {
    prob = 0;
    nsp = splits;
    t = u / splits;
    sp = u - t * splits;
    mb = t % P[0].m_tiles;
    nb = t / P[0].m_tiles;
    return;
  }
  prob = 0;
  while (prob + 1 < gs->n_probs && u >= gs->tile_begin[prob + 1]) ++prob;
  const int rel = u - gs->tile_begin[prob];
  nsp = 1;
  t = rel;
  sp = 0;
  nb = t % P[prob].n_tiles;
  mb = t / P[prob].n_tiles;
}

template <int BN, bool kTF32, bool kPair, bool kFullEpi, bool kGroup>
__device__ __forceinline__ void engine_body(const EngineParams* P, const GroupSched* gs) {
  using Cfg = EngineCfg<BN, kPair>;
  constexpr int kStages = Cfg::kStages;
  constexpr int kMmaWarp = Cfg::kMmaWarp;
  constexpr int kProducers = Cfg::kProducers;
  // BN = 64 compact epilogues: the two epilogue warp groups take alternate tiles and each warp
  // drains all 64 columns of its 32 rows (one x64 TMEM load, one TMA store) instead of every
  // warp draining 32 columns of every tile through 64-byte generic stores
  constexpr bool kAlt = BN == 64 && !kFullEpi && !kGroup;
  constexpr int kCW = kAlt ? 64 : Cfg::kColsPerWarp;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * Cfg::kStageBytes + Cfg::kEpiStageBytes);
  uint64_t* empty = full + kStages;
  constexpr int kAcc = Cfg::kAcc;
  uint64_t* tfull = empty + kStages;  // [kAcc]
  uint64_t* tempty = tfull + kAcc;    // [kAcc]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + kAcc);
  uint32_t* split_flag = tmem_slot + 1;
  uint32_t* deps_seq = tmem_slot + 2;  // grouped launches: tiles whose dependencies producer 0 acquired

  const int warp = warp_id();
  const int lane = threadIdx.x & 31;
  const uint32_t rank = kPair ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int unit0 = kPair ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int n_units = kPair ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
  const EngineParams& p0 = P[0];
  const int splits = (gs == nullptr && p0.k_splits > 1) ? p0.k_splits : 1;
  const int num_work = gs == nullptr ? p0.m_tiles * p0.n_tiles * splits : gs->tile_begin[gs->n_probs];
  const int n_probs = gs == nullptr ? 1 : gs->n_probs;
  if (threadIdx.x == 0) BRK_TS(0);

  if (warp == kMmaWarp + 1 && lane == 0) {
    for (int q = 0; q < n_probs; ++q) {
      tma_prefetch_desc(&P[q].map_a);
      tma_prefetch_desc(&P[q].map_b);
    }
    *deps_seq = 0u;
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < kAcc; ++a) {
      mbar_init(&tfull[a], 1);
      constexpr uint32_t kDrainers = kAlt ? kEpiWarps / 2 : kEpiWarps;  // epilogue warps per tile
      mbar_init(&tempty[a], kPair ? 2 * kDrainers : kDrainers);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) {
    if constexpr (kPair) tmem_alloc_pair(tmem_slot, Cfg::kTmemCols);
    else tmem_alloc(tmem_slot, Cfg::kTmemCols);
  }
  tc_fence_before();
  if constexpr (kPair) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) BRK_TS(1);
  pdl_launch_dependents();  // let the next kernel's prologue start early

  if (warp >= kMmaWarp) asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
  else asm volatile("setmaxnreg.inc.sync.aligned.u32 192;" ::: "memory");

  if (warp > kMmaWarp) {
    // ------------------------------------------------------------ producers
    const int pid = warp - kMmaWarp - 1;
    if (pid < kProducers && elect_one()) {
      pdl_wait();  // inputs are produced by the previous kernel
      int g = 0;  // global k-step counter of this CTA (same sequence as the MMA issuer)
      int ltile = 0;
      for (int u = unit0; u < num_work; u += n_units) {
        int prob, mb, nb, t, sp, nsp;
        locate(P, gs, u, splits, prob, mb, nb, t, sp, nsp);
        const EngineParams& p = P[prob];
        const int ks_per = (p.k_steps + nsp - 1) / nsp;
        const uint32_t bytes = (p.ca.n_loads * p.ca.load_bytes + p.cb.n_loads * p.cb.load_bytes) * (kPair ? 2 : 1);
        // deps are acquired before the first A load of this producer's k-steps (and before
        // its B load unless the problem's B operand is independent of them)
        // (producer 0 polls the counters first thing and publishes; with b_first the
        // others issue their first B block before waiting for that)
        const uint32_t ordinal = static_cast<uint32_t>(ltile + 1);
        // chunk dependencies are acquired per k-step by the producer that loads it; producer 0
        // publishes the tile ordinal (for the epilogue's operands) after its first such acquire
        const bool chunked = gs != nullptr && has_dep_mode(gs, prob, true);
        bool published = !chunked;
        bool deps_pending = gs != nullptr && (!chunked || has_dep_mode(gs, prob, false));
        if (gs != nullptr && pid == 0) {
          wait_deps(gs, P, prob, mb, kPair ? 2 : 1);
          if (!chunked) publish_deps(deps_seq, ordinal);
          deps_pending = false;
        } else if (deps_pending && !p.b_first) {
          wait_published(deps_seq, ordinal, true);
          deps_pending = false;
        }
        if (pid == 0) BRK_TT(ltile, 0);
        ++ltile;
        const int arow = kPair ? mb * 2 + static_cast<int>(rank) : mb;
        const int brow = kPair ? nb * 2 + static_cast<int>(rank) : nb;
        const int s_begin = sp * ks_per;
        const int n_steps = min(p.k_steps, s_begin + ks_per) - s_begin;
        // Rotate the batch-list start per tile so concurrently running tiles read
        // different blocks; the order is fixed per tile (deterministic results).
        const int rot = (p.debug_flags & 4) ? 0 : (mb * 7 + nb * 3) % n_steps;
        int s0 = (pid - g % kProducers + kProducers) % kProducers;  // first step owned by pid
        for (; s0 < n_steps; s0 += kProducers) {
          const int gg = g + s0;
          const int stage = gg % kStages;
          const uint32_t phase = (gg / kStages) & 1;
          const int s = s_begin + (s0 + rot < n_steps ? s0 + rot : s0 + rot - n_steps);
          if (chunked) {  // before the ring wait: the poll latency overlaps the slot becoming free
            wait_chunk(gs, prob, mb, static_cast<int>(rank), s);
            if (pid == 0 && !published) {  // only producer 0 publishes: the ordinal must not go back
              publish_deps(deps_seq, ordinal);
              published = true;
            }
          }
          BRK_CLK(tp0);
          if (p.debug_flags & 256) mbar_wait(&empty[stage], phase ^ 1);
          else mbar_wait_sleep(&empty[stage], phase ^ 1);
          if (pid == 0) BRK_ACC(4, tp0);
          uint8_t* sa = smem + stage * Cfg::kStageBytes;
          uint8_t* sb = sa + kTileABytes;
          if (p.debug_flags & 2) {
            if (leader) mbar_arrive(&full[stage]);
          } else {
            if (leader) mbar_arrive_expect_tx(&full[stage], bytes);
            if (deps_pending) {
              issue_operand<kPair>(&p.map_b, p.cb, brow, s, sb, &full[stage]);
              wait_published(deps_seq, ordinal, true);
              deps_pending = false;
              issue_operand<kPair>(&p.map_a, p.ca, arow, s, sa, &full[stage]);
            } else {
              issue_operand<kPair>(&p.map_a, p.ca, arow, s, sa, &full[stage]);
              issue_operand<kPair>(&p.map_b, p.cb, brow, s, sb, &full[stage]);
            }
          }
          if (gg == 0 && pid == 0) BRK_TS(2);
        }
        if (!published && pid == 0) {  // producer 0 had no k-step of this tile
          wait_chunk(gs, prob, mb, static_cast<int>(rank), s_begin);
          publish_deps(deps_seq, ordinal);
        }
        g += n_steps;
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    // The operand descriptors are built once per tile for stage 0 and advanced by constants (stage: kStageBytes, sub-step kk: 32 B of K or 16 / 8 MN-major
    // K-rows, all in the 16-byte units of the start-address field): building them per MMA from
    // the addresses cost ~100 uniform-datapath instructions per k-step, ~600 cycles of issue
    // against 128 cycles of tensor work at N = 64 (tensor pipe 22 % on the 3x3 / K = 64 conv).
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      const uint32_t s0 = smem_u32(smem);
      for (int u = unit0; u < num_work; u += n_units, ++local) {
        int prob, mb, nb, t, sp, nsp;
        locate(P, gs, u, splits, prob, mb, nb, t, sp, nsp);
        const EngineParams& p = P[prob];
        const uint32_t idesc = make_idesc(kTF32 ? kFmtTF32 : kFmtBF16, kPair ? 256 : kEngineBM, BN,
                                          p.ca.mn_major, p.cb.mn_major);
        const uint64_t a0 = operand_desc<kTF32>(s0, p.ca.mn_major, 0);
        const uint64_t b0 = operand_desc<kTF32>(s0 + kTileABytes, p.cb.mn_major, 0);
        constexpr uint32_t kMnInc = (kTF32 ? 8 : 16) * 128 / 16;
        const uint32_t a_inc = p.ca.mn_major ? kMnInc : 2u, b_inc = p.cb.mn_major ? kMnInc : 2u;
        const bool skip_mma = (p.debug_flags & 1) != 0;
        const int ks_per = (p.k_steps + nsp - 1) / nsp;
        const int s_begin = sp * ks_per;
        const int n_steps = min(p.k_steps, s_begin + ks_per) - s_begin;
        const int acc = local % kAcc;
        BRK_CLK(tw0);
        mbar_wait(&tempty[acc], ((local / kAcc) & 1) ^ 1);
        if (lane == 0) BRK_ACC(0, tw0);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int s = 0; s < n_steps; ++s) {
          BRK_CLK(tf0);
          mbar_wait(&full[stage], phase);
          if (lane == 0) BRK_ACC(1, tf0);
          tc_fence_after();
          if (local == 0 && s == 0 && lane == 0) BRK_TS(3);
          if (s == 0 && lane == 0) BRK_TT(local, 1);
          const bool issuer = elect_one();
          if (!issuer) {
          } else if (skip_mma) {
            if constexpr (kPair) {
              mma_commit_pair(&empty[stage]);
              if (s == n_steps - 1) mma_commit_pair(&tfull[acc]);
            } else {
              mbar_arrive(&empty[stage]);
              if (s == n_steps - 1) mbar_arrive(&tfull[acc]);
            }
          } else {
            const uint64_t so = static_cast<uint64_t>(stage * (Cfg::kStageBytes / 16));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t accum = (s > 0 || kk > 0) ? 1u : 0u;
              const uint64_t ad = a0 + so + kk * a_inc, bd = b0 + so + kk * b_inc;
              if constexpr (kPair) mma_ss_pair<kTF32>(d_tmem, ad, bd, idesc, accum);
              else mma_ss<kTF32>(d_tmem, ad, bd, idesc, accum);
            }
            if constexpr (kPair) {
              mma_commit_pair(&empty[stage]);
              if (s == n_steps - 1) mma_commit_pair(&tfull[acc]);
            } else {
              mma_commit(&empty[stage]);
              if (s == n_steps - 1) mma_commit(&tfull[acc]);
            }
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) BRK_TS(4);
        if (lane == 0) BRK_TT(local, 2);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 0..7)
    pdl_wait();  // outputs may be read by the previous kernel (WAR) — wait before writing
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int chalf = warp >> 2;   // column half this warp drains
    const int cbeg = kAlt ? 0 : chalf * kCW;
    // (draining the first 64-column chunk of a tile with all eight warps before the second —
    //  64 B store segments, two releases per warp — was measured slower: 109.7 vs 102.7 us
    //  per MLP step)
    auto colw = [&](int c) { return cbeg + c * 32; };
    const int row_in_tile = quarter * 32 + lane;
    const uint32_t tempty_leader = kPair ? mapa_shared(smem_u32(&tempty[0]), 0) : 0u;
    const int halves = kPair ? 2 : 1;
    int local = 0;
    for (int u = unit0; u < num_work; u += n_units, ++local) {
      if (kAlt && (local & 1) != chalf) continue;  // the other warp group's tile
      int prob, mb, nb, t, sp, nsp;
      locate(P, gs, u, splits, prob, mb, nb, t, sp, nsp);
      const EngineParams& p = P[prob];
      const EpiView ev(p);
      const int acc = local % kAcc;
      // bias for this warp's columns, one value per lane per 32-column chunk, loaded before
      // the accumulator wait (the staged epilogue broadcasts it with shuffles)
      float bias_r[kCW / 32];
#pragma unroll
      for (int c = 0; c < kCW / 32; ++c) {
        const int col = nb * BN + colw(c) + lane;
        bias_r[c] = (p.bias != nullptr && col < p.cols) ? __ldg(p.bias + col) : 0.0f;
      }
      const uint32_t stage = smem_u32(smem + kStages * Cfg::kStageBytes + warp * 4096);
      const int tile_row0 = kPair ? mb * 256 + static_cast<int>(rank) * 128 : mb * kEngineBM;
      const int row = tile_row0 + row_in_tile;
      const int warp_row0 = tile_row0 + quarter * 32;
      const bool row_ok = row < p.rows;
      // 32-bit index math (rows and block extents < 2^31)
      const uint32_t ur = static_cast<uint32_t>(row);
      const uint32_t q2 = ur / static_cast<uint32_t>(p.om.rb2), rem2 = ur - q2 * static_cast<uint32_t>(p.om.rb2);
      const uint32_t q1 = rem2 / static_cast<uint32_t>(p.om.rb), rem1 = rem2 - q1 * static_cast<uint32_t>(p.om.rb);
      const int64_t roff = static_cast<int64_t>(q2) * p.om.rh2 + static_cast<int64_t>(q1) * p.om.rh +
                           static_cast<int64_t>(rem1) * p.om.rl +
                           (splits > 1 && p.split_ws == nullptr ? sp * p.split_slice : 0);
      const uint32_t tbase = tmem_base + acc * BN + (static_cast<uint32_t>(quarter * 32) << 16);  // + colw(c)
      // Everything the epilogue needs besides the accumulator is set up before waiting for it:
      // row-offset and bias tables in shared memory, and the flush's global operands.
      const bool staged = !kFullEpi || kGroup || (p.beta == 0.0f && p.split_ws == nullptr);
      uint32_t ok_bits = 0;
      constexpr int kSegLanes = kCW == 32 ? 4 : 8;  // bf16 segments of 32 columns are 64 B
      uint4 pre[2][8];
      if (staged && (splits == 1 || p.split_ws == nullptr)) {
        ok_bits = __ballot_sync(0xffffffffu, row_ok);
        if constexpr (kFullEpi) {
          // grouped launches: the prefetched operands (e.g. the ReLU mask) may be produced by
          // earlier problems of this launch, so the epilogue acquires the tile's dependencies too
          if (gs != nullptr && flush_src(ev) != nullptr) wait_published(deps_seq, local + 1, false);
          const int cfirst = nb * BN + cbeg;
          const int seg_cols = (p.out_bf16 && kSegLanes == 8) ? 64 : 32;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int col = cfirst + j * seg_cols;
            if (col - cfirst >= kCW || col >= p.cols) break;
            const int cq = col / static_cast<int>(p.om.cb), cr = col - cq * static_cast<int>(p.om.cb);
            const int64_t coff = static_cast<int64_t>(cq) * p.om.ch + static_cast<int64_t>(cr) * p.om.cl;
            if (ev.out_bf16 && kSegLanes == 4) epilogue_prefetch<4>(ev, roff, ok_bits, coff, lane, pre[j]);
            else epilogue_prefetch<8>(ev, roff, ok_bits, coff, lane, pre[j]);
          }
        }
      }
      BRK_CLK(te0);
      if (p.debug_flags & 256) mbar_wait(&tfull[acc], (local / kAcc) & 1);
      else mbar_wait_sleep(&tfull[acc], (local / kAcc) & 1);
      if (threadIdx.x == 0) BRK_ACC(2, te0);
      BRK_CLK(te1);
      tc_fence_after();
      if (threadIdx.x == 0) BRK_TS(5);
      if (threadIdx.x == 0) BRK_TT(local, 4);
      if (splits == 1 || p.split_ws == nullptr) {
        // column offset maintained incrementally (32 columns never straddle an
        // output block: cb % 32 == 0, host guarantees); TMEM loads are software-
        // pipelined one chunk ahead so the ld latency overlaps the epilogue math.
        const int cfirst = nb * BN + cbeg;
        // plain epilogue: staging tile, and the row offsets each lane stores in epilogue_flush
        // diagnostics (debug_flags & 128): run the chunk loop twice (i-cache cold vs warm timing)
        const int reps = (p.debug_flags & 128) ? 2 : 1;
        // compact epilogue, bf16 output, whole 64-column segments per warp: one x64 TMEM load per
        // segment (one exposed load latency per 64 columns, not per 32), and the accumulator is
        // released to the MMA as soon as its last segment is in registers
        const bool fast = !kFullEpi && !kGroup && kCW % 64 == 0 && p.out_bf16 && reps == 1;
        if constexpr (!kFullEpi && !kGroup && kCW % 64 == 0) {
          if (fast) {
            const bool tma_out = p.tma_out != 0;
#pragma unroll
            for (int sg = 0; sg < kCW / 64; ++sg) {
              uint32_t v[64];
              tmem_ld64(tbase + cbeg + sg * 64, v);
              tmem_ld_wait();
              if (sg == kCW / 64 - 1) {  // the whole accumulator slice is in registers: free it
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                  if constexpr (kPair) mbar_arrive_cluster_relaxed(tempty_leader + acc * 8);
                  else mbar_arrive_relaxed(&tempty[acc]);
                }
              }
              if (p.debug_flags & 512) continue;  // diagnostics: accumulator drained, nothing stored
              if (tma_out) {  // an earlier store may still be reading the staging tile
                if (lane == 0) bulk_wait_read0();
                __syncwarp();
              }
              const int col_seg = nb * BN + cbeg + sg * 64;
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                float f[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[32 * hh + j]);
                epilogue_stage(ev, f, pick(bias_r, 2 * sg + hh), stage + lane * 128, lane, hh ? 4 : 0);
              }
              if (col_seg >= ev.cols || p.out == nullptr) {
                __syncwarp();
              } else if (tma_out && warp_row0 % p.out_rb + 32 <= p.out_rb) {
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                  const int img = warp_row0 / p.out_rb, pix = warp_row0 - img * p.out_rb;
                  tma_store3(&p.map_out, smem + kStages * Cfg::kStageBytes + warp * 4096, 0, pix,
                             img * (p.cols >> 6) + (col_seg >> 6));
                  bulk_commit();
                }
              } else {  // generic coalesced flush (rows crossing an outer block, non-TMA layouts)
                const int sq = col_seg / static_cast<int>(p.om.cb), sr = col_seg - sq * static_cast<int>(p.om.cb);
                epilogue_flush<8, false>(ev, stage, roff, ok_bits,
                                         static_cast<int64_t>(sq) * p.om.ch + static_cast<int64_t>(sr) * p.om.cl,
                                         lane);
              }
            }
          }
        }
        for (int rep = 0; rep < (fast ? 0 : reps); ++rep) {
        int64_t seg_coff = 0;
        int seg_col = 0;
        int seg = 0;  // staged flush index (the first two use prefetched operands)
        // problems without mask / aux / SGD / column sums take the compact store-only flush
        const bool plain_here = ev.mask == nullptr && ev.aux_in == nullptr && ev.sgd_w == nullptr &&
                                ev.colsum_ws == nullptr;
        int cq = cfirst / static_cast<int>(p.om.cb);
        int cr = cfirst - cq * static_cast<int>(p.om.cb);
        uint32_t v[32];
        const bool tma_out = !kFullEpi && !kGroup && kCW % 64 == 0 && p.out_bf16 && p.tma_out;
        if (tma_out && local > 0) {  // the previous tile's last store has read the staging tile
          if (lane == 0) bulk_wait_read0();
          __syncwarp();
        }
        tmem_ld32(tbase + colw(0), v);
        // the full (grouped / fused-feature) epilogue keeps one copy of the chunk body
#pragma unroll(kFullEpi ? 1 : kCW / 32)
        for (int c = 0; c < kCW / 32; ++c) {
          tmem_ld_wait();
          float f[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
          if (kFullEpi && p.alpha != 1.0f) {
#pragma unroll
            for (int j = 0; j < 32; ++j) f[j] *= p.alpha;
          }
          if (c + 1 < kCW / 32) tmem_ld32(tbase + colw(c + 1), v);
          const int col0 = nb * BN + colw(c);
          const int64_t off = roff + static_cast<int64_t>(cq) * p.om.ch + static_cast<int64_t>(cr) * p.om.cl;
          cr += 32;
          if (cr == p.om.cb) { cr = 0; ++cq; }
          if (p.out == nullptr) continue;  // diagnostic: mainloop-only timing
          if (kFullEpi && !kGroup && !staged) {
            if constexpr (kFullEpi && !kGroup) {
              if (threadIdx.x == 0 && c < 2) BRK_TS(8 + 2 * c);
              epilogue_finish(p, f, row_ok && col0 < p.cols, off, col0, warp_row0, lane, bias_r[c]);
              if (threadIdx.x == 0 && c < 2) BRK_TS(9 + 2 * c);
            }
          } else {
            const int64_t coff = off - roff;
            if (threadIdx.x == 0 && c < 2) BRK_TS(8 + 2 * c);
            if (kCW == 32 && p.out_bf16) {  // 64 B row segments
              epilogue_stage(ev, f, pick(bias_r, c), stage + lane * 128, lane, 0);
              if (col0 < ev.cols) epilogue_flush<4, kFullEpi>(ev, stage, roff, ok_bits, coff, lane, warp_row0, col0,
                                                             seg == 0 ? pre[0] : (seg == 1 ? pre[1] : nullptr));
              else __syncwarp();
              ++seg;
            } else {
              const bool second = p.out_bf16 && (c & 1);
              if (!second) { seg_coff = coff; seg_col = col0; }
              if (tma_out && !second && seg > 0) {  // the previous segment's store has read the tile
                if (lane == 0) bulk_wait_read0();
                __syncwarp();
              }
              epilogue_stage(ev, f, pick(bias_r, c), stage + lane * 128, lane, second ? 4 : 0);
              if (!p.out_bf16 || second) {
                if (threadIdx.x == 0 && c < 2) BRK_TS(9 + 2 * c);
                if (col0 >= ev.cols) __syncwarp();
                else if (tma_out && warp_row0 % p.out_rb + 32 <= p.out_rb) {
                  // the staging tile is the 128B-swizzled TMA box: one store of 32 rows x 64 columns
                  // (a warp whose rows cross an outer block takes the generic flush below)
                  fence_proxy_async_smem();
                  __syncwarp();
                  if (lane == 0) {
                    const int img = warp_row0 / p.out_rb, pix = warp_row0 - img * p.out_rb;
                    tma_store3(&p.map_out, smem + kStages * Cfg::kStageBytes + warp * 4096, 0, pix,
                               img * (p.cols >> 6) + (seg_col >> 6));
                    bulk_commit();
                  }
                }
                else if (kFullEpi && !plain_here)
                  epilogue_flush<8, true>(ev, stage, roff, ok_bits, seg_coff, lane, warp_row0, seg_col,
                                          seg == 0 ? pre[0] : (seg == 1 ? pre[1] : nullptr));
                else epilogue_flush<8, false>(ev, stage, roff, ok_bits, seg_coff, lane);
                ++seg;
                }
            }
          }
        }
        tmem_ld_wait();
        if (threadIdx.x == 0) BRK_TS(14 + rep);
        }
        if (!fast) {
          tc_fence_before();
          __syncwarp();
          if (threadIdx.x == 0) BRK_TS(12);
          if (lane == 0) {
            if constexpr (kPair) mbar_arrive_cluster_relaxed(tempty_leader + acc * 8);
            else mbar_arrive_relaxed(&tempty[acc]);
          }
        }
        if (threadIdx.x == 0) BRK_TS(13);
        if constexpr (kGroup && kCW % 64 == 0) {
          // release this warp's 32 rows of each 64-column chunk it stored (dep_mode 2 consumers)
#pragma unroll
          for (int c = 0; c < kCW / 64; ++c)
            release_chunk(gs, prob, mb, static_cast<int>(rank), ((nb * BN + cbeg) >> 6) + c, lane);
        }
      } else if constexpr (kFullEpi && !kGroup) {
        // split-K: park the partial accumulator, last chunk reduces in chunk order
        float* ws_tile = p.split_ws + (static_cast<int64_t>(t) * halves + rank) * splits * (kEngineBM * BN);
        float* mine = ws_tile + static_cast<int64_t>(sp) * (kEngineBM * BN) + row_in_tile * BN + cbeg;
#pragma unroll
        for (int c = 0; c < kCW / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(tbase + c * 32, v);
          tmem_ld_wait();
          float4* d4 = reinterpret_cast<float4*>(mine + c * 32);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            d4[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (kPair) mbar_arrive_cluster_relaxed(tempty_leader + acc * 8);
          else mbar_arrive_relaxed(&tempty[acc]);
        }
        __threadfence();
        named_bar_sync(1, kEpiThreads);
        if (threadIdx.x == 0) {
          const unsigned prev = atomicAdd(&p.split_counters[t * halves + rank], 1u);
          *split_flag = (prev == static_cast<unsigned>(splits - 1)) ? 1u : 0u;
        }
        named_bar_sync(1, kEpiThreads);
        if (*split_flag) {
          __threadfence();
          int64_t cq = (static_cast<int64_t>(nb) * BN + cbeg) / p.om.cb;
          int64_t cr = (static_cast<int64_t>(nb) * BN + cbeg) % p.om.cb;
#pragma unroll
          for (int c = 0; c < kCW / 32; ++c) {
            float f[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) f[j] = 0.0f;
            for (int q = 0; q < splits; ++q) {
              const float4* s4 = reinterpret_cast<const float4*>(ws_tile + static_cast<int64_t>(q) * (kEngineBM * BN) +
                                                                 row_in_tile * BN + cbeg + c * 32);
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 x = __ldcg(s4 + j);
                f[4 * j] += x.x; f[4 * j + 1] += x.y; f[4 * j + 2] += x.z; f[4 * j + 3] += x.w;
              }
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) f[j] *= p.alpha;
            const int col0 = nb * BN + cbeg + c * 32;
            const int64_t off = roff + cq * p.om.ch + cr * p.om.cl;
            cr += 32;
            if (cr == p.om.cb) { cr = 0; ++cq; }
            if (p.out == nullptr) continue;
            epilogue_finish(p, f, row_ok && col0 < p.cols, off, col0, warp_row0, lane, bias_r[c]);
          }
          if (threadIdx.x == 0) p.split_counters[t * halves + rank] = 0u;  // self-reset
        }
      }
      // bias gradient from column-sum partials of a previous pass (+ fused bias SGD)
      if (kFullEpi && p.db_partials != nullptr && mb == 0 && rank == 0 && (kGroup || sp == 0)) {
        if (gs != nullptr) wait_published(deps_seq, local + 1, false);  // partials come from an earlier problem
        // kG thread groups per column, each summing a contiguous run of partials with batched
        // independent loads; the groups' sums meet in shared memory in group order (deterministic)
        constexpr int kG = kEpiThreads / BN > 0 ? kEpiThreads / BN : 1;
        const int c = threadIdx.x % BN, g = threadIdx.x / BN;
        const int col = nb * BN + c;
        float s = 0.0f;
        if (g < kG && col < p.cols) {
          const int per = (p.db_parts + kG - 1) / kG;
          const int q1 = min(p.db_parts, (g + 1) * per);
          for (int q = g * per; q < q1; q += 8) {
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
              v[j] = q + j < q1 ? __ldcg(p.db_partials + static_cast<int64_t>(q + j) * p.cols + col) : 0.0f;
#pragma unroll
            for (int j = 0; j < 8; ++j) s += v[j];
          }
        }
        // each thread parks its sum in its own warp's staging tile (free after the flushes)
        const uint32_t red0 = smem_u32(smem + kStages * Cfg::kStageBytes);
        const uint32_t red = red0 + warp * 4096 + lane * 4;
        if (kG > 1) {
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(red), "f"(s) : "memory");
          named_bar_sync(1, kEpiThreads);
        }
        if (g == 0 && col < p.cols) {
#pragma unroll
          for (int h = 1; h < kG; ++h) {
            float o;
            const int t2 = threadIdx.x + h * BN;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(o) : "r"(red0 + (t2 >> 5) * 4096 + (t2 & 31) * 4) : "memory");
            s += o;
          }
          p.db_out[col] = s;
          if (p.bias_sgd != nullptr) p.bias_sgd[col] -= p.bias_lr * s;
        }
        if (kG > 1) named_bar_sync(1, kEpiThreads);  // staging tiles are reused by the next tile
      }
      if (gs != nullptr) {
        // release this CTA's half of the tile to dependent problems (their TMA reads it)
        if (threadIdx.x == 0) BRK_TT(local, 5);
        asm volatile("fence.proxy.async.global;" ::: "memory");
        named_bar_sync(1, kEpiThreads);
        if (threadIdx.x == 0) BRK_TT(local, 6);
        if (threadIdx.x == 0) {
          __threadfence();
          atomicAdd(gs->counters + prob * kCounterStride + mb, 1u);
          atomicAdd(gs->counters + prob * kCounterStride + kCounterStride - 1, 1u);
          BRK_TT(local, 3);
        }
      }
      if (threadIdx.x == 0) BRK_TS(6);
      if (threadIdx.x == 0) BRK_ACC(3, te1);
    }
    if (!kFullEpi && !kGroup && lane == 0) bulk_wait0();  // TMA stores done before the CTA exits
  }
  tc_fence_before();
  if constexpr (kPair) cluster_sync_all(); else __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    if constexpr (kPair) tmem_dealloc_pair(tmem_base, Cfg::kTmemCols);
    else tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
  if (gs != nullptr) {
    // every CTA is done with the dependency counters: the last one out re-zeroes them
    // (all its threads, in parallel)
    unsigned* exit_ctr = gs->counters + gs->n_probs * kCounterStride;
    if (threadIdx.x == 0) {
      __threadfence();  // this CTA's counter increments precede its exit ticket
      *split_flag = atomicAdd(exit_ctr, 1u) == gridDim.x - 1 ? 1u : 0u;
    }
    __syncthreads();
    if (*split_flag) {
      for (int i = threadIdx.x; i <= gs->n_probs * kCounterStride; i += blockDim.x) gs->counters[i] = 0u;
      if (gs->chunk_counters != nullptr) {
        const int nc = gs->n_probs * gs->chunk_mb * 2 * gs->chunk_n;
        for (int i = threadIdx.x; i < nc; i += blockDim.x) gs->chunk_counters[i] = 0u;
      }
    }
  }
  if (threadIdx.x == 0) BRK_TS(7);
}

template <int BN, bool kTF32, bool kPair, bool kFullEpi>
__global__ void __launch_bounds__(EngineCfg<BN, kPair>::kThreads, 1)
    engine_kernel(const __grid_constant__ EngineParams p) {
  engine_body<BN, kTF32, kPair, kFullEpi, false>(&p, nullptr);
}

// Several dependent problems in one persistent launch (e.g. a whole MLP step):
// tiles of all problems in one global order, tile-level dependency counters.
template <int BN, bool kPair>
__global__ void __launch_bounds__(EngineCfg<BN, kPair>::kThreads, 1)
    engine_group_kernel(const __grid_constant__ EngineGroup G) {
  engine_body<BN, false, kPair, true, true>(G.probs, &G.sched);
}

template <int BN, bool kTF32, bool kPair, bool kFullEpi>
int launch_engine_t(const EngineParams& p, int grid, cudaStream_t stream, bool pdl) {
  using Cfg = EngineCfg<BN, kPair>;
  auto kern = engine_kernel<BN, kTF32, kPair, kFullEpi>;
  static int attr_set = 0;  // per instantiation; the attribute is per-context state
  cudaError_t err;
  if (!attr_set) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
    if (err != cudaSuccess) return set_cuda_error(err, "engine smem attribute");
    attr_set = 1;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(Cfg::kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  if (kPair) {
    attrs[na].id = cudaLaunchAttributeClusterDimension;
    attrs[na].val.clusterDim.x = 2;
    attrs[na].val.clusterDim.y = 1;
    attrs[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl) {
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  err = cudaLaunchKernelEx(&cfg, kern, p);
  if (err != cudaSuccess) return set_cuda_error(err, "engine launch");
  return BRK_OK;
}

}  // namespace

int engine_sm_count() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// bn: 64 / 128 / 256; pair: CTA-pair (tile rows 256) — p.m_tiles is in units of
// 128 (single) or 256 (pair) rows and the B operand coordinates in units of
// BN (single) or BN/2 (pair) rows, as set up by the caller.
int launch_engine(const EngineParams& p, int bn, int tf32, int pair, int max_units, cudaStream_t stream) {
  const int splits = p.k_splits > 1 ? p.k_splits : 1;
  const int work = p.m_tiles * p.n_tiles * splits;
  if (work <= 0) return BRK_OK;
  if (splits > 1 && (splits - 1) * ((p.k_steps + splits - 1) / splits) >= p.k_steps)
    return set_error(BRK_ERR_CONTRACT, "engine: a split-K chunk would be empty (splits > ceil(k/ceil(k/splits)))");
  if (splits > 1 && p.split_slice == 0 && (p.split_ws == nullptr || p.split_counters == nullptr))
    return set_error(BRK_ERR_CONTRACT, "engine: split-K needs a workspace");
  const int sms = engine_sm_count();
  int units = pair ? sms / 2 : sms;
  if (work < units) units = work;
  if (max_units > 0 && units > max_units) units = max_units;
  const int grid = pair ? units * 2 : units;
  const bool pdl = true;
  // the compact epilogue serves plain stores with optional bias + ReLU
  const bool full = p.mask != nullptr || p.colsum_ws != nullptr || p.sgd_w != nullptr || p.beta != 0.0f ||
                    p.alpha != 1.0f || (p.act != kActNone && p.act != kActRelu) ||
                    p.db_partials != nullptr || (splits > 1 && p.split_ws != nullptr) || (p.debug_flags & 8) ||
                    (p.debug_flags & 64);  // bit6: force the full epilogue (diagnostic)
  // compact epilogue into a blocked [outer][cols / 64][rb][64] bf16 output (conv activations,
  // FC activations): TMA stores from the staging tiles (BRK_ENGINE_TMA_OUT=0: generic stores)
  static EngineParams q;
  const EngineParams* pp = &p;
  {
    const OutMap& om = p.om;
    static const char* env = std::getenv("BRK_ENGINE_TMA_OUT");
    const bool layout = om.cl == 1 && om.cb == 64 && om.rl == 64 && om.ch == om.rb * 64 && om.rb >= 32 &&
                        p.cols % 64 == 0 &&
                        ((om.rb2 >= 0x7fffffff && om.rh == (p.cols / 64) * om.ch) ||
                         (om.rb2 == om.rb && om.rh == 0 && om.rh2 == (p.cols / 64) * om.ch));
    if (!full && !tf32 && p.out_bf16 && p.zf_w == 0 && (bn >= 128 || (bn == 64 && !pair)) && splits == 1 && layout &&
        !(env != nullptr && std::atoi(env) == 0)) {
      q = p;
      const int64_t outer = (static_cast<int64_t>(p.rows) + om.rb - 1) / om.rb;
      const uint64_t dims[3] = {64, static_cast<uint64_t>(om.rb), static_cast<uint64_t>(outer * (p.cols / 64))};
      const uint64_t strides[3] = {1, 64, static_cast<uint64_t>(om.rb) * 64};
      const uint32_t box[3] = {64, 32, 1};
      if (encode_tmap(&q.map_out, p.out, true, 3, dims, strides, box) == BRK_OK) {
        q.tma_out = 1;
        q.out_rb = static_cast<int32_t>(om.rb);
        pp = &q;
      }
    }
  }
  // (a resident-B variant for BN = 64 single-column-tile launches — the weights loaded once per
  //  CTA, the ring carrying only A — was measured slower: 3x3 K = 64 fwd 101.8 -> 107.0 us)
#define BRK_ENGINE_CASE(BN_, PAIR_)                                                                  \
  if (bn == BN_ && pair == PAIR_) {                                                                  \
    if (full) return tf32 ? launch_engine_t<BN_, true, PAIR_, true>(*pp, grid, stream, pdl)          \
                          : launch_engine_t<BN_, false, PAIR_, true>(*pp, grid, stream, pdl);        \
    return tf32 ? launch_engine_t<BN_, true, PAIR_, false>(*pp, grid, stream, pdl)                   \
                : launch_engine_t<BN_, false, PAIR_, false>(*pp, grid, stream, pdl);                 \
  }
  BRK_ENGINE_CASE(256, true)
  BRK_ENGINE_CASE(128, true)
  BRK_ENGINE_CASE(256, false)
  BRK_ENGINE_CASE(128, false)
  BRK_ENGINE_CASE(64, false)
#undef BRK_ENGINE_CASE
  return set_error(BRK_ERR_CONTRACT, "engine: BN must be 128 or 256 (pair) / 64, 128, 256 (single)");
}

template <int BN, bool kPair>
int launch_group_t(const EngineGroup& G, int grid, cudaStream_t stream) {
  using Cfg = EngineCfg<BN, kPair>;
  auto kern = engine_group_kernel<BN, kPair>;
  static int attr_set = 0;
  cudaError_t err;
  if (!attr_set) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
    if (err != cudaSuccess) return set_cuda_error(err, "engine group smem attribute");
    attr_set = 1;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(Cfg::kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  if (kPair) {
    attrs[na].id = cudaLaunchAttributeClusterDimension;
    attrs[na].val.clusterDim.x = 2;
    attrs[na].val.clusterDim.y = 1;
    attrs[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  // The grouped kernel's tiles spin on completion counters of earlier problems, so every
  // CTA of the grid must be resident at once.  Verified once per instantiation against the
  // occupancy calculator (clusters for CTA pairs); a grid that cannot be co-resident is a
  // contract error instead of a hang.  (Concurrent work that occupies SMs — another stream,
  // MPS with an SM limit — can still delay residency; the step is launched alone.)
  static int resident_units = -1;
  if (resident_units < 0) {
    int units = 0;
    if (kPair) {
      err = cudaOccupancyMaxActiveClusters(&units, kern, &cfg);
    } else {
      int per_sm = 0;
      err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::kThreads, Cfg::kSmem);
      units = per_sm * engine_sm_count();
    }
    if (err != cudaSuccess) return set_cuda_error(err, "engine group occupancy");
    resident_units = units;
  }
  if (resident_units * (kPair ? 2 : 1) < grid) {
    char buf[160];
    std::snprintf(buf, sizeof(buf), "engine group: %d CTAs must be co-resident, the device holds %d",
                  grid, resident_units * (kPair ? 2 : 1));
    return set_error(BRK_ERR_CONTRACT, buf);
  }
  attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[na].val.programmaticStreamSerializationAllowed = 1;
  ++na;
  cfg.numAttrs = na;
  err = cudaLaunchKernelEx(&cfg, kern, G);
  if (err != cudaSuccess) return set_cuda_error(err, "engine group launch");
  return BRK_OK;
}

size_t engine_split_ws_bytes(int tiles, int splits, int bn, int pair) {
  return static_cast<size_t>(tiles) * (pair ? 2 : 1) * splits * kEngineBM * bn * sizeof(float);
}

// Persistent grouped launch: one CTA (pair) per SM (pair of SMs), all co-resident,
// so tiles may wait on tiles of earlier problems (dependencies point backwards
// in the global tile order, which every CTA walks in increasing order).
int launch_engine_group(const EngineGroup& G, int bn, int pair, cudaStream_t stream) {
  const GroupSched& gs = G.sched;
  if (gs.n_probs < 1 || gs.n_probs > kMaxProbs || gs.counters == nullptr)
    return set_error(BRK_ERR_CONTRACT, "engine group: 1..12 problems and a counter buffer");
  for (int q = 0; q < gs.n_probs; ++q) {
    // (splitting a grouped problem in two halves that meet in the epilogue was measured
    // slower at the MLP shape: the weight-update units are epilogue-bound)
    const EngineParams& p = G.probs[q];
    if (p.k_splits > 1) return set_error(BRK_ERR_CONTRACT, "engine group: no split-K");
    if (gs.tile_begin[q + 1] - gs.tile_begin[q] != p.m_tiles * p.n_tiles)
      return set_error(BRK_ERR_CONTRACT, "engine group: tile_begin does not match the problem's work units");
    if (G.probs[q].m_tiles > kCounterStride - 1) return set_error(BRK_ERR_CONTRACT, "engine group: > 64 row blocks");
    if (gs.chunk_counters != nullptr && (p.m_tiles > gs.chunk_mb || p.n_tiles * bn > 64 * gs.chunk_n))
      return set_error(BRK_ERR_CONTRACT, "engine group: chunk counter table smaller than a problem's tiles");
    for (int d = 0; d < kMaxDeps; ++d) {
      if (gs.dep_prob[q][d] >= q) return set_error(BRK_ERR_CONTRACT, "engine group: dependencies must point back");
      if (gs.dep_prob[q][d] >= 0 && gs.dep_mode[q][d] == 2) {
        const EngineParams& src = G.probs[gs.dep_prob[q][d]];
        if (gs.chunk_counters == nullptr || bn != 128 || !pair || p.k_steps > gs.chunk_n ||
            src.cols > 64 * gs.chunk_n || p.m_tiles > gs.chunk_mb || src.m_tiles != p.m_tiles)
          return set_error(BRK_ERR_CONTRACT, "engine group: chunk dependencies need BN 128 CTA pairs, "
                                             "matching row blocks and a large enough chunk counter table");
      }
    }
  }
  const int work = gs.tile_begin[gs.n_probs];
  if (work <= 0) return BRK_OK;
  const int sms = engine_sm_count();
  const int units = pair ? sms / 2 : sms;
  const int grid = pair ? units * 2 : units;
  if (bn == 128 && pair) return launch_group_t<128, true>(G, grid, stream);
  if (bn == 256 && pair) return launch_group_t<256, true>(G, grid, stream);
  if (bn == 128 && !pair) return launch_group_t<128, false>(G, grid, stream);
  return set_error(BRK_ERR_CONTRACT, "engine group: BN 128/256 pair or 128 single");
}

}  // namespace brk
