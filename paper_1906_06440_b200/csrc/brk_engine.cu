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

#include "brk_engine.h"
#include "brk_internal.h"
#include "brk_ptx.cuh"

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
  static constexpr int kEpiStageBytes = kEpiWarps * 4096;
  static constexpr int kAvail = 232448 - 1024 - 256 - kEpiStageBytes;  // 227 KB opt-in max
  // ring depth: as many stages as fit (<= 8), rounded down to a multiple of 4
  // or 3 so that 3-4 producer warps share it (one issuing warp sustains only
  // ~12 B/clk/SM of TMA traffic, profiles/r01_summary.md)
  static constexpr int kFit = kAvail / kStageBytes > 8 ? 8 : kAvail / kStageBytes;
  static constexpr int kStages = kFit >= 8 ? 8 : (kFit >= 6 ? 6 : (kFit >= 4 ? 4 : kFit));
  static constexpr int kTmemCols = 2 * BN;
  static constexpr int kSmem = kStages * kStageBytes + kEpiStageBytes + 1024 + 256;
  static constexpr int kProducers = kStages % 4 == 0 ? 4 : (kStages % 3 == 0 ? 3 : (kStages % 2 == 0 ? 2 : 1));
  static constexpr int kMmaWarp = kEpiWarps;
  static constexpr int kThreads = (kEpiWarps + 1 + kProducers) * 32;
  static constexpr int kColsPerWarp = BN >= 64 ? BN / 2 : BN;  // column half per epilogue warp
};

template <bool kPair>
__device__ __forceinline__ void issue_operand(const CUtensorMap* map, const OperandCoords& oc, int rowblk, int s,
                                              uint8_t* dst, uint64_t* bar) {
  const int d0 = s % oc.kdiv0, t = s / oc.kdiv0;
  const int d1 = t % oc.kdiv1, d2 = t / oc.kdiv1;
  int32_t cs[5];
#pragma unroll
  for (int d = 0; d < 5; ++d) cs[d] = oc.base[d] + oc.rc[d] * rowblk + oc.kc[0][d] * d0 + oc.kc[1][d] * d1 + oc.kc[2][d] * d2;
  uint16_t off[3] = {0, 0, 0};
  if (oc.kind != 0) {
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
    if (oc.kind != 0) {
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
  // MN-major, 128B swizzle: atom = 128 B of MN x BK rows; 8 K-rows = 1024 B.
  constexpr uint32_t kRowsPerMma = kTF32 ? 8 : 16;
  constexpr uint32_t kAtomBytes = (kTF32 ? 32 : 64) * 128;  // BK rows x 128 B
  return make_smem_desc(base + kk * kRowsPerMma * 128, kAtomBytes, 1024, kSwizzle128B);
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define BRK_TS(slot)                                                              \
  do {                                                                            \
    if (p.debug_ts != nullptr) p.debug_ts[blockIdx.x * 16 + (slot)] = gtimer();   \
  } while (0)

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
      if (p.colsum_ws != nullptr) {  // column sums see the stored (rounded) values
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

// Plain epilogue, part 1: bias (+ReLU) on one 32-column chunk of this lane's
// row, written into the warp's staging tile (32 rows x 128 B, 16 B slot j of
// row r at slot j ^ (r % 8): conflict-free for both the row-wise writes here
// and the segment-wise reads of epilogue_flush).  bf16: chunk = 4 slots
// (two chunks fill a 128 B row segment); fp32: chunk = 8 slots.
__device__ __forceinline__ void epilogue_stage(const EngineParams& p, float (&f)[32], float bias_lane, uint8_t* row,
                                               int lane, int slot0) {
  if (p.bias != nullptr) {
#pragma unroll
    for (int j = 0; j < 32; ++j) f[j] += __shfl_sync(0xffffffffu, bias_lane, j);
  }
  if (p.act == kActRelu) {
#pragma unroll
    for (int j = 0; j < 32; ++j) f[j] = fmaxf(f[j], 0.0f);
  }
  if (p.out_bf16) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      *reinterpret_cast<uint4*>(row + (((slot0 + q) ^ (lane & 7)) << 4)) =
          make_uint4(pack_bf16x2(f[q * 8 + 0], f[q * 8 + 1]), pack_bf16x2(f[q * 8 + 2], f[q * 8 + 3]),
                     pack_bf16x2(f[q * 8 + 4], f[q * 8 + 5]), pack_bf16x2(f[q * 8 + 6], f[q * 8 + 7]));
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      *reinterpret_cast<float4*>(row + ((q ^ (lane & 7)) << 4)) =
          make_float4(f[q * 4], f[q * 4 + 1], f[q * 4 + 2], f[q * 4 + 3]);
  }
}

// Plain epilogue, part 2: write the staged 32 x 128 B tile as coalesced
// 16 B stores (8 lanes per row segment, 4 rows per instruction) instead of
// one 16 B store per row per lane (32 lines per instruction).  ro[i] is the
// element offset of row 4i + lane/8, ok its validity bit; coff the segment's
// column offset.  Stride-2 scatters also zero the three skipped positions.
// kLanes = 16 B slots per row segment: 8 (128 B) or 4 (64 B, bf16 BN=64 tiles).
template <int kLanes>
__device__ __forceinline__ void epilogue_flush(const EngineParams& p, const uint8_t* stage, const int64_t (&ro)[8],
                                               uint32_t ok, int64_t coff, int lane) {
  __syncwarp();
  constexpr int kRowsPer = 32 / kLanes;
  const int s = lane & (kLanes - 1);
  const int esz = p.out_bf16 ? 2 : 4;
  uint8_t* out = static_cast<uint8_t*>(p.out);
#pragma unroll
  for (int i = 0; i < kLanes; ++i) {
    const int r = kRowsPer * i + lane / kLanes;
    const uint4 v = *reinterpret_cast<const uint4*>(stage + r * 128 + ((s ^ (r & 7)) << 4));
    if ((ok >> r) & 1u) {
      uint8_t* dst = out + (ro[i] + coff) * esz + s * 16;
      *reinterpret_cast<uint4*>(dst) = v;
      if (p.zf_w != 0) {
        const uint4 z = make_uint4(0u, 0u, 0u, 0u);
        *reinterpret_cast<uint4*>(dst + p.zf_w * 2) = z;
        *reinterpret_cast<uint4*>(dst + p.zf_h * 2) = z;
        *reinterpret_cast<uint4*>(dst + (p.zf_w + p.zf_h) * 2) = z;
      }
    }
  }
  __syncwarp();
}

template <int BN, bool kTF32, bool kPair, bool kFullEpi>
__global__ void __launch_bounds__(EngineCfg<BN, kPair>::kThreads, 1)
    engine_kernel(const __grid_constant__ EngineParams p) {
  using Cfg = EngineCfg<BN, kPair>;
  constexpr int kStages = Cfg::kStages;
  constexpr int kMmaWarp = Cfg::kMmaWarp;
  constexpr int kProducers = Cfg::kProducers;
  constexpr int kCW = Cfg::kColsPerWarp;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * Cfg::kStageBytes + Cfg::kEpiStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;  // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint32_t* split_flag = tmem_slot + 1;

  const int warp = warp_id();
  const int lane = threadIdx.x & 31;
  const uint32_t rank = kPair ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int unit0 = kPair ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int n_units = kPair ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
  const int splits = p.k_splits > 1 ? p.k_splits : 1;
  const int ks_per = (p.k_steps + splits - 1) / splits;
  const int num_work = p.m_tiles * p.n_tiles * splits;
  if (threadIdx.x == 0) BRK_TS(0);

  if (warp == kMmaWarp + 1 && lane == 0) {
    tma_prefetch_desc(&p.map_a);
    tma_prefetch_desc(&p.map_b);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kPair ? 2 * kEpiWarps : kEpiWarps);
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

  if (warp > kMmaWarp) {
    // ------------------------------------------------------------ producers
    const int pid = warp - kMmaWarp - 1;
    if (elect_one()) {
      pdl_wait();  // inputs are produced by the previous kernel
      const uint32_t bytes = (p.ca.n_loads * p.ca.load_bytes + p.cb.n_loads * p.cb.load_bytes) * (kPair ? 2 : 1);
      int g = 0;  // global k-step counter of this CTA (same sequence as the MMA issuer)
      for (int u = unit0; u < num_work; u += n_units) {
        const int t = u / splits, sp = u - t * splits;
        const int mb = t % p.m_tiles, nb = t / p.m_tiles;
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
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::kStageBytes;
          uint8_t* sb = sa + kTileABytes;
          if (p.debug_flags & 2) {
            if (leader) mbar_arrive(&full[stage]);
          } else {
            if (leader) mbar_arrive_expect_tx(&full[stage], bytes);
            issue_operand<kPair>(&p.map_a, p.ca, arow, s, sa, &full[stage]);
            issue_operand<kPair>(&p.map_b, p.cb, brow, s, sb, &full[stage]);
          }
          if (gg == 0 && pid == 0) BRK_TS(2);
        }
        g += n_steps;
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    if (leader) {
      const uint32_t idesc = make_idesc(kTF32 ? kFmtTF32 : kFmtBF16, kPair ? 256 : kEngineBM, BN,
                                        p.ca.mn_major, p.cb.mn_major);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int u = unit0; u < num_work; u += n_units, ++local) {
        const int sp = u % splits;
        const int s_begin = sp * ks_per;
        const int n_steps = min(p.k_steps, s_begin + ks_per) - s_begin;
        const int acc = local & 1;
        mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int s = 0; s < n_steps; ++s) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (local == 0 && s == 0 && lane == 0) BRK_TS(3);
          if (elect_one()) {
            if (p.debug_flags & 1) {
              if constexpr (kPair) {
                mma_commit_pair(&empty[stage]);
                if (s == n_steps - 1) mma_commit_pair(&tfull[acc]);
              } else {
                mbar_arrive(&empty[stage]);
                if (s == n_steps - 1) mbar_arrive(&tfull[acc]);
              }
            } else {
              const uint32_t sa = smem_u32(smem + stage * Cfg::kStageBytes);
              const uint32_t sb = sa + kTileABytes;
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                const uint64_t ad = operand_desc<kTF32>(sa, p.ca.mn_major, kk);
                const uint64_t bd = operand_desc<kTF32>(sb, p.cb.mn_major, kk);
                const uint32_t accum = (s > 0 || kk > 0) ? 1u : 0u;
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
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) BRK_TS(4);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 0..7)
    pdl_wait();  // outputs may be read by the previous kernel (WAR) — wait before writing
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int chalf = warp >> 2;   // column half this warp drains
    const int cbeg = chalf * kCW;
    const int row_in_tile = quarter * 32 + lane;
    const uint32_t tempty_leader = kPair ? mapa_shared(smem_u32(&tempty[0]), 0) : 0u;
    const int halves = kPair ? 2 : 1;
    int local = 0;
    for (int u = unit0; u < num_work; u += n_units, ++local) {
      const int t = u / splits, sp = u - t * splits;
      const int mb = t % p.m_tiles, nb = t / p.m_tiles;
      const int acc = local & 1;
      // bias for this warp's columns, one value per lane per 32-column chunk
      float bias_r[kCW / 32];
#pragma unroll
      for (int c = 0; c < kCW / 32; ++c) {
        const int col = nb * BN + cbeg + c * 32 + lane;
        bias_r[c] = (p.bias != nullptr && col < p.cols) ? __ldg(p.bias + col) : 0.0f;
      }
      mbar_wait(&tfull[acc], (local >> 1) & 1);
      tc_fence_after();
      if (threadIdx.x == 0) BRK_TS(5);
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
      const uint32_t tbase = tmem_base + acc * BN + (static_cast<uint32_t>(quarter * 32) << 16) + cbeg;
      if (splits == 1 || p.split_ws == nullptr) {
        // column offset maintained incrementally (32 columns never straddle an
        // output block: cb % 32 == 0, host guarantees); TMEM loads are software-
        // pipelined one chunk ahead so the ld latency overlaps the epilogue math.
        const int cfirst = nb * BN + cbeg;
        // plain epilogue: staging tile, and the row offsets each lane stores in epilogue_flush
        uint8_t* stage = smem + kStages * Cfg::kStageBytes + warp * 4096;
        int64_t ro[8];
        uint32_t ok_bits = 0;
        int64_t seg_coff = 0;
        if constexpr (!kFullEpi) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            ro[i] = __shfl_sync(0xffffffffu, roff,
                                (kCW == 32 && p.out_bf16) ? 8 * (i & 3) + (lane >> 2) : 4 * i + (lane >> 3));
          ok_bits = __ballot_sync(0xffffffffu, row_ok);
        }
        int cq = cfirst / static_cast<int>(p.om.cb);
        int cr = cfirst - cq * static_cast<int>(p.om.cb);
        uint32_t v[32];
        tmem_ld32(tbase, v);
#pragma unroll
        for (int c = 0; c < kCW / 32; ++c) {
          tmem_ld_wait();
          float f[32];
          if (kFullEpi && p.alpha != 1.0f) {
#pragma unroll
            for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]) * p.alpha;
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
          }
          if (c + 1 < kCW / 32) tmem_ld32(tbase + (c + 1) * 32, v);
          const int col0 = cfirst + c * 32;
          const int64_t off = roff + static_cast<int64_t>(cq) * p.om.ch + static_cast<int64_t>(cr) * p.om.cl;
          cr += 32;
          if (cr == p.om.cb) { cr = 0; ++cq; }
          if (p.out == nullptr) continue;  // diagnostic: mainloop-only timing
          if constexpr (kFullEpi) {
            if (threadIdx.x == 0 && c < 2) BRK_TS(8 + 2 * c);
            epilogue_finish(p, f, row_ok && col0 < p.cols, off, col0, warp_row0, lane, bias_r[c]);
            if (threadIdx.x == 0 && c < 2) BRK_TS(9 + 2 * c);
          } else {
            const int64_t coff = off - roff;
            if (kCW == 32 && p.out_bf16) {  // 64 B row segments
              epilogue_stage(p, f, bias_r[c], stage + lane * 128, lane, 0);
              if (col0 < p.cols) epilogue_flush<4>(p, stage, ro, ok_bits, coff, lane);
              else __syncwarp();
            } else {
              const bool second = p.out_bf16 && (c & 1);
              if (!second) seg_coff = coff;
              epilogue_stage(p, f, bias_r[c], stage + lane * 128, lane, second ? 4 : 0);
              if (!p.out_bf16 || second) {
                if (col0 < p.cols) epilogue_flush<8>(p, stage, ro, ok_bits, seg_coff, lane);
                else __syncwarp();
              }
            }
          }
        }
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (threadIdx.x == 0) BRK_TS(12);
        if (lane == 0) {
          if constexpr (kPair) mbar_arrive_cluster_relaxed(tempty_leader + acc * 8);
          else mbar_arrive_relaxed(&tempty[acc]);
        }
        if (threadIdx.x == 0) BRK_TS(13);
      } else if constexpr (kFullEpi) {
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
      if (kFullEpi && p.db_partials != nullptr && mb == 0 && rank == 0 && sp == 0) {
        for (int c = threadIdx.x; c < BN; c += kEpiThreads) {
          const int col = nb * BN + c;
          if (col >= p.cols) continue;
          float s = 0.0f;
          for (int q = 0; q < p.db_parts; ++q) s += p.db_partials[static_cast<int64_t>(q) * p.cols + col];
          p.db_out[col] = s;
          if (p.bias_sgd != nullptr) p.bias_sgd[col] -= p.bias_lr * s;
        }
      }
      if (threadIdx.x == 0) BRK_TS(6);
    }
  }
  tc_fence_before();
  if constexpr (kPair) cluster_sync_all(); else __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    if constexpr (kPair) tmem_dealloc_pair(tmem_base, Cfg::kTmemCols);
    else tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
  if (threadIdx.x == 0) BRK_TS(7);
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
#define BRK_ENGINE_CASE(BN_, PAIR_)                                                                  \
  if (bn == BN_ && pair == PAIR_) {                                                                  \
    if (full) return tf32 ? launch_engine_t<BN_, true, PAIR_, true>(p, grid, stream, pdl)            \
                          : launch_engine_t<BN_, false, PAIR_, true>(p, grid, stream, pdl);          \
    return tf32 ? launch_engine_t<BN_, true, PAIR_, false>(p, grid, stream, pdl)                     \
                : launch_engine_t<BN_, false, PAIR_, false>(p, grid, stream, pdl);                   \
  }
  BRK_ENGINE_CASE(256, true)
  BRK_ENGINE_CASE(128, true)
  BRK_ENGINE_CASE(256, false)
  BRK_ENGINE_CASE(128, false)
  BRK_ENGINE_CASE(64, false)
#undef BRK_ENGINE_CASE
  return set_error(BRK_ERR_CONTRACT, "engine: BN must be 128 or 256 (pair) / 64, 128, 256 (single)");
}

size_t engine_split_ws_bytes(int tiles, int splits, int bn, int pair) {
  return static_cast<size_t>(tiles) * (pair ? 2 : 1) * splits * kEngineBM * bn * sizeof(float);
}

}  // namespace brk
