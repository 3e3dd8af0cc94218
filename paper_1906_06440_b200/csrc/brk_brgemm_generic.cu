// brk_brgemm_generic.cu — the reference-API BRGEMM on tcgen05.
//
// Computes, for each job j (one output block C_j):
//     C_j = beta * C_j + alpha * sum_i  B_ij @ A_ij          (reference view)
// in the storage contract of brgemm.py:1-24 (reference):
//     a block (k, m) with row stride lda  (m contiguous)
//     b block (n, k) with row stride ldb  (k contiguous)
//     c       (n, m) with row stride ldc  (m contiguous)
// The batch entries come from one of the three BRGEMM variants of the paper:
//     address list (brgemm.py:260), fixed strides (brgemm.py:296) or
//     per-entry element offsets from a base (the north-star offset variant).
//
// This kernel serves arbitrary (unaligned, tiny, odd-strided) blocks, so the
// operands are gathered by all 128 threads with plain loads (no TMA alignment
// rules apply), converted to the MMA input type (TF32 by cvt.rna or BF16 by
// RN) and written into the SWIZZLE_NONE K-major canonical layout.  The single
// elected thread issues tcgen05.mma into a TMEM accumulator that lives across
// the whole batch (the reduction over i never leaves TMEM), and the 4 warps
// drain TMEM once with tcgen05.ld, apply alpha/beta and store.
//
// TMEM lanes  <-> reference n (rows of C),  TMEM columns <-> reference m.
// tcgen05 A operand = reference B blocks (n x k, K-major)
// tcgen05 B operand = reference A blocks (k x m) transposed into K-major rows of m.
#include <algorithm>

#include "brk_internal.h"
#include "brk_ptx.cuh"
#include "brk_tma_host.h"

namespace brk {
namespace {

constexpr int kRows = 128;         // C rows (reference n) per tile = MMA M
constexpr int kCols = 256;         // C cols (reference m) per tile = max MMA N
constexpr int kGatherWarps = 8;    // warps 0-7: operand gather (cp.async / converting loads)
constexpr int kMmaWarp = 8;        // warp 8: tcgen05.mma issuer
constexpr int kTmaWarp = 9;        // warps 9-12: TMA producers (stride / offset variants)
constexpr int kTmaWarps = 4;       // a warp keeps ~one box in flight: four of them per SM
constexpr int kEpiWarp0 = kTmaWarp + kTmaWarps;  // warps 13-16: epilogue (one per TMEM lane quarter)
constexpr int kEpiWarps = 4;
constexpr int kThreads = (kEpiWarp0 + kEpiWarps) * 32;
constexpr int kMaxStages = 16;  // (16 only for the compact small-block ring; other rings hold <= 8)
constexpr int kRingBytes = 4 * (kRows * 128 + kCols * 128);  // 192 KB of operand ring
constexpr int kAtomColsBf16 = 64;  // bf16 elements per 128 B swizzle-atom row
constexpr int kAOpBytes = kRows * 128;    // K-major, 128B swizzle: 128 rows x 128 B of K
constexpr int kSmemBytes = kRingBytes + 1024 + 1024;
constexpr int kMaxAcc = 8;
#ifndef BRK_GATHER_GROUPS
#define BRK_GATHER_GROUPS 1  // non-tiny gathered stages: two groups of four warps (0: all eight)
#endif  // TMEM accumulators (512 columns / the widest tile's columns)  // ring + alignment slack + barriers / TMEM slot

struct EntryPtrs {
  const char* a;
  const char* b;
};

__device__ __forceinline__ EntryPtrs entry_ptrs(const GenericParams& p, int job, int i) {
  const size_t esz = p.in_bf16 ? 2 : 4;
  EntryPtrs e;
  const int64_t idx = static_cast<int64_t>(job) * p.batch + i;
  if (p.mode == kModeAddr) {
    e.a = static_cast<const char*>(p.a_ptrs[idx]);
    e.b = static_cast<const char*>(p.b_ptrs[idx]);
  } else if (p.mode == kModeOffs) {
    e.a = static_cast<const char*>(p.a_base) + p.a_offs[idx] * esz;
    e.b = static_cast<const char*>(p.b_base) + p.b_offs[idx] * esz;
  } else {
    e.a = static_cast<const char*>(p.a_base) + (job * p.jstride_a + i * p.stride_a) * esz;
    e.b = static_cast<const char*>(p.b_base) + (job * p.jstride_b + i * p.stride_b) * esz;
  }
  return e;
}

__device__ __forceinline__ float load_in(const char* base, int64_t idx, bool bf16) {
  if (bf16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[idx]);
  return reinterpret_cast<const float*>(base)[idx];
}

// 16 B of MMA input (8 bf16 or 4 tf32) from `cnt` elements at base + i*step
// (contiguous & aligned: one vector load); elements past `cnt` are zero.
template <bool kTF32>
__device__ __forceinline__ uint4 load_chunk(const char* base, int64_t first, int64_t step, int cnt, bool bf16_in,
                                            bool vec) {
  constexpr int kE = kTF32 ? 4 : 8;
  if (vec && cnt >= kE) {
    if (bf16_in) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(base) + first));
      if constexpr (!kTF32) return v;
      // bf16 storage on a TF32 computation: widen (exact)
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
      const float2 f0 = __bfloat1622float2(h[0]), f1 = __bfloat1622float2(h[1]);
      return make_uint4(f32_to_tf32(f0.x), f32_to_tf32(f0.y), f32_to_tf32(f1.x), f32_to_tf32(f1.y));
    }
    const float4* f4 = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(base) + first);
    const float4 f = __ldg(f4);
    if constexpr (kTF32) {
      return make_uint4(f32_to_tf32(f.x), f32_to_tf32(f.y), f32_to_tf32(f.z), f32_to_tf32(f.w));
    } else {  // fp32 storage, bf16 tensor-core input: 8 elements = two 16 B loads
      const float4 g = __ldg(f4 + 1);
      return make_uint4(pack_bf16x2(f.x, f.y), pack_bf16x2(f.z, f.w), pack_bf16x2(g.x, g.y), pack_bf16x2(g.z, g.w));
    }
  }
  float v[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) v[t] = (t < kE && t < cnt) ? load_in(base, first + t * step, bf16_in) : 0.0f;
  if constexpr (kTF32) return make_uint4(f32_to_tf32(v[0]), f32_to_tf32(v[1]), f32_to_tf32(v[2]), f32_to_tf32(v[3]));
  return make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                    pack_bf16x2(v[6], v[7]));
}

// element offsets of an entry's blocks from the buffer bases (offset / stride variants, and
// address lists with views); false when an address-list block is not inside its view
__device__ __forceinline__ bool entry_offs(const GenericParams& p, int job, int i, int64_t& oa, int64_t& ob) {
  const int64_t idx = static_cast<int64_t>(job) * p.batch + i;
  if (p.mode == kModeAddr) {
    const int64_t esz = p.in_bf16 ? 2 : 4;
    const int64_t da = static_cast<const char*>(p.a_ptrs[idx]) - static_cast<const char*>(p.a_base);
    const int64_t db = static_cast<const char*>(p.b_ptrs[idx]) - static_cast<const char*>(p.b_base);
    oa = da / esz;
    ob = db / esz;
    return da >= 0 && db >= 0 && da % esz == 0 && db % esz == 0 &&
           oa + static_cast<int64_t>(p.k - 1) * p.a_sk + p.m <= p.a_view &&
           ob + static_cast<int64_t>(p.n - 1) * p.b_sn + p.k <= p.b_view;
  }
  if (p.mode == kModeOffs) {
    oa = p.a_offs[idx];
    ob = p.b_offs[idx];
  } else {
    oa = job * p.jstride_a + i * p.stride_a;
    ob = job * p.jstride_b + i * p.stride_b;
  }
  return true;
}

// Persistent: CTA walks job tiles (job, n-tile, m-tile) with four decoupled roles:
//  * the TMA warps load each entry's (reference b block, reference a block) pair as one box
//    each when no block of the launch wraps a row of its buffer's 2-d view (stride variant:
//    decided on the host; offset / address-with-views: by box_check_kernel just before);
//  * otherwise warps 0-7 gather every entry (cp.async for aligned contiguous bf16 rows, else
//    converting loads) — reference b rows -> K-major 128B-swizzled A operand, reference a
//    rows -> MN-major (bf16) or K-major (TF32) B operand; with TF32 boxes they round the
//    landed stages to TF32 instead;
//  * warp 8 issues the tcgen05.mma chain (the whole batch reduces in TMEM), two
//    accumulators so a tile's MMAs overlap the previous tile's epilogue;
//  * warps 10-13 drain TMEM and apply alpha / beta / bias / act / mask.
// Ring stages are sized by the tile (16 KB A + the B atoms actually used).
// diagnostics build: stamps of CTA 0 — stage g < 64: [g*4 + 0] producer / gather issued,
// [g*4 + 1] MMA saw it full, [g*4 + 2] MMAs issued; tile l < 16: [256 + l*4 + 0] MMA got the
// accumulator, [+1] epilogue saw it done, [+2] epilogue released it
#ifdef BRK_DIAG
__device__ __forceinline__ unsigned long long gen_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define GEN_TS(cond, idx)                                                     \
  do {                                                                        \
    if (p.ts != nullptr && blockIdx.x == 0 && (cond)) p.ts[idx] = gen_gtimer(); \
  } while (0)
#else
#define GEN_TS(cond, idx) \
  do {                    \
  } while (0)
#endif

template <bool kTF32>
__global__ void __launch_bounds__(kThreads, 1) brgemm_generic_kernel(const __grid_constant__ GenericParams p) {
  constexpr int kE = kTF32 ? 4 : 8;              // elements per 16 B
  constexpr int kKC = kTF32 ? 32 : 64;           // K elements per stage (128 B)
  constexpr int kMmaK = kTF32 ? 8 : 16;          // K per tcgen05.mma
  constexpr int kAtomCols = kTF32 ? 32 : 64;     // MN elements per 128 B atom row
  constexpr int kAtomBytes = kKC * 128;          // one MN-major atom: kKC K-rows x 128 B

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRingBytes);
  uint64_t* empty = full + kMaxStages;
  uint64_t* done = empty + kMaxStages;  // [kMaxAcc] accumulator complete
  uint64_t* drained = done + kMaxAcc;   // [kMaxAcc] epilogue finished reading TMEM
  uint64_t* rounded = drained + kMaxAcc;  // [kMaxStages] TF32 TMA stages rounded in place (RNA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rounded + kMaxStages);

  const int tid = threadIdx.x;
  const int warp = tid / 32;
  const int lane = tid % 32;
  const int m_tiles = (p.m + kCols - 1) / kCols;
  const int n_tiles = (p.n + kRows - 1) / kRows;
  const int tiles = m_tiles * n_tiles * p.n_jobs;
  const bool bf16_in = p.in_bf16 != 0;
  const int n_chunks = (p.k + kKC - 1) / kKC;
  const int steps = (p.alpha == 0.0f) ? 0 : p.batch * n_chunks;
  // TF32 with TMA (stride variant, every entry one box per operand): fp32 blocks land as they
  // are — A K-major, B MN-major in 32-element atoms (128B swizzle of 32 B chunks) — and the
  // idle gather warps round each stage to TF32 in place (RNA, like the gather path's
  // cvt.rna) before the MMA reads it; the tensor core alone would truncate the mantissa
  // every entry of the launch is one box per operand: known on the host (stride variant) or
  // checked on the device just before (offset variant, address variant with views).  A launch
  // either boxes every entry or gathers every entry: the producer and gather roles never
  // interleave on the ring (a role that skips the other role's stages could run two phases
  // ahead on a stage, where the parity waits alias)
  const bool boxes = p.tma && (p.all_tma || (p.tma_ok != nullptr && *p.tma_ok != 0));
  const bool tf32_tma = kTF32 && boxes;
  const bool b_mn = !kTF32 || tf32_tma;  // B operand MN-major (atoms) vs K-major rows
  // ring geometry: the B operand of the widest tile (MN-major atoms, or K-major rows for gathered TF32)
  const int m_max = min(p.m, kCols);
  const int b_bytes = b_mn ? (m_max + kAtomCols - 1) / kAtomCols * kAtomBytes : ((m_max + 15) & ~15) * 128;
  // Small blocks (one K chunk per entry, k <= 64, bf16 gathers): the gather copies only each
  // entry's valid rows / chunks.  The ring starts zeroed, the MMA B operand's K-rows past k are
  // never written (stay zero), so stale A chunks past k multiply zeros; rows / columns past the
  // block only feed accumulator rows / columns the epilogue does not store.
  const bool sparse = !kTF32 && !p.tma && p.in_bf16 && n_chunks == 1;
  // Compact ring (sparse, k <= 32, one B atom): a stage holds only the block's A rows and B
  // K-rows (m = n = k = 32: 8 KB instead of 24 KB), so 16 stages are in flight instead of 8.
  // The M = 128 MMA still reads 128 A rows from the stage start: rows past the block come from
  // the following stages (or unused ring) and only feed accumulator rows the epilogue does not
  // store; the MMAs stop at K = ceil16(k), so only the stage's own B K-rows are read.
  const int a_bytes_c = ((((min(p.n, kRows) + 7) & ~7) * 128) + 1023) & ~1023;
  const int b_bytes_c = (((p.k + 15) & ~15) * 128 + 1023) & ~1023;
  const bool compact = sparse && m_max <= kAtomCols && p.k <= 32 &&
                       (kMaxStages - 1) * (a_bytes_c + b_bytes_c) + kAOpBytes <= kRingBytes;
  // 64B-swizzle boxes (m = k = 32, TMA): A rows of 64 B, B 32 K-rows x 64 B, compact stages
  // read like the compact ring (the M = 128 MMA reads 8 KB of A rows from the stage start)
  const bool sw64 = boxes && p.sw64 != 0;
  const int a_bytes_s = ((p.nbox * 64) + 1023) & ~1023;
  const int b_off = compact ? a_bytes_c : (sw64 ? a_bytes_s : kAOpBytes);  // B operand offset inside a stage
  const int stage_bytes = compact ? a_bytes_c + b_bytes_c
                                  : (sw64 ? a_bytes_s + 2048 : (kAOpBytes + b_bytes + 1023) & ~1023);
  // (a multiple of the TMA producer count: each stage always has the same producer, so the
  // parity waits on its empty barrier cannot alias)
  const int n_stages = (compact || sw64)
                           ? kMaxStages
                           : min(min(kMaxStages, 8), kRingBytes / stage_bytes) / kTmaWarps * kTmaWarps;
  // (4, 8 or 16: stage slot and phase by mask and shift — the MMA issuer's per-stage work is
  // on the serial path of every tile)
  const int st_shift = n_stages >= 16 ? 4 : (n_stages >= 8 ? 3 : 2);
  const int st_mask = n_stages - 1;
  // TMEM accumulators: 512 columns split into as many as the widest tile allows (2 of 256
  // columns, ... 8 of 64), so short tiles (small batch) keep up to 7 tiles of MMAs ahead of
  // the epilogue instead of one
  const int n_cols_max = kTF32 ? (m_max + 15) & ~15 : (m_max + kAtomCols - 1) / kAtomCols * kAtomCols;
  const int acc_cols = n_cols_max <= 64 ? 64 : (n_cols_max <= 128 ? 128 : 256);
  const int acc_shift = acc_cols == 64 ? 3 : (acc_cols == 128 ? 2 : 1);  // log2(accumulators)
  const int acc_mask = (1 << acc_shift) - 1;

  if (tid == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(&full[s], 1);  // TMA: the producer's expect_tx; gather: one arrive after the copies
      mbar_init(&empty[s], 1);
      mbar_init(&rounded[s], 1);
    }
    for (int a = 0; a < kMaxAcc; ++a) {
      mbar_init(&done[a], 1);
      mbar_init(&drained[a], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_slot, 2 * kCols);
  if (sparse) {
    for (int i = tid; i < kRingBytes / 16; i += kThreads)
      asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(smem_u32(smem) + i * 16), "r"(0u) : "memory");
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // Does batch entry `entry` of `job` go through TMA (all roles evaluate it identically), and
  // where do its boxes start in the 2-d views.  Evaluated once per entry, not per K chunk.
  struct EntryBox {
    bool tma;
    int32_t ca, ra, cb, rb;
  };
  auto entry_box = [&](int job, int entry) -> EntryBox {
    EntryBox eb{false, 0, 0, 0, 0};
    if (!boxes) return eb;
    if (p.all_tma) {
      eb.tma = true;
      eb.ra = static_cast<int32_t>(job * p.rj_a + entry * p.rs_a);
      eb.rb = static_cast<int32_t>(job * p.rj_b + entry * p.rs_b);
      return eb;
    }
    int64_t oa, ob;
    if (!entry_offs(p, job, entry, oa, ob)) return eb;
    int64_t qa, qb;
    if (((oa | ob) >> 32) == 0) {  // 32-bit division when the offsets allow it
      qa = static_cast<uint32_t>(oa) / static_cast<uint32_t>(p.a_sk);
      qb = static_cast<uint32_t>(ob) / static_cast<uint32_t>(p.b_sn);
    } else {
      qa = oa / p.a_sk;
      qb = ob / p.b_sn;
    }
    eb.ra = static_cast<int32_t>(qa);
    eb.ca = static_cast<int32_t>(oa - qa * p.a_sk);
    eb.rb = static_cast<int32_t>(qb);
    eb.cb = static_cast<int32_t>(ob - qb * p.b_sn);
    eb.tma = eb.cb + p.k <= p.b_sn && eb.ca + p.m <= p.a_sk;
    return eb;
  };

  if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    // stage-0 operand descriptors.  MN-major B: bf16 atoms of 64 K-rows (8-row swizzle
    // groups, SBO 1024 B); TF32 atoms of 32 K-rows in the 32 B-chunk swizzle (4-row groups,
    // SBO 512 B); K-major TF32 rows.  Per K-step: A +32 B; B +32 B (K-major) or +kMmaK rows.
    const uint32_t ring0 = smem_u32(smem);
    // 64B swizzle (sw64): 8-row groups of 512 B for both; B K-step = 16 K-rows of 64 B
    const uint64_t a_desc0 = sw64 ? make_smem_desc(ring0, 16, 512, kSwizzle64B)
                                  : make_smem_desc(ring0, 16, 1024, kSwizzle128B);
    const uint64_t b_desc0 =
        sw64 ? make_smem_desc(ring0 + b_off, 2048, 512, kSwizzle64B)
             : (!b_mn ? make_smem_desc(ring0 + b_off, 16, 1024, kSwizzle128B)
                      : (kTF32 ? make_smem_desc(ring0 + b_off, kAtomBytes, 512, kSwizzle128B32)
                               : make_smem_desc(ring0 + b_off, kAtomBytes, 1024, kSwizzle128B)));
    const uint32_t b_kstep = sw64 ? kMmaK * 64 / 16 : (b_mn ? kMmaK * 128 / 16 : 2);
    int local = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++local) {
      if (steps == 0) continue;
      const int mt = t % m_tiles;
      const int m_here = min(kCols, p.m - mt * kCols);
      const int n_cols =
          sw64 ? 32 : (kTF32 ? (m_here + 15) & ~15 : (m_here + kAtomCols - 1) / kAtomCols * kAtomCols);
      const uint32_t idesc = make_idesc(kTF32 ? kFmtTF32 : kFmtBF16, kRows, n_cols, 0, b_mn ? 1 : 0);
      const int acc = local & acc_mask;
      mbar_wait(&drained[acc], ((local >> acc_shift) & 1) ^ 1);  // the epilogue read this accumulator
      GEN_TS(local < 16 && lane == 0, 256 + local * 4 + 0);
      tc_fence_after();
      const uint32_t d_tmem = tmem + acc * acc_cols;
      const int g0 = local * steps;
      for (int s = 0; s < steps; ++s) {
        const int g = g0 + s, st = g & st_mask;
        mbar_wait(tf32_tma ? &rounded[st] : &full[st], (g >> st_shift) & 1);
        GEN_TS(g < 64 && lane == 0, g * 4 + 1);
        tc_fence_after();
        // gathered / rounded stages were written through the generic proxy (TMA boxes land
        // through the async proxy already: the fence cost ~0.1 us per stage on the serial issuer)
        if (!boxes || tf32_tma) fence_proxy_async_smem();
        if (elect_one()) {
          // descriptors built once per launch and advanced by constants (16-byte units): the
          // issuer's per-stage work is on the serial path of every tile (small blocks: ~0.3 us
          // per stage); start-address field = bits 0-13, the ring sits below 256 KB
          const uint32_t so = static_cast<uint32_t>(st * stage_bytes) >> 4;
          const uint64_t ad = a_desc0 + so;
          const uint64_t bd = b_desc0 + so;
          const int ksteps = (compact || sw64) ? (p.k + kMmaK - 1) / kMmaK : kKC / kMmaK;
#pragma unroll
          for (int kk = 0; kk < kKC / kMmaK; ++kk) {
            if (kk >= ksteps) break;
            mma_ss<kTF32>(d_tmem, ad + kk * 2, bd + kk * b_kstep, idesc, (s > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&empty[st]);
          if (s == steps - 1) mma_commit(&done[acc]);
          GEN_TS(g < 64, g * 4 + 2);
        }
        __syncwarp();
      }
    }
  } else if (warp >= kTmaWarp && warp < kTmaWarp + kTmaWarps) {
    // ------------------------------------------------------------ TMA producers (stage g: warp g % 4)
    const int pid = warp - kTmaWarp;
    if (boxes && elect_one()) {
      int local = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++local) {
        const int mt = t % m_tiles;
        const int nt = (t / m_tiles) % n_tiles;
        const int job = t / (m_tiles * n_tiles);
        const int n0 = nt * kRows, m0 = mt * kCols;
        const int m_here = min(kCols, p.m - m0);
        const int atoms = (m_here + kAtomCols - 1) / kAtomCols;
        const uint32_t bytes =
            sw64 ? static_cast<uint32_t>(p.nbox * 64 + 2048) : static_cast<uint32_t>(p.nbox * 128 + atoms * p.abox * 128);
        int g = local * steps;
        // offset / address tables: this job's entries are contiguous — pull their lines into L1
        // once, so the per-entry reads below do not each pay an L2 round trip
        if (!p.all_tma && steps > 0 && (p.mode == kModeOffs || p.mode == kModeAddr)) {
          const char* ta = p.mode == kModeOffs ? reinterpret_cast<const char*>(p.a_offs)
                                               : reinterpret_cast<const char*>(p.a_ptrs);
          const char* tb = p.mode == kModeOffs ? reinterpret_cast<const char*>(p.b_offs)
                                               : reinterpret_cast<const char*>(p.b_ptrs);
          const int64_t first = static_cast<int64_t>(job) * p.batch * 8;
          for (int64_t o = first & ~int64_t(127); o < first + p.batch * 8; o += 128) {
            asm volatile("prefetch.global.L1 [%0];" ::"l"(ta + o));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(tb + o));
          }
        }
        for (int entry = 0; entry < p.batch && steps > 0; ++entry) {
          // entries none of whose chunks this producer issues are skipped without reading them
          bool mine = n_chunks >= kTmaWarps;
          for (int ch = 0; ch < n_chunks && !mine; ++ch) mine = (g + ch) % kTmaWarps == pid;
          if (!mine) { g += n_chunks; continue; }
          const EntryBox eb = entry_box(job, entry);
          if (!eb.tma) { g += n_chunks; continue; }
          for (int ch = 0; ch < n_chunks; ++ch, ++g) {
            if (g % kTmaWarps != pid) continue;
            const int k0 = ch * kKC, st = g & st_mask;
            if (g >= n_stages) mbar_wait(&empty[st], ((g >> st_shift) + 1) & 1);
            uint8_t* a_op = smem + st * stage_bytes;
            GEN_TS(g < 64, g * 4 + 0);
            mbar_arrive_expect_tx(&full[st], bytes);
            const int32_t cA[2] = {eb.cb + k0, eb.rb + n0};
            tma_load<2>(a_op, &p.map_bop, &full[st], cA);
            for (int at = 0; at < atoms; ++at) {
              const int32_t cB[2] = {eb.ca + m0 + at * kAtomCols, eb.ra + k0};
              tma_load<2>(a_op + b_off + at * kAtomBytes, &p.map_aop, &full[st], cB);
            }
          }
        }
      }
    }
  } else if (warp < kGatherWarps && tf32_tma) {
    // ------------------------------------------------------------ TF32 rounding (RNA) of TMA stages
    const int gt = tid;  // 0 .. 255
    int local = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++local) {
      const int mt = t % m_tiles;
      const int m_here = min(kCols, p.m - mt * kCols);
      const int atoms = (m_here + kAtomCols - 1) / kAtomCols;
      const int vecs = (p.nbox * 128 + atoms * kAtomBytes) / 16;  // the stage bytes the boxes wrote
      const int g0 = local * steps;
      for (int s = 0; s < steps; ++s) {
        const int g = g0 + s, st = g & st_mask;
        mbar_wait(&full[st], (g >> st_shift) & 1);
        uint4* v4 = reinterpret_cast<uint4*>(smem + st * stage_bytes);
        const int a_vecs = p.nbox * 8;
        for (int i = gt; i < vecs; i += kGatherWarps * 32) {
          // A rows [0, nbox) then the B atoms at kAOpBytes
          uint4* q = i < a_vecs ? v4 + i : reinterpret_cast<uint4*>(smem + st * stage_bytes + kAOpBytes) + (i - a_vecs);
          uint4 v = *q;
          v = make_uint4(f32_to_tf32(__uint_as_float(v.x)), f32_to_tf32(__uint_as_float(v.y)),
                         f32_to_tf32(__uint_as_float(v.z)), f32_to_tf32(__uint_as_float(v.w)));
          *q = v;
        }
        fence_proxy_async_smem();  // generic-proxy rewrites -> the MMA's async-proxy reads
        asm volatile("bar.sync 1, %0;" ::"r"(kGatherWarps * 32) : "memory");
        if (gt == 0) mbar_arrive(&rounded[st]);
      }
    }
  } else if (warp < kGatherWarps) {
    // ------------------------------------------------------------ gather
    const int gt = tid;  // 0 .. 255
    const bool a_contig = p.b_sk == 1;   // reference b block: k contiguous
    const bool b_contig = p.a_sm == 1;   // reference a block: m contiguous
    int local = 0;
    for (int t = boxes ? tiles : blockIdx.x; t < tiles; t += gridDim.x, ++local) {
      const int mt = t % m_tiles;
      const int nt = (t / m_tiles) % n_tiles;
      const int job = t / (m_tiles * n_tiles);
      const int n0 = nt * kRows, m0 = mt * kCols;
      const int m_here = min(kCols, p.m - m0);
      const int n_here = min(kRows, p.n - n0);
      const int n_cols = kTF32 ? (m_here + 15) & ~15 : (m_here + kAtomCols - 1) / kAtomCols * kAtomCols;
      const int n_rows8 = (n_here + 7) & ~7;
      const int col_chunks = n_cols / kE;
      const int g0 = local * steps;
      // Per-tile unit tables for the all-cp.async case (bf16 in, contiguous rows): this thread's
      // (row, 16 B chunk) -> (ring offset, element offset) map is the same for every entry and
      // K chunk of the tile, so a stage costs one add and one clamp per copy.  (The loops below
      // recompute it per unit and stage with integer divisions: ~300 instructions per gather
      // warp per stage, which bounded small blocks at ~1.1 us per stage whatever its bytes.)
      constexpr int kUnits = 4;
      int ta_dst[kUnits], ta_src[kUnits], ta_kk[kUnits], tb_dst[kUnits], tb_src[kUnits], tb_kr[kUnits],
          tb_mc[kUnits];
      const int k1 = min(kKC, p.k);  // k_here of a sparse tile (one K chunk per entry)
      const int a_cpr_t = sparse ? (k1 + kE - 1) / kE : 8;
      const int a_units_t = sparse ? n_here * a_cpr_t : n_rows8 * 8;
      const int b_cpr_t = sparse ? (m_here + kE - 1) / kE : col_chunks;
      const int b_units_t = sparse ? k1 * b_cpr_t : kKC * col_chunks;
      // Tiny stages (<= 4 copies per lane of one warp, e.g. 32 x 32 blocks): each stage is
      // gathered by ONE warp (stage g by warp g % 8, so eight stages are in flight at once and
      // no cross-warp barrier is paid per stage); with 8 ring stages a slot always has the
      // same warp, so its parity waits cannot alias.  Otherwise all 8 warps share each stage.
      const bool tiny = n_stages % kGatherWarps == 0 && a_units_t <= kUnits * 32 && b_units_t <= kUnits * 32;
      // Mid-size stages: two groups of four warps, stage g by group g % 2 (two stages in flight,
      // a 128-thread named barrier per group); with an even ring a slot keeps its group.
      // (only when the group's unit tables hold the stage — m = 128 stages, 8 copies per thread
      //  through the per-unit loops, measured 2.3 -> 3.5 us per stage as two groups)
      const bool grouped = BRK_GATHER_GROUPS && !kTF32 && bf16_in && a_contig && b_contig &&
                           a_units_t <= kUnits * 128 && b_units_t <= kUnits * 128;
      const int gw = tiny ? 1 : (grouped ? 4 : kGatherWarps);  // warps per stage
      const int n_groups = kGatherWarps / gw, grp = warp / gw;
      const int ubase = (warp % gw) * 32 + lane, ustride = gw * 32;
      const bool tab = !kTF32 && bf16_in && a_contig && b_contig && a_units_t <= kUnits * ustride &&
                       b_units_t <= kUnits * ustride &&
                       static_cast<int64_t>(n0 + kRows) * p.b_sn + p.k + kKC < (1ll << 31) &&
                       static_cast<int64_t>(p.k + kKC) * p.a_sk + m0 + kCols < (1ll << 31);
      // (tiny: only a warp that owns one of the tile's stages builds them)
      if (tab && (steps >= n_groups || ((grp - g0) & (n_groups - 1)) < steps)) {
#pragma unroll
        for (int j = 0; j < kUnits; ++j) {
          const int u = ubase + j * ustride;
          ta_dst[j] = -1;
          tb_dst[j] = -1;
          if (u < a_units_t) {
            const int r = sparse ? u / a_cpr_t : u >> 3, c = sparse ? u - r * a_cpr_t : u & 7;
            ta_dst[j] = r * 128 + ((c ^ (r & 7)) << 4);
            ta_src[j] = (n0 + r) * p.b_sn + c * kE;
            ta_kk[j] = r < n_here ? c * kE : (1 << 20);  // rows past the block: zero-filled
          }
          if (u < b_units_t) {
            const int kr = u / b_cpr_t, c = u - kr * b_cpr_t;
            const int col = c * kE;
            const int atom = c / (kAtomCols / kE), cc = c % (kAtomCols / kE);
            tb_dst[j] = b_off + atom * kAtomBytes + kr * 128 + ((cc ^ (kr & 7)) << 4);
            tb_src[j] = kr * p.a_sk + m0 + col;
            tb_kr[j] = kr;
            tb_mc[j] = m_here - col;
          }
        }
      }
      // (this loop runs only when the launch gathers every entry, see `boxes`; tiny: the warp
      // visits only its own stages, g = warp mod 8)
      const int s_first = (grp - g0) & (n_groups - 1), s_step = n_groups;
      for (int s = s_first; s < steps; s += s_step) {
        const int entry = n_chunks == 1 ? s : s / n_chunks;
        const int g = g0 + s, st = g & st_mask;
        const int k0 = (s - entry * n_chunks) * kKC;
        const int k_here = min(kKC, p.k - k0);
        if (g >= n_stages) mbar_wait(&empty[st], ((g >> st_shift) + 1) & 1);
        uint8_t* a_op = smem + st * stage_bytes;
        uint8_t* b_op = a_op + b_off;
        const EntryPtrs e = entry_ptrs(p, job, entry);
        const size_t esz = bf16_in ? 2 : 4;
        const bool a_vec = a_contig && ((reinterpret_cast<uintptr_t>(e.b) & 15) == 0) && ((p.b_sn * esz) % 16 == 0);
        const bool b_vec = b_contig && ((reinterpret_cast<uintptr_t>(e.a) & 15) == 0) && ((p.a_sk * esz) % 16 == 0);
        // bf16 in / bf16 MMA with 16 B-aligned contiguous rows: asynchronous copies (cp.async,
        // zero-filled tails), so each gather thread keeps all ring stages' loads in flight
        const bool fast_a = !kTF32 && bf16_in && a_vec;
        const bool fast_b = !kTF32 && bf16_in && b_vec;
        if (tab && fast_a && fast_b) {
          const uint32_t ring = smem_u32(a_op);
          const char* pa = e.b + static_cast<int64_t>(k0) * 2;
          const char* pb = e.a + static_cast<int64_t>(k0) * p.a_sk * 2;
#pragma unroll
          for (int j = 0; j < kUnits; ++j) {
            if (ta_dst[j] >= 0) {
              const int bytes = max(0, min(16, (k_here - ta_kk[j]) * 2));
              cp_async16(ring + ta_dst[j], bytes > 0 ? pa + static_cast<int64_t>(ta_src[j]) * 2 : e.b, bytes);
            }
            if (tb_dst[j] >= 0) {
              const int bytes = tb_kr[j] < k_here ? max(0, min(16, tb_mc[j] * 2)) : 0;
              cp_async16(ring + tb_dst[j], bytes > 0 ? pb + static_cast<int64_t>(tb_src[j]) * 2 : e.a, bytes);
            }
          }
        } else {
        // A operand (K-major) <- reference b block rows: (row r, 16 B chunk c) along k
        // (sparse: only the n_here rows x chunks holding k)
        const int a_cpr = sparse ? (k_here + kE - 1) / kE : 8;
        const int a_units = sparse ? n_here * a_cpr : n_rows8 * 8;
        for (int u = ubase; u < a_units; u += ustride) {
          const int r = sparse ? u / a_cpr : u >> 3, c = sparse ? u - r * a_cpr : u & 7;
          const int kk = c * kE;
          if (fast_a) {
            const int bytes = r < n_here ? max(0, min(16, (k_here - kk) * 2)) : 0;
            const char* src = bytes > 0 ? e.b + (static_cast<int64_t>(n0 + r) * p.b_sn + (k0 + kk)) * 2 : e.b;
            cp_async16(smem_u32(a_op + r * 128 + ((c ^ (r & 7)) << 4)), src, bytes);
            continue;
          }
          uint4 v;
          if (r < n_here) {
            v = load_chunk<kTF32>(e.b, static_cast<int64_t>(n0 + r) * p.b_sn + static_cast<int64_t>(k0 + kk) * p.b_sk,
                                  p.b_sk, k_here - kk, bf16_in, a_vec && (k0 + kk) % kE == 0);
          } else {
            v = make_uint4(0u, 0u, 0u, 0u);
          }
          *reinterpret_cast<uint4*>(a_op + r * 128 + ((c ^ (r & 7)) << 4)) = v;
        }
        // B operand <- reference a block.  bf16: MN-major, (k-row kr, 16 B chunk c along m);
        // TF32 (K-major only): row i = m index, 16 B chunk c along k (strided gather)
        if constexpr (kTF32) {
          for (int u = ubase; u < n_cols * 8; u += ustride) {
            const int i = u >> 3, c = u & 7;
            const int kk = c * kE;
            const uint4 v = (i < m_here)
                                ? load_chunk<kTF32>(e.a, static_cast<int64_t>(k0 + kk) * p.a_sk +
                                                             static_cast<int64_t>(m0 + i) * p.a_sm,
                                                    p.a_sk, k_here - kk, bf16_in, false)
                                : make_uint4(0u, 0u, 0u, 0u);
            *reinterpret_cast<uint4*>(b_op + i * 128 + ((c ^ (i & 7)) << 4)) = v;
          }
        } else {
          // (sparse: only the k_here K-rows x chunks holding m)
          const int b_cpr = sparse ? (m_here + kE - 1) / kE : col_chunks;
          const int b_units = sparse ? k_here * b_cpr : kKC * col_chunks;
          for (int u = ubase; u < b_units; u += ustride) {
            const int kr = u / b_cpr, c = u - kr * b_cpr;
            const int col = c * kE;
            const int atom = c / (kAtomCols / kE), cc = c % (kAtomCols / kE);
            if (fast_b) {
              const int bytes = kr < k_here ? max(0, min(16, (m_here - col) * 2)) : 0;
              const char* src = bytes > 0 ? e.a + (static_cast<int64_t>(k0 + kr) * p.a_sk + (m0 + col)) * 2 : e.a;
              cp_async16(smem_u32(b_op + atom * kAtomBytes + kr * 128 + ((cc ^ (kr & 7)) << 4)), src, bytes);
              continue;
            }
            uint4 v;
            if (kr < k_here && col < m_here) {
              v = load_chunk<kTF32>(e.a,
                                    static_cast<int64_t>(k0 + kr) * p.a_sk + static_cast<int64_t>(m0 + col) * p.a_sm,
                                    p.a_sm, m_here - col, bf16_in, b_vec && (m0 + col) % kE == 0);
            } else {
              v = make_uint4(0u, 0u, 0u, 0u);
            }
            *reinterpret_cast<uint4*>(b_op + atom * kAtomBytes + kr * 128 + ((cc ^ (kr & 7)) << 4)) = v;
          }
        }
        }  // per-unit loops
        fence_proxy_async_smem();   // this thread's st.shared -> the MMA's async-proxy reads
        cp_async_arrive(&full[st]);  // pending +1 now, -1 when this thread's copies land
        if (gw == 1) {
          __syncwarp();
        } else {
          asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(gw * 32) : "memory");
        }
        if (ubase == 0) mbar_arrive(&full[st]);  // the stage's one expected arrival
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 13-16)
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const float* bias_base = p.bias;
    int local = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++local) {
      const int mt = t % m_tiles;
      const int nt = (t / m_tiles) % n_tiles;
      const int job = t / (m_tiles * n_tiles);
      const int n0 = nt * kRows, m0 = mt * kCols;
      const int m_here = min(kCols, p.m - m0);
      const int n_cols = kTF32 ? (m_here + 15) & ~15 : (m_here + kAtomCols - 1) / kAtomCols * kAtomCols;
      const int acc = local & acc_mask;
      if (steps > 0) {
        mbar_wait(&done[acc], (local >> acc_shift) & 1);
        GEN_TS(local < 16 && threadIdx.x == kEpiWarp0 * 32, 256 + local * 4 + 1);
        tc_fence_after();
      }
      const int row = n0 + quarter * 32 + lane;
      char* c_ptr = p.mode == kModeStride ? static_cast<char*>(p.c_base) + job * p.jstride_c * (p.out_bf16 ? 2 : 4)
                                          : static_cast<char*>(p.c_ptrs[job]);
      const float* bias_row = bias_base != nullptr ? bias_base + p.bias_offs[job] : nullptr;
      const char* mask_ptr = p.mask_ptrs != nullptr ? static_cast<const char*>(p.mask_ptrs[job]) : nullptr;
      // plain fp32 output with 16 B-aligned rows: one float4 store per 4 columns
      // (beta != 0: the lane's row of C is read back as float4 too — the scalar path below
      //  touches 32 rows per warp instruction)
      const bool vec_out = !p.out_bf16 && bias_row == nullptr && mask_ptr == nullptr &&
                           p.act == 0 && (p.ldc & 3) == 0 && (reinterpret_cast<uintptr_t>(c_ptr) & 15) == 0;
      for (int c0 = 0; c0 < n_cols; c0 += 32) {
        uint32_t accv[32];
        if (steps > 0) {
          tmem_ld32(tmem + acc * acc_cols + (static_cast<uint32_t>(quarter * 32) << 16) + c0, accv);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) accv[j] = 0u;
        }
        if (row < p.n && vec_out && m0 + c0 + 32 <= p.m) {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(c_ptr) + static_cast<int64_t>(row) * p.ldc +
                                                  m0 + c0);
          if (p.beta != 0.0f) {
            float4 old[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) old[q] = dst[q];
#pragma unroll
            for (int q = 0; q < 8; ++q)
              dst[q] = make_float4(__fadd_rn(__fmul_rn(p.alpha, __uint_as_float(accv[4 * q])), __fmul_rn(p.beta, old[q].x)),
                                   __fadd_rn(__fmul_rn(p.alpha, __uint_as_float(accv[4 * q + 1])), __fmul_rn(p.beta, old[q].y)),
                                   __fadd_rn(__fmul_rn(p.alpha, __uint_as_float(accv[4 * q + 2])), __fmul_rn(p.beta, old[q].z)),
                                   __fadd_rn(__fmul_rn(p.alpha, __uint_as_float(accv[4 * q + 3])), __fmul_rn(p.beta, old[q].w)));
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q)
              dst[q] = make_float4(p.alpha * __uint_as_float(accv[4 * q]), p.alpha * __uint_as_float(accv[4 * q + 1]),
                                   p.alpha * __uint_as_float(accv[4 * q + 2]), p.alpha * __uint_as_float(accv[4 * q + 3]));
          }
        } else if (row < p.n) {
#pragma unroll 4
        for (int j = 0; j < 32; ++j) {
          const int col = m0 + c0 + j;
          if (col >= p.m) continue;
          const int64_t off = static_cast<int64_t>(row) * p.ldc + col;
          float out = steps > 0 ? p.alpha * __uint_as_float(accv[j]) : 0.0f;
          if (p.beta != 0.0f)
            out = __fadd_rn(out, __fmul_rn(p.beta, p.out_bf16 ? __bfloat162float(reinterpret_cast<__nv_bfloat16*>(c_ptr)[off])
                                        : reinterpret_cast<float*>(c_ptr)[off]));
          if (bias_row != nullptr) out += bias_row[col];
          if (p.act == 1) {
            out = fmaxf(out, 0.0f);
          } else if (p.act == 2) {
            const float ex = __expf(-fabsf(out));
            out = out >= 0.0f ? 1.0f / (1.0f + ex) : ex / (1.0f + ex);
          }
          if (mask_ptr != nullptr) {
            const float mv = p.out_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(mask_ptr)[off])
                                        : reinterpret_cast<const float*>(mask_ptr)[off];
            if (!(mv > 0.0f)) out = 0.0f;
          }
          if (p.out_bf16) reinterpret_cast<__nv_bfloat16*>(c_ptr)[off] = __float2bfloat16_rn(out);
          else reinterpret_cast<float*>(c_ptr)[off] = out;
        }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (steps > 0 && lane == 0) mbar_arrive(&drained[acc]);
      GEN_TS(local < 16 && threadIdx.x == kEpiWarp0 * 32, 256 + local * 4 + 2);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem, 2 * kCols);
  }
}

// Offset / address-with-views launches: is every (job, entry) one in-view box per operand?
// One thread per entry (the same arithmetic as entry_box); an entry that is not clears the
// verdict, which the host set non-zero just before (every writer writes 0: no ordering needed).
__global__ void __launch_bounds__(256) box_check_kernel(const __grid_constant__ GenericParams p, int64_t rows_a,
                                                        int64_t rows_b, int* ok_out) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(p.n_jobs) * p.batch) return;
  const int job = static_cast<int>(idx / p.batch), i = static_cast<int>(idx - static_cast<int64_t>(job) * p.batch);
  int64_t oa, ob;
  bool ok = entry_offs(p, job, i, oa, ob) && oa >= 0 && ob >= 0;
  if (ok) {
    int64_t qa, qb;
    if (((oa | ob) >> 32) == 0) {
      qa = static_cast<uint32_t>(oa) / static_cast<uint32_t>(p.a_sk);
      qb = static_cast<uint32_t>(ob) / static_cast<uint32_t>(p.b_sn);
    } else {
      qa = oa / p.a_sk;
      qb = ob / p.b_sn;
    }
    ok = (oa - qa * p.a_sk) + p.m <= p.a_sk && (ob - qb * p.b_sn) + p.k <= p.b_sn &&
         qa + ((p.k + 31) & ~31) <= rows_a && qb + p.n <= rows_b;
  }
  if (!ok) *ok_out = 0;
}

__device__ int g_box_ok[256];  // one verdict slot per launch (round robin)

// Launch the entry check ahead of a box launch whose entries are not known to be boxes on the
// host; the main kernel reads the verdict (false: the whole launch gathers).
bool attach_box_check(GenericParams& q, uint64_t rows_a, uint64_t rows_b, cudaStream_t stream) {
  static int* slots = nullptr;
  static std::atomic<unsigned> next{0};
  if (slots == nullptr && cudaGetSymbolAddress(reinterpret_cast<void**>(&slots), g_box_ok) != cudaSuccess) {
    slots = nullptr;
    return false;
  }
  int* ok = slots + (next.fetch_add(1) & 255u);
  const int64_t entries = static_cast<int64_t>(q.n_jobs) * q.batch;
  if (cudaMemsetAsync(ok, 1, sizeof(int), stream) != cudaSuccess) return false;  // 0x01010101: true
  g_launches.fetch_add(1);
  box_check_kernel<<<static_cast<unsigned>((entries + 255) / 256), 256, 0, stream>>>(
      q, static_cast<int64_t>(rows_a), static_cast<int64_t>(rows_b), ok);
  q.tma_ok = ok;
  return true;
}

}  // namespace

int launch_brgemm_generic(const GenericParams& p, int compute_tf32, cudaStream_t stream) {
  if (p.n_jobs <= 0 || p.m <= 0 || p.n <= 0) return BRK_OK;
  const int64_t tiles = static_cast<int64_t>((p.m + kCols - 1) / kCols) * ((p.n + kRows - 1) / kRows) * p.n_jobs;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = static_cast<int>(tiles < sms ? tiles : sms);
  // TMA operand fetch: bf16 in and MMA, contiguous rows of 16 B-aligned strides, whole
  // 64-deep K chunks, box extents that stay inside each block (no reads past a block)
  GenericParams q = p;
  q.tma = 0;
  q.sw64 = 0;
#ifdef BRK_DIAG
  q.ts = g_debug_ts;
#else
  q.ts = nullptr;
#endif
  // m = k = 32 blocks (64 B rows): 64B-swizzle boxes, one per operand and entry
  const bool sw64 = p.m == 32 && p.k == 32 && p.n <= kRows;
  const bool rows_ok = (p.n <= kRows || p.n % kRows == 0) && (p.m % kAtomColsBf16 == 0 || sw64);
  const bool addr_views = p.mode == kModeAddr && p.a_view > 0 && p.b_view > 0 && p.a_base != nullptr &&
                          p.b_base != nullptr;
  if (!compute_tf32 && p.in_bf16 && (p.mode != kModeAddr || addr_views) && (p.k % 64 == 0 || sw64) && rows_ok &&
      p.a_sm == 1 &&
      p.b_sk == 1 &&
      (p.a_sk * 2) % 16 == 0 && (p.b_sn * 2) % 16 == 0 && p.a_sk >= p.m && p.b_sn >= p.k &&
      (reinterpret_cast<uintptr_t>(p.a_base) & 15) == 0 && (reinterpret_cast<uintptr_t>(p.b_base) & 15) == 0 &&
      std::getenv("BRK_GENERIC_NO_TMA") == nullptr) {
    q.nbox = std::min(p.n, kRows);
    q.abox = sw64 ? 32 : kAtomColsBf16;
    q.sw64 = sw64 ? 1 : 0;
    // the views span every row an in-bounds offset can address (the kernel reads only boxes
    // inside blocks, so the declared extent is never dereferenced beyond them)
    uint64_t rows_b = std::min<uint64_t>(0x7fffffffull, (1ull << 38) / (p.b_sn * 2));
    uint64_t rows_a = std::min<uint64_t>(0x7fffffffull, (1ull << 38) / (p.a_sk * 2));
    if (addr_views) {  // the views' own extents (rounded up: the kernel bounds-checks each block)
      rows_b = std::min<uint64_t>(rows_b, static_cast<uint64_t>((p.b_view + p.b_sn - 1) / p.b_sn));
      rows_a = std::min<uint64_t>(rows_a, static_cast<uint64_t>((p.a_view + p.a_sk - 1) / p.a_sk));
    }
    const uint64_t db[2] = {static_cast<uint64_t>(p.b_sn), rows_b}, sb[2] = {1, static_cast<uint64_t>(p.b_sn)};
    const uint64_t da[2] = {static_cast<uint64_t>(p.a_sk), rows_a}, sa[2] = {1, static_cast<uint64_t>(p.a_sk)};
    const uint32_t kb = sw64 ? 32 : 64;
    const uint32_t bb[2] = {kb, static_cast<uint32_t>(q.nbox)}, ba[2] = {static_cast<uint32_t>(q.abox), kb};
    if (encode_tmap(&q.map_bop, p.b_base, true, 2, db, sb, bb, false, nullptr, sw64) == BRK_OK &&
        encode_tmap(&q.map_aop, p.a_base, true, 2, da, sa, ba, false, nullptr, sw64) == BRK_OK)
      q.tma = 1;
    q.all_tma = 0;
    if (q.tma && p.mode != kModeStride && !attach_box_check(q, rows_a, rows_b, stream)) q.tma = 0;
    if (q.tma && p.mode == kModeStride && p.stride_a % p.a_sk == 0 && p.jstride_a % p.a_sk == 0 &&
        p.stride_b % p.b_sn == 0 && p.jstride_b % p.b_sn == 0 &&
        static_cast<int64_t>(p.n_jobs) * (p.jstride_a / p.a_sk + p.batch * (p.stride_a / p.a_sk)) < (1ll << 31) &&
        static_cast<int64_t>(p.n_jobs) * (p.jstride_b / p.b_sn + p.batch * (p.stride_b / p.b_sn)) < (1ll << 31)) {
      q.all_tma = 1;
      q.rs_a = p.stride_a / p.a_sk;
      q.rj_a = p.jstride_a / p.a_sk;
      q.rs_b = p.stride_b / p.b_sn;
      q.rj_b = p.jstride_b / p.b_sn;
    }
  }
  // TF32 on fp32 blocks: the stride variant whose blocks start at view column 0 (every entry
  // one box per operand; the kernel rounds the landed stages to TF32 in place)
  if (compute_tf32 && !p.in_bf16 && p.mode == kModeStride && p.k % 32 == 0 &&
      (p.n <= kRows || p.n % kRows == 0) && p.m % 32 == 0 && p.a_sm == 1 && p.b_sk == 1 && (p.a_sk * 4) % 16 == 0 &&
      (p.b_sn * 4) % 16 == 0 && p.a_sk >= p.m && p.b_sn >= p.k && p.stride_a % p.a_sk == 0 &&
      p.jstride_a % p.a_sk == 0 && p.stride_b % p.b_sn == 0 && p.jstride_b % p.b_sn == 0 &&
      static_cast<int64_t>(p.n_jobs) * (p.jstride_a / p.a_sk + p.batch * (p.stride_a / p.a_sk)) < (1ll << 31) &&
      static_cast<int64_t>(p.n_jobs) * (p.jstride_b / p.b_sn + p.batch * (p.stride_b / p.b_sn)) < (1ll << 31) &&
      (reinterpret_cast<uintptr_t>(p.a_base) & 15) == 0 && (reinterpret_cast<uintptr_t>(p.b_base) & 15) == 0 &&
      std::getenv("BRK_GENERIC_NO_TMA") == nullptr) {
    q.nbox = std::min(p.n, kRows);
    q.abox = 32;
    const uint64_t rows_b = std::min<uint64_t>(0x7fffffffull, (1ull << 38) / (p.b_sn * 4));
    const uint64_t rows_a = std::min<uint64_t>(0x7fffffffull, (1ull << 38) / (p.a_sk * 4));
    const uint64_t db[2] = {static_cast<uint64_t>(p.b_sn), rows_b}, sb[2] = {1, static_cast<uint64_t>(p.b_sn)};
    const uint64_t da[2] = {static_cast<uint64_t>(p.a_sk), rows_a}, sa[2] = {1, static_cast<uint64_t>(p.a_sk)};
    const uint32_t bb[2] = {32, static_cast<uint32_t>(q.nbox)}, ba[2] = {32, 32};
    if (encode_tmap(&q.map_bop, p.b_base, false, 2, db, sb, bb) == BRK_OK &&
        encode_tmap(&q.map_aop, p.a_base, false, 2, da, sa, ba, /*atom32=*/true) == BRK_OK) {
      q.tma = 1;
      q.all_tma = 1;
      q.rs_a = p.stride_a / p.a_sk;
      q.rj_a = p.jstride_a / p.a_sk;
      q.rs_b = p.stride_b / p.b_sn;
      q.rj_b = p.jstride_b / p.b_sn;
    }
  }
  // TF32 offset variant / address variant with views: the same TMA path when a check kernel
  // finds every entry one in-view box per operand (otherwise the launch gathers, as before)
  const bool tf32_views = p.mode == kModeOffs || addr_views;
  if (compute_tf32 && !q.tma && !p.in_bf16 && tf32_views && p.k % 32 == 0 && (p.n <= kRows || p.n % kRows == 0) &&
      p.m % 32 == 0 && p.a_sm == 1 && p.b_sk == 1 && (p.a_sk * 4) % 16 == 0 && (p.b_sn * 4) % 16 == 0 &&
      p.a_sk >= p.m && p.b_sn >= p.k && (reinterpret_cast<uintptr_t>(p.a_base) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(p.b_base) & 15) == 0 && std::getenv("BRK_GENERIC_NO_TMA") == nullptr) {
    q.nbox = std::min(p.n, kRows);
    q.abox = 32;
    uint64_t rows_b = std::min<uint64_t>(0x7fffffffull, (1ull << 38) / (p.b_sn * 4));
    uint64_t rows_a = std::min<uint64_t>(0x7fffffffull, (1ull << 38) / (p.a_sk * 4));
    if (addr_views) {
      rows_b = std::min<uint64_t>(rows_b, static_cast<uint64_t>((p.b_view + p.b_sn - 1) / p.b_sn));
      rows_a = std::min<uint64_t>(rows_a, static_cast<uint64_t>((p.a_view + p.a_sk - 1) / p.a_sk));
    }
    const uint64_t db[2] = {static_cast<uint64_t>(p.b_sn), rows_b}, sb[2] = {1, static_cast<uint64_t>(p.b_sn)};
    const uint64_t da[2] = {static_cast<uint64_t>(p.a_sk), rows_a}, sa[2] = {1, static_cast<uint64_t>(p.a_sk)};
    const uint32_t bb[2] = {32, static_cast<uint32_t>(q.nbox)}, ba[2] = {32, 32};
    if (encode_tmap(&q.map_bop, p.b_base, false, 2, db, sb, bb) == BRK_OK &&
        encode_tmap(&q.map_aop, p.a_base, false, 2, da, sa, ba, /*atom32=*/true) == BRK_OK &&
        attach_box_check(q, rows_a, rows_b, stream)) {
      q.tma = 1;
      q.all_tma = 0;
    }
  }
  cudaError_t err;
  if (compute_tf32) {
    err = cudaFuncSetAttribute(brgemm_generic_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (err == cudaSuccess) brgemm_generic_kernel<true><<<grid, kThreads, kSmemBytes, stream>>>(q);
  } else {
    err = cudaFuncSetAttribute(brgemm_generic_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (err == cudaSuccess) brgemm_generic_kernel<false><<<grid, kThreads, kSmemBytes, stream>>>(q);
  }
  if (err == cudaSuccess) err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error(err, "brgemm_generic launch");
  return BRK_OK;
}

}  // namespace brk
