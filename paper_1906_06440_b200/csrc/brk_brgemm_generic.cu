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
#include "brk_internal.h"
#include "brk_ptx.cuh"

namespace brk {
namespace {

constexpr int kRows = 128;         // C rows (reference n) per tile = MMA M
constexpr int kCols = 256;         // C cols (reference m) per tile = max MMA N
constexpr int kGatherWarps = 8;    // gather + epilogue warps
constexpr int kThreads = (kGatherWarps + 1) * 32;  // + 1 MMA warp
constexpr int kStages = 4;
constexpr int kAOpBytes = kRows * 128;    // K-major, 128B swizzle: 128 rows x 128 B of K
constexpr int kBOpBytes = kCols * 128;    // MN-major, 128B swizzle atoms: up to 256 cols
constexpr int kStageBytes = kAOpBytes + kBOpBytes;
constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256;

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

// Persistent: CTA walks job tiles (job, n-tile, m-tile).  Warps 0-7 gather the
// (reference b block, reference a block) pair of each batch entry into a
// 4-stage ring (reference b rows -> K-major 128B-swizzled A operand, reference
// a rows -> MN-major 128B-swizzled B operand: both straight 16 B copies along
// the contiguous dimension, vector loads when aligned), warp 8 issues the
// tcgen05.mma chain (the whole batch reduces in TMEM), and warps 0-7 drain
// TMEM and apply alpha/beta/bias/act/mask.
template <bool kTF32>
__global__ void __launch_bounds__(kThreads, 1) brgemm_generic_kernel(const GenericParams p) {
  constexpr int kE = kTF32 ? 4 : 8;              // elements per 16 B
  constexpr int kKC = kTF32 ? 32 : 64;           // K elements per stage (128 B)
  constexpr int kMmaK = kTF32 ? 8 : 16;          // K per tcgen05.mma
  constexpr int kAtomCols = kTF32 ? 32 : 64;     // MN elements per 128 B atom row
  constexpr int kAtomBytes = kKC * 128;          // one MN-major atom: kKC K-rows x 128 B

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* done = empty + kStages;  // accumulator complete
  uint64_t* drained = done + 1;      // epilogue finished reading TMEM
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(drained + 1);

  const int tid = threadIdx.x;
  const int warp = tid / 32;
  const int lane = tid % 32;
  const int m_tiles = (p.m + kCols - 1) / kCols;
  const int n_tiles = (p.n + kRows - 1) / kRows;
  const int tiles = m_tiles * n_tiles * p.n_jobs;
  const bool bf16_in = p.in_bf16 != 0;
  const int n_chunks = (p.k + kKC - 1) / kKC;
  const int steps = (p.alpha == 0.0f) ? 0 : p.batch * n_chunks;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], kGatherWarps);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    mbar_init(drained, kGatherWarps);
    fence_barrier_init();
  }
  if (warp == kGatherWarps) tmem_alloc(tmem_slot, kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  int local = 0;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++local) {
    const int mt = t % m_tiles;
    const int nt = (t / m_tiles) % n_tiles;
    const int job = t / (m_tiles * n_tiles);
    const int n0 = nt * kRows, m0 = mt * kCols;
    const int m_here = min(kCols, p.m - m0);
    const int n_here = min(kRows, p.n - n0);
    // MMA N: bf16 B operand is MN-major (whole 128 B swizzle atoms, zero-filled past m);
    // TF32 operands must be K-major (multiple of 16 rows)
    const int n_cols = kTF32 ? (m_here + 15) & ~15 : (m_here + kAtomCols - 1) / kAtomCols * kAtomCols;
    const int g0 = local * steps;             // global step index of this tile's first step

    if (warp == kGatherWarps) {
      // ---------------------------------------------------------- MMA issuer
      const uint32_t idesc = make_idesc(kTF32 ? kFmtTF32 : kFmtBF16, kRows, n_cols, 0, kTF32 ? 0 : 1);
      if (steps > 0) mbar_wait(drained, (local & 1) ^ 1);  // the previous tile's accumulator was read
      tc_fence_after();
      for (int s = 0; s < steps; ++s) {
        const int g = g0 + s, st = g % kStages;
        mbar_wait(&full[st], (g / kStages) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a_base = smem_u32(smem + st * kStageBytes);
          const uint32_t b_base = a_base + kAOpBytes;
#pragma unroll
          for (int kk = 0; kk < kKC / kMmaK; ++kk) {
            const uint64_t ad = make_smem_desc(a_base + kk * 32, 16, 1024, kSwizzle128B);
            const uint64_t bd = kTF32 ? make_smem_desc(b_base + kk * 32, 16, 1024, kSwizzle128B)
                                      : make_smem_desc(b_base + kk * kMmaK * 128, kAtomBytes, 1024, kSwizzle128B);
            mma_ss<kTF32>(tmem, ad, bd, idesc, (s > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&empty[st]);
          if (s == steps - 1) mma_commit(done);
        }
        __syncwarp();
      }
    } else {
      // ---------------------------------------------------------- gather
      const int gt = tid;  // 0 .. 255
      const bool a_contig = p.b_sk == 1;   // reference b block: k contiguous
      const bool b_contig = p.a_sm == 1;   // reference a block: m contiguous
      const int n_rows8 = (n_here + 7) & ~7;
      const int col_chunks = n_cols / kE;
      for (int s = 0; s < steps; ++s) {
        const int g = g0 + s, st = g % kStages;
        const int entry = s / n_chunks;
        const int k0 = (s % n_chunks) * kKC;
        const int k_here = min(kKC, p.k - k0);
        if (g >= kStages) mbar_wait(&empty[st], ((g / kStages) + 1) & 1);
        uint8_t* a_op = smem + st * kStageBytes;
        uint8_t* b_op = a_op + kAOpBytes;
        const EntryPtrs e = entry_ptrs(p, job, entry);
        const size_t esz = bf16_in ? 2 : 4;
        const bool a_vec = a_contig && ((reinterpret_cast<uintptr_t>(e.b) & 15) == 0) && ((p.b_sn * esz) % 16 == 0);
        const bool b_vec = b_contig && ((reinterpret_cast<uintptr_t>(e.a) & 15) == 0) && ((p.a_sk * esz) % 16 == 0);
        // A operand (K-major) <- reference b block rows: (row r, 16 B chunk c) along k
        for (int u = gt; u < n_rows8 * 8; u += kGatherWarps * 32) {
          const int c = u & 7, r = u >> 3;
          const int kk = c * kE;
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
          for (int u = gt; u < n_cols * 8; u += kGatherWarps * 32) {
            const int i = u >> 3, c = u & 7;
            const int kk = c * kE;
            const uint4 v = (i < m_here)
                                ? load_chunk<kTF32>(e.a, static_cast<int64_t>(k0 + kk) * p.a_sk +
                                                             static_cast<int64_t>(m0 + i) * p.a_sm,
                                                    p.a_sk, k_here - kk, bf16_in, false)
                                : make_uint4(0u, 0u, 0u, 0u);
            *reinterpret_cast<uint4*>(b_op + i * 128 + ((c ^ (i & 7)) << 4)) = v;
          }
        } else
        for (int u = gt; u < kKC * col_chunks; u += kGatherWarps * 32) {
          const int kr = u / col_chunks, c = u - kr * col_chunks;
          const int col = c * kE;
          uint4 v;
          if (kr < k_here && col < m_here) {
            v = load_chunk<kTF32>(e.a, static_cast<int64_t>(k0 + kr) * p.a_sk + static_cast<int64_t>(m0 + col) * p.a_sm,
                                  p.a_sm, m_here - col, bf16_in, b_vec && (m0 + col) % kE == 0);
          } else {
            v = make_uint4(0u, 0u, 0u, 0u);
          }
          const int atom = c / (kAtomCols / kE), cc = c % (kAtomCols / kE);
          *reinterpret_cast<uint4*>(b_op + atom * kAtomBytes + kr * 128 + ((cc ^ (kr & 7)) << 4)) = v;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[st]);
      }
      // ---------------------------------------------------------- epilogue
      if (steps > 0) {
        mbar_wait(done, local & 1);
        tc_fence_after();
      }
      const int quarter = warp & 3, half = warp >> 2;
      const int row = n0 + quarter * 32 + lane;
      char* c_ptr = p.mode == kModeStride ? static_cast<char*>(p.c_base) + job * p.jstride_c * (p.out_bf16 ? 2 : 4)
                                          : static_cast<char*>(p.c_ptrs[job]);
      const float* bias_row = p.bias != nullptr ? p.bias + p.bias_offs[job] : nullptr;
      const char* mask_ptr = p.mask_ptrs != nullptr ? static_cast<const char*>(p.mask_ptrs[job]) : nullptr;
      for (int c0 = half * 128; c0 < min(n_cols, half * 128 + 128); c0 += 32) {
        uint32_t acc[32];
        if (steps > 0) {
          tmem_ld32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + c0, acc);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[j] = 0u;
        }
        if (row < p.n) {
#pragma unroll 4
          for (int j = 0; j < 32; ++j) {
            const int col = m0 + c0 + j;
            if (col >= p.m) continue;
            const int64_t off = static_cast<int64_t>(row) * p.ldc + col;
            float out = steps > 0 ? p.alpha * __uint_as_float(acc[j]) : 0.0f;
            if (p.beta != 0.0f)
              out += p.beta * (p.out_bf16 ? __bfloat162float(reinterpret_cast<__nv_bfloat16*>(c_ptr)[off])
                                          : reinterpret_cast<float*>(c_ptr)[off]);
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
      if (lane == 0) mbar_arrive(drained);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kGatherWarps) {
    tc_fence_after();
    tmem_dealloc(tmem, kCols);
  }
}

}  // namespace

int launch_brgemm_generic(const GenericParams& p, int compute_tf32, cudaStream_t stream) {
  if (p.n_jobs <= 0 || p.m <= 0 || p.n <= 0) return BRK_OK;
  const int64_t tiles = static_cast<int64_t>((p.m + kCols - 1) / kCols) * ((p.n + kRows - 1) / kRows) * p.n_jobs;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = static_cast<int>(tiles < sms ? tiles : sms);
  cudaError_t err;
  if (compute_tf32) {
    err = cudaFuncSetAttribute(brgemm_generic_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (err == cudaSuccess) brgemm_generic_kernel<true><<<grid, kThreads, kSmemBytes, stream>>>(p);
  } else {
    err = cudaFuncSetAttribute(brgemm_generic_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (err == cudaSuccess) brgemm_generic_kernel<false><<<grid, kThreads, kSmemBytes, stream>>>(p);
  }
  if (err == cudaSuccess) err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error(err, "brgemm_generic launch");
  return BRK_OK;
}

}  // namespace brk
