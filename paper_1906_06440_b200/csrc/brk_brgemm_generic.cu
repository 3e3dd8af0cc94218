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

constexpr int kRows = 128;        // C rows (reference n) per CTA = MMA M
constexpr int kCols = 256;        // C cols (reference m) per CTA = max MMA N
constexpr int kChunkBytes = 128;  // K bytes staged per step (one 128B row)
constexpr int kThreads = 128;
constexpr int kStages = 2;
constexpr int kAOpBytes = kRows * kChunkBytes;  // 16 KB
constexpr int kBOpBytes = kCols * kChunkBytes;  // 32 KB
constexpr int kStageBytes = kAOpBytes + kBOpBytes;
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align slack*/ + 256 /*barriers*/;

// canonical SWIZZLE_NONE K-major: core matrix = 8 rows x 16 B (128 B contiguous);
// K-adjacent cores at LBO = 128 B, 8-row groups at SBO = 1024 B.
__device__ __forceinline__ uint32_t canon_off(int row, int chunk16) {
  return static_cast<uint32_t>((row >> 3) * 1024 + chunk16 * 128 + (row & 7) * 16);
}

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
  if (bf16) {
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[idx]);
  }
  return reinterpret_cast<const float*>(base)[idx];
}

template <bool kTF32>
__device__ __forceinline__ uint4 pack16(const float* v) {
  uint4 r;
  if constexpr (kTF32) {
    r.x = f32_to_tf32(v[0]);
    r.y = f32_to_tf32(v[1]);
    r.z = f32_to_tf32(v[2]);
    r.w = f32_to_tf32(v[3]);
  } else {
    r.x = pack_bf16x2(v[0], v[1]);
    r.y = pack_bf16x2(v[2], v[3]);
    r.z = pack_bf16x2(v[4], v[5]);
    r.w = pack_bf16x2(v[6], v[7]);
  }
  return r;
}

template <bool kTF32>
__global__ void __launch_bounds__(kThreads, 1) brgemm_generic_kernel(const GenericParams p) {
  constexpr int kElems = kTF32 ? 4 : 8;            // elements per 16 B chunk
  constexpr int kChunkElems = kChunkBytes / (kTF32 ? 4 : 2);
  constexpr int kMmaK = kTF32 ? 8 : 16;            // K per tcgen05.mma (32 B)
  constexpr int kMmaPerChunk = kChunkElems / kMmaK;  // = 4

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);  // [kStages] + done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kStages + 1);

  const int tid = threadIdx.x;
  const int warp = tid / 32;
  const int lane = tid % 32;
  const int job = blockIdx.z;
  const int n0 = blockIdx.y * kRows;
  const int m0 = blockIdx.x * kCols;
  const int m_here = min(kCols, p.m - m0);
  const int n_cols = (m_here + 15) & ~15;  // MMA N: multiple of 16 for M=128

  if (tid == 0) {
    for (int s = 0; s < kStages + 1; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const bool bf16_in = p.in_bf16 != 0;
  const int n_chunks = (p.k + kChunkElems - 1) / kChunkElems;
  const int steps = (p.alpha == 0.0f) ? 0 : p.batch * n_chunks;
  const uint32_t idesc = make_idesc(kTF32 ? kFmtTF32 : kFmtBF16, kRows, n_cols, 0, 0);

  for (int s = 0; s < steps; ++s) {
    const int st = s % kStages;
    const int entry = s / n_chunks;
    const int k0 = (s % n_chunks) * kChunkElems;
    if (s >= kStages) mbar_wait(&bars[st], ((s / kStages) + 1) & 1);
    uint8_t* a_op = smem + st * kStageBytes;
    uint8_t* b_op = a_op + kAOpBytes;
    const EntryPtrs e = entry_ptrs(p, job, entry);
    // A operand <- reference b block rows (n, k): row r, 16B chunk c
    for (int u = tid; u < kRows * 8; u += kThreads) {
      const int c = u & 7, r = u >> 3;
      const int row = n0 + r;
      float v[8];
#pragma unroll
      for (int t = 0; t < kElems; ++t) {
        const int kk = k0 + c * kElems + t;
        v[t] = (row < p.n && kk < p.k) ? load_in(e.b, static_cast<int64_t>(row) * p.b_sn + static_cast<int64_t>(kk) * p.b_sk, bf16_in)
                                       : 0.0f;
      }
      *reinterpret_cast<uint4*>(a_op + canon_off(r, c)) = pack16<kTF32>(v);
    }
    // B operand <- reference a block (k, m) transposed: row i (m index), 16B chunk c
    for (int u = tid; u < kCols * 8; u += kThreads) {
      const int i = u % kCols, c = u / kCols;
      const int col = m0 + i;
      float v[8];
#pragma unroll
      for (int t = 0; t < kElems; ++t) {
        const int kk = k0 + c * kElems + t;
        v[t] = (col < p.m && kk < p.k) ? load_in(e.a, static_cast<int64_t>(kk) * p.a_sk + static_cast<int64_t>(col) * p.a_sm, bf16_in)
                                       : 0.0f;
      }
      *reinterpret_cast<uint4*>(b_op + canon_off(i, c)) = pack16<kTF32>(v);
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t a_base = smem_u32(a_op), b_base = smem_u32(b_op);
#pragma unroll
      for (int kk = 0; kk < kMmaPerChunk; ++kk) {
        const uint64_t ad = make_smem_desc(a_base + kk * 256, 128, 1024, kSwizzleNone);
        const uint64_t bd = make_smem_desc(b_base + kk * 256, 128, 1024, kSwizzleNone);
        mma_ss<kTF32>(tmem, ad, bd, idesc, (s > 0 || kk > 0) ? 1u : 0u);
      }
      mma_commit(&bars[st]);
      if (s == steps - 1) mma_commit(&bars[kStages]);
    }
  }

  // ---- epilogue: TMEM -> registers -> alpha/beta -> C -------------------------
  if (steps > 0) {
    mbar_wait(&bars[kStages], 0);
    tc_fence_after();
  }
  const int row = n0 + warp * 32 + lane;
  char* c_ptr;
  if (p.mode == kModeStride) {
    c_ptr = static_cast<char*>(p.c_base) + job * p.jstride_c * (p.out_bf16 ? 2 : 4);
  } else {
    c_ptr = static_cast<char*>(p.c_ptrs[job]);
  }
  const double alpha = p.alpha, beta = p.beta;
  const float* bias_row = p.bias != nullptr ? p.bias + p.bias_offs[job] : nullptr;
  const char* mask_ptr = p.mask_ptrs != nullptr ? static_cast<const char*>(p.mask_ptrs[job]) : nullptr;
  for (int c0 = 0; c0 < n_cols; c0 += 32) {
    uint32_t acc[32];
    if (steps > 0) {
      tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, acc);
      tmem_ld_wait();
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0u;
    }
    if (row < p.n) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int col = m0 + c0 + j;
        if (col < p.m) {
          const int64_t off = static_cast<int64_t>(row) * p.ldc + col;
          double out = alpha * static_cast<double>(__uint_as_float(acc[j]));
          if (steps == 0) out = 0.0;
          if (beta != 0.0) {
            const double old = p.out_bf16 ? __bfloat162float(reinterpret_cast<__nv_bfloat16*>(c_ptr)[off])
                                          : reinterpret_cast<float*>(c_ptr)[off];
            out += beta * old;
          }
          if (bias_row != nullptr) out += static_cast<double>(bias_row[col]);
          if (p.act == 1) {
            out = out > 0.0 ? out : 0.0;
          } else if (p.act == 2) {
            const double e = exp(-fabs(out));
            out = out >= 0.0 ? 1.0 / (1.0 + e) : e / (1.0 + e);
          }
          if (mask_ptr != nullptr) {
            const float mv = p.out_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(mask_ptr)[off])
                                        : reinterpret_cast<const float*>(mask_ptr)[off];
            if (!(mv > 0.0f)) out = 0.0;
          }
          if (p.out_bf16) {
            reinterpret_cast<__nv_bfloat16*>(c_ptr)[off] = __float2bfloat16_rn(static_cast<float>(out));
          } else {
            reinterpret_cast<float*>(c_ptr)[off] = static_cast<float>(out);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, kCols);
}

}  // namespace

int launch_brgemm_generic(const GenericParams& p, int compute_tf32, cudaStream_t stream) {
  if (p.n_jobs <= 0 || p.m <= 0 || p.n <= 0) return BRK_OK;
  dim3 grid((p.m + kCols - 1) / kCols, (p.n + kRows - 1) / kRows, p.n_jobs);
  if (grid.z > 65535) return set_error(BRK_ERR_CONTRACT, "too many jobs in one launch (max 65535)");
  cudaError_t err;
  if (compute_tf32) {
    err = cudaFuncSetAttribute(brgemm_generic_kernel<true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (err == cudaSuccess) brgemm_generic_kernel<true><<<grid, kThreads, kSmemBytes, stream>>>(p);
  } else {
    err = cudaFuncSetAttribute(brgemm_generic_kernel<false>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (err == cudaSuccess) brgemm_generic_kernel<false><<<grid, kThreads, kSmemBytes, stream>>>(p);
  }
  if (err == cudaSuccess) err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error(err, "brgemm_generic launch");
  return BRK_OK;
}

}  // namespace brk
