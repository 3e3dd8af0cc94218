// brk_internal.h — shared host/device declarations behind the C-ABI (include/brk.h).
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/brk.h"

namespace brk {

// diagnostics: engine launches record %globaltimer stamps / wait sums here when set
// (brk_diag_set_timestamps; only the BRK_DIAG build writes them)
extern unsigned long long* g_debug_ts;

enum EntryMode : int { kModeAddr = 0, kModeOffs = 1, kModeStride = 2 };

// Parameters of one generic BRGEMM launch (see brk_brgemm_generic.cu).
struct GenericParams {
  // TMA path (set by launch_brgemm_generic, not by the callers): 2-d views of the
  // reference b buffer ([rows][b_sn], box 64 k x nbox rows) and of the reference a
  // buffer ([rows][a_sk], box abox m x 64 k), 128B swizzle.  An entry whose block
  // start (element offset o) satisfies o % ld + extent <= ld is one box per operand
  // at (o % ld + k0, o / ld + row0).  A launch boxes every entry or gathers every entry
  // (tma_ok: the device check of the offset / address tables).
  alignas(64) CUtensorMap map_bop;
  alignas(64) CUtensorMap map_aop;
  int tma, nbox, abox;
  // m = k = 32 blocks: 64 B rows, 64B-swizzle boxes of 32 elements (A: 32 k x nbox rows,
  // B: 32 m x 32 k), compact stages, MMA N = 32
  int sw64;
  // diagnostics build: CTA 0 stamps (%globaltimer) of its first 64 stages / 16 tiles, or null
  unsigned long long* ts;
  // stride variant whose block starts all sit at column 0 of the views: every entry is one
  // box per operand at view row job * rj + i * rs (no per-entry division, no gather work)
  int all_tma;
  int64_t rs_a, rj_a, rs_b, rj_b;
  // offset / address-with-views launches: device flag written by a check kernel just before
  // (1: every entry is one in-view box per operand, so the launch runs like all_tma)
  const int* tma_ok;
  int mode;    // EntryMode
  int n_jobs;  // number of independent output blocks C_j
  int m, n, k, batch;
  int64_t lda, ldb, ldc;
  // element strides of one block: A element (kk, col) at a[kk*a_sk + col*a_sm],
  // B element (row, kk) at b[row*b_sn + kk*b_sk]  (a_sk = lda, a_sm = 1 by default)
  int64_t a_sk, a_sm, b_sn, b_sk;
  float alpha, beta;
  int in_bf16;   // A/B storage: 0 = fp32, 1 = bf16
  int out_bf16;  // C storage:   0 = fp32, 1 = bf16
  // mode == kModeAddr: device tables of n_jobs*batch block addresses
  const void* const* a_ptrs;
  const void* const* b_ptrs;
  // mode == kModeOffs / kModeStride: base pointers
  const void* a_base;
  const void* b_base;
  // mode == kModeAddr with views (brk_brgemm_addr_views): a_base/b_base are allocations of
  // a_view/b_view elements that hold the blocks; an entry whose pointers fall inside them
  // (element-aligned, block in bounds) is fetched by TMA like an offset entry
  int64_t a_view, b_view;
  // mode == kModeOffs: device tables of n_jobs*batch element offsets
  const int64_t* a_offs;
  const int64_t* b_offs;
  // mode == kModeStride: block i of job j at base + j*jstride + i*stride (elements)
  int64_t stride_a, stride_b;
  int64_t jstride_a, jstride_b, jstride_c;
  // outputs: mode Addr/Offs use c_ptrs[n_jobs]; mode Stride uses c_base + j*jstride_c
  void* const* c_ptrs;
  void* c_base;
  // fused epilogue: out = act(alpha*acc + beta*c + bias[bias_offs[j] + col])
  int act;                  // 0 none, 1 relu, 2 sigmoid
  const float* bias;        // may be null
  const int64_t* bias_offs; // per job (device), used when bias != null
  const void* const* mask_ptrs;  // per job, layout of C (ldc), dtype of C; out *= (mask > 0)
};

extern std::atomic<uint64_t> g_launches;

int launch_brgemm_generic(const GenericParams& p, int compute_tf32, cudaStream_t stream);

// error reporting (thread-local message, returned by brk_last_error())
int set_error(int code, const char* msg);
int set_cuda_error(cudaError_t err, const char* where);

}  // namespace brk
