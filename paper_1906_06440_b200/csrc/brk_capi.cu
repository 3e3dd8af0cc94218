// brk_capi.cu — extern "C" entry points of libbrk_sm100.so (declared in include/brk.h).
#include <atomic>
#include <cstdio>
#include <cstring>
#include <string>

#include "brk_internal.h"

namespace brk {

static thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

int set_error(int code, const char* msg) {
  g_last_error = msg;
  return code;
}

int set_cuda_error(cudaError_t err, const char* where) {
  char buf[512];
  std::snprintf(buf, sizeof(buf), "%s: %s (%s)", where, cudaGetErrorString(err),
                cudaGetErrorName(err));
  g_last_error = buf;
  return BRK_ERR_CUDA;
}

static int check_common(int m, int n, int k, int batch, int64_t lda, int64_t ldb, int64_t ldc,
                        int in_dtype, int out_dtype, int compute, int n_jobs) {
  char buf[256];
  if (m < 0 || n < 0 || k < 0 || batch < 0 || n_jobs < 0) {
    std::snprintf(buf, sizeof(buf), "extents must be >= 0 (m=%d n=%d k=%d batch=%d jobs=%d)", m, n,
                  k, batch, n_jobs);
    return set_error(BRK_ERR_CONTRACT, buf);
  }
  if (lda < m || ldb < k || ldc < m) {
    std::snprintf(buf, sizeof(buf), "leading dimensions too small (lda=%lld m=%d ldb=%lld k=%d ldc=%lld)",
                  (long long)lda, m, (long long)ldb, k, (long long)ldc);
    return set_error(BRK_ERR_CONTRACT, buf);
  }
  if ((in_dtype != BRK_F32 && in_dtype != BRK_BF16) || (out_dtype != BRK_F32 && out_dtype != BRK_BF16))
    return set_error(BRK_ERR_CONTRACT, "dtype must be BRK_F32 or BRK_BF16");
  if (compute != BRK_COMPUTE_TF32 && compute != BRK_COMPUTE_BF16)
    return set_error(BRK_ERR_CONTRACT, "compute must be BRK_COMPUTE_TF32 or BRK_COMPUTE_BF16");
  if (compute == BRK_COMPUTE_TF32 && in_dtype == BRK_BF16)
    return set_error(BRK_ERR_CONTRACT, "TF32 compute needs fp32 inputs");
  return BRK_OK;
}

static int run_generic(GenericParams& p, int compute, void* stream) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return launch_brgemm_generic(p, compute == BRK_COMPUTE_TF32, static_cast<cudaStream_t>(stream));
}

}  // namespace brk

using namespace brk;

extern "C" {

BRK_API int brk_brgemm_grouped(const brk_grouped_desc* d, void* stream) {
  if (d == nullptr) return set_error(BRK_ERR_CONTRACT, "null descriptor");
  int rc = check_common(d->m, d->n, d->k, d->batch, d->m, d->k, d->ldc, d->in_dtype, d->out_dtype,
                        d->compute, d->n_jobs);
  if (rc) return rc;
  if (d->act < 0 || d->act > 2) return set_error(BRK_ERR_CONTRACT, "unknown activation");
  if (d->n_jobs == 0 || d->m == 0 || d->n == 0) return BRK_OK;
  if (d->c_ptrs == nullptr || (d->batch > 0 && (d->a_ptrs == nullptr || d->b_ptrs == nullptr)))
    return set_error(BRK_ERR_CONTRACT, "null pointer table");
  if (d->bias != nullptr && d->bias_offs == nullptr) return set_error(BRK_ERR_CONTRACT, "bias needs bias_offs");
  GenericParams p{};
  p.mode = kModeAddr;
  p.n_jobs = d->n_jobs;
  p.m = d->m; p.n = d->n; p.k = d->k; p.batch = d->batch;
  p.lda = d->a_sk; p.ldb = d->b_sn; p.ldc = d->ldc;
  p.a_sk = d->a_sk; p.a_sm = d->a_sm; p.b_sn = d->b_sn; p.b_sk = d->b_sk;
  p.alpha = d->alpha; p.beta = d->beta;
  p.in_bf16 = d->in_dtype == BRK_BF16;
  p.out_bf16 = d->out_dtype == BRK_BF16;
  p.a_ptrs = d->a_ptrs; p.b_ptrs = d->b_ptrs; p.c_ptrs = d->c_ptrs;
  p.bias = d->bias; p.bias_offs = d->bias_offs; p.act = d->act;
  p.mask_ptrs = d->mask_ptrs;
  return run_generic(p, d->compute, stream);
}

const char* brk_last_error(void) { return g_last_error.c_str(); }

int brk_version(void) { return 1; }

uint64_t brk_launch_count(void) { return g_launches.load(); }

int brk_brgemm_addr(const void* const* a_ptrs, const void* const* b_ptrs, void* const* c_ptrs,
                    int n_jobs, int m, int n, int k, int batch, int64_t lda, int64_t ldb,
                    int64_t ldc, float alpha, float beta, int in_dtype, int out_dtype, int compute,
                    void* stream) {
  int rc = check_common(m, n, k, batch, lda, ldb, ldc, in_dtype, out_dtype, compute, n_jobs);
  if (rc) return rc;
  if (n_jobs == 0 || m == 0 || n == 0) return BRK_OK;
  if (c_ptrs == nullptr || (batch > 0 && (a_ptrs == nullptr || b_ptrs == nullptr)))
    return set_error(BRK_ERR_CONTRACT, "null pointer table");
  GenericParams p{};
  p.mode = kModeAddr;
  p.n_jobs = n_jobs;
  p.m = m; p.n = n; p.k = k; p.batch = batch;
  p.lda = lda; p.ldb = ldb; p.ldc = ldc;
  p.a_sk = lda; p.a_sm = 1; p.b_sn = ldb; p.b_sk = 1;
  p.alpha = alpha; p.beta = beta;
  p.in_bf16 = in_dtype == BRK_BF16;
  p.out_bf16 = out_dtype == BRK_BF16;
  p.a_ptrs = a_ptrs; p.b_ptrs = b_ptrs; p.c_ptrs = c_ptrs;
  return run_generic(p, compute, stream);
}

int brk_brgemm_addr_views(const void* const* a_ptrs, const void* const* b_ptrs, void* const* c_ptrs,
                          const void* a_view, int64_t a_view_elems, const void* b_view, int64_t b_view_elems,
                          int n_jobs, int m, int n, int k, int batch, int64_t lda, int64_t ldb, int64_t ldc,
                          float alpha, float beta, int in_dtype, int out_dtype, int compute, void* stream) {
  int rc = check_common(m, n, k, batch, lda, ldb, ldc, in_dtype, out_dtype, compute, n_jobs);
  if (rc) return rc;
  if (n_jobs == 0 || m == 0 || n == 0) return BRK_OK;
  if (c_ptrs == nullptr || (batch > 0 && (a_ptrs == nullptr || b_ptrs == nullptr)))
    return set_error(BRK_ERR_CONTRACT, "null pointer table");
  if (a_view_elems < 0 || b_view_elems < 0 || (a_view_elems > 0 && a_view == nullptr) ||
      (b_view_elems > 0 && b_view == nullptr))
    return set_error(BRK_ERR_CONTRACT, "brgemm_addr_views: a view needs a base and a non-negative extent");
  GenericParams p{};
  p.mode = kModeAddr;
  p.n_jobs = n_jobs;
  p.m = m; p.n = n; p.k = k; p.batch = batch;
  p.lda = lda; p.ldb = ldb; p.ldc = ldc;
  p.a_sk = lda; p.a_sm = 1; p.b_sn = ldb; p.b_sk = 1;
  p.alpha = alpha; p.beta = beta;
  p.in_bf16 = in_dtype == BRK_BF16;
  p.out_bf16 = out_dtype == BRK_BF16;
  p.a_ptrs = a_ptrs; p.b_ptrs = b_ptrs; p.c_ptrs = c_ptrs;
  p.a_base = a_view; p.b_base = b_view;
  p.a_view = a_view_elems; p.b_view = b_view_elems;
  return run_generic(p, compute, stream);
}

int brk_brgemm_offs(const void* a_base, const void* b_base, const int64_t* a_offs,
                    const int64_t* b_offs, void* const* c_ptrs, int n_jobs, int m, int n, int k,
                    int batch, int64_t lda, int64_t ldb, int64_t ldc, float alpha, float beta,
                    int in_dtype, int out_dtype, int compute, void* stream) {
  int rc = check_common(m, n, k, batch, lda, ldb, ldc, in_dtype, out_dtype, compute, n_jobs);
  if (rc) return rc;
  if (n_jobs == 0 || m == 0 || n == 0) return BRK_OK;
  if (c_ptrs == nullptr || (batch > 0 && (a_offs == nullptr || b_offs == nullptr || a_base == nullptr ||
                                          b_base == nullptr)))
    return set_error(BRK_ERR_CONTRACT, "null base or offset table");
  GenericParams p{};
  p.mode = kModeOffs;
  p.n_jobs = n_jobs;
  p.m = m; p.n = n; p.k = k; p.batch = batch;
  p.lda = lda; p.ldb = ldb; p.ldc = ldc;
  p.a_sk = lda; p.a_sm = 1; p.b_sn = ldb; p.b_sk = 1;
  p.alpha = alpha; p.beta = beta;
  p.in_bf16 = in_dtype == BRK_BF16;
  p.out_bf16 = out_dtype == BRK_BF16;
  p.a_base = a_base; p.b_base = b_base;
  p.a_offs = a_offs; p.b_offs = b_offs;
  p.c_ptrs = c_ptrs;
  return run_generic(p, compute, stream);
}

int brk_brgemm_stride(const void* a_base, const void* b_base, int64_t stride_a, int64_t stride_b,
                      void* c_base, int n_jobs, int64_t jstride_a, int64_t jstride_b,
                      int64_t jstride_c, int m, int n, int k, int batch, int64_t lda, int64_t ldb,
                      int64_t ldc, float alpha, float beta, int in_dtype, int out_dtype,
                      int compute, void* stream) {
  int rc = check_common(m, n, k, batch, lda, ldb, ldc, in_dtype, out_dtype, compute, n_jobs);
  if (rc) return rc;
  if (stride_a < 0 || stride_b < 0 || jstride_a < 0 || jstride_b < 0 || jstride_c < 0)
    return set_error(BRK_ERR_CONTRACT, "strides must be >= 0");
  if (n_jobs == 0 || m == 0 || n == 0) return BRK_OK;
  if (c_base == nullptr || (batch > 0 && (a_base == nullptr || b_base == nullptr)))
    return set_error(BRK_ERR_CONTRACT, "null base pointer");
  GenericParams p{};
  p.mode = kModeStride;
  p.n_jobs = n_jobs;
  p.m = m; p.n = n; p.k = k; p.batch = batch;
  p.lda = lda; p.ldb = ldb; p.ldc = ldc;
  p.a_sk = lda; p.a_sm = 1; p.b_sn = ldb; p.b_sk = 1;
  p.alpha = alpha; p.beta = beta;
  p.in_bf16 = in_dtype == BRK_BF16;
  p.out_bf16 = out_dtype == BRK_BF16;
  p.a_base = a_base; p.b_base = b_base;
  p.stride_a = stride_a; p.stride_b = stride_b;
  p.jstride_a = jstride_a; p.jstride_b = jstride_b; p.jstride_c = jstride_c;
  p.c_base = c_base;
  return run_generic(p, compute, stream);
}

}  // extern "C"
