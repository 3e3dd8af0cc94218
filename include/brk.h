/* brk.h — C-ABI of libbrk_sm100.so, the B200 (sm_100a) batch-reduce GEMM
 * engine and the DL primitives built on it.
 *
 * The reference (arxiv 1906.06440, package `brkernels`, pure Python/NumPy)
 * has no native boundary; these entry points are what its Python operator
 * API binds through ctypes.  Each function cites the
 * reference interface it replaces.
 *
 * Conventions
 *  - All pointers are DEVICE pointers unless stated; the caller owns memory.
 *  - Every call is stream-ordered on `stream` (a cudaStream_t, may be NULL)
 *    and never synchronises the device.
 *  - Return 0 (BRK_OK) on success, BRK_ERR_CONTRACT (1) for a shape / layout
 *    contract violation (the Python shim maps it to BrgemmError/LayoutError),
 *    BRK_ERR_CUDA (2) for a CUDA error.  brk_last_error() returns the
 *    thread-local message of the last failure.
 *  - dtype codes: BRK_F32 / BRK_BF16 storage; compute codes BRK_COMPUTE_TF32
 *    (kind::tf32 tensor cores) / BRK_COMPUTE_BF16 (kind::f16, bf16 inputs);
 *    accumulation is always fp32 in TMEM.
 */
#ifndef BRK_H_
#define BRK_H_

#include <stdint.h>

#if defined(__GNUC__)
#define BRK_API __attribute__((visibility("default")))
#else
#define BRK_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define BRK_OK 0
#define BRK_ERR_CONTRACT 1
#define BRK_ERR_CUDA 2

#define BRK_F32 0
#define BRK_BF16 1

#define BRK_COMPUTE_TF32 0
#define BRK_COMPUTE_BF16 1

/* Library / device information. */
BRK_API const char* brk_last_error(void);
BRK_API int brk_version(void);
/* Number of kernel launches issued by this library since load (host counter). */
BRK_API uint64_t brk_launch_count(void);

/* ---------------------------------------------------------------------------
 * BRGEMM, address variant.   Replaces brkernels.brgemm.brgemm
 * (reference pkg/src/brkernels/brgemm.py:260-293) and, with batch=1 per job,
 * brkernels.brgemm.batched_gemm (brgemm.py:340-353).
 *
 * For each job j in [0, n_jobs):
 *   C_j = beta*C_j + alpha * sum_{i<batch} B_ji @ A_ji     (reference view)
 * a_ptrs/b_ptrs: device arrays of n_jobs*batch block addresses (job-major);
 * c_ptrs: device array of n_jobs output block addresses.
 * Block shapes: A (k, m) row stride lda; B (n, k) row stride ldb; C (n, m)
 * row stride ldc (brgemm.py:5-15).  The accumulator for one C block stays in
 * TMEM for the whole batch; C is read (beta != 0) and written once.
 * ------------------------------------------------------------------------- */
BRK_API int brk_brgemm_addr(const void* const* a_ptrs, const void* const* b_ptrs, void* const* c_ptrs,
                    int n_jobs, int m, int n, int k, int batch, int64_t lda, int64_t ldb,
                    int64_t ldc, float alpha, float beta, int in_dtype, int out_dtype,
                    int compute, void* stream);

/* BRGEMM, offset variant (north star; no reference function — equivalent to
 * the address variant with A_ji = a_base + a_offs[j*batch+i] elements). */
BRK_API int brk_brgemm_offs(const void* a_base, const void* b_base, const int64_t* a_offs,
                    const int64_t* b_offs, void* const* c_ptrs, int n_jobs, int m, int n, int k,
                    int batch, int64_t lda, int64_t ldb, int64_t ldc, float alpha, float beta,
                    int in_dtype, int out_dtype, int compute, void* stream);

/* BRGEMM, stride variant.  Replaces brkernels.brgemm.brgemm_strided
 * (brgemm.py:296-337): A_ji = a_base + j*jstride_a + i*stride_a elements,
 * likewise B; C_j = c_base + j*jstride_c elements. */
BRK_API int brk_brgemm_stride(const void* a_base, const void* b_base, int64_t stride_a, int64_t stride_b,
                      void* c_base, int n_jobs, int64_t jstride_a, int64_t jstride_b,
                      int64_t jstride_c, int m, int n, int k, int batch, int64_t lda, int64_t ldb,
                      int64_t ldc, float alpha, float beta, int in_dtype, int out_dtype,
                      int compute, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* BRK_H_ */
