// brk_diag.cu — diagnostic microbenchmark: TMA global->shared throughput for
// the box shapes the engine uses (used to derive the operand-delivery
// roofline in DESIGN.md; not on the product path).
#include <cstdio>
#include <cstring>

#include "brk_internal.h"
#include "brk_ptx.cuh"
#include "brk_tma_host.h"

namespace brk {
namespace {

constexpr int kMaxStages = 12;

// Each CTA streams `iters` boxes (n_loads x load_bytes) through a ring of `stages`
// slots of `slot_bytes`; coordinates walk a [rows][cols] bf16 matrix (2-D map,
// box (64 cols, box_rows rows)) so every load is distinct.
__global__ void __launch_bounds__(256, 1) tma_bw_kernel(const __grid_constant__ CUtensorMap map, int iters,
                                                      int stages, int slot_bytes, int box_rows, int loads_per_slot,
                                                      int rows, int cols, int spin) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * slot_bytes);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int nw = blockDim.x / 32, w = threadIdx.x / 32;
  if ((threadIdx.x & 31) != 0) return;
  const int row_blocks = rows / box_rows, col_blocks = cols / 64;
  int k = blockIdx.x * 7919 + w * 131;
  for (int i = w; i < iters; i += nw) {
    const int s = i % stages;
    if (i >= stages) {
      if (spin) mbar_wait_spin(&full[s], ((i / stages) - 1) & 1);
      else mbar_wait(&full[s], ((i / stages) - 1) & 1);
    }
    mbar_arrive_expect_tx(&full[s], slot_bytes);
    for (int l = 0; l < loads_per_slot; ++l, ++k) {
      const int32_t c[2] = {(k % col_blocks) * 64, ((k / col_blocks) % row_blocks) * box_rows};
      tma_load<2>(smem + s * slot_bytes + l * (slot_bytes / loads_per_slot), &map, &full[s], c);
    }
  }
  for (int i = iters + w; i < iters + stages; i += nw) {
    const int s = i % stages;
    if (i >= stages) mbar_wait(&full[s], ((i / stages) - 1) & 1);
  }
}

// One producer warp whose first `lanes` lanes each issue one box per round (round r fills
// slot r % 2 of every lane; a lane re-fills its slot after the slot's previous box landed):
// does issuing from several lanes of one warp keep several boxes in flight?
__global__ void __launch_bounds__(32, 1) tma_bw_lanes_kernel(const __grid_constant__ CUtensorMap map, int iters,
                                                             int lanes, int box_rows, int rows, int cols) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int slot_bytes = box_rows * 128;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * lanes * slot_bytes);
  const int lane = threadIdx.x;
  if (lane < 2 * lanes) mbar_init(&bars[lane], 1);
  fence_barrier_init();
  __syncwarp();
  const int row_blocks = rows / box_rows, col_blocks = cols / 64;
  int k = blockIdx.x * 7919 + lane * 131;
  if (lane < lanes) {
    for (int i = 0; i < iters; ++i) {
      const int s = i & 1;
      uint64_t* b = &bars[lane * 2 + s];
      if (i >= 2) mbar_wait(b, ((i >> 1) - 1) & 1);
      mbar_arrive_expect_tx(b, slot_bytes);
      const int32_t c[2] = {(k % col_blocks) * 64, ((k / col_blocks) % row_blocks) * box_rows};
      ++k;
      tma_load<2>(smem + (lane * 2 + s) * slot_bytes, &map, b, c);
    }
    for (int i = iters; i < iters + 2; ++i) mbar_wait(&bars[lane * 2 + (i & 1)], ((i >> 1) - 1) & 1);
  }
}

// 4 warps: each times `iters` x (tcgen05.ld 32x32b.x32 + wait) with clock64.
__global__ void __launch_bounds__(128, 1) tmem_ld_kernel(int iters, long long* cycles, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot + (static_cast<uint32_t>(warp * 32) << 16);
  float acc = 0.0f;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t v[32];
    tmem_ld32(base + (i & 7) * 32, v);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 32; ++j) acc += __uint_as_float(v[j]);
  }
  const long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) cycles[blockIdx.x * 4 + warp] = t1 - t0;
  if (acc == 1234.5f) sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(slot, 256);
}

// Back-to-back SS-mode tcgen05.mma (M = 128, N = n, K = 16 bf16, 4 per "k-step" of 64) from
// fixed shared-memory operands into one TMEM accumulator, issued by one thread: cycles per
// MMA, i.e. the tensor pipe's rate for the shape with no operand delivery, barriers or epilogue.
__global__ void __launch_bounds__(128, 1) mma_rate_kernel(int n, int iters, int b_mn, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* done = reinterpret_cast<uint64_t*>(smem + 2 * (16384 + 32768));
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 2 * (16384 + 32768) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u);
  if (threadIdx.x == 0) {
    mbar_init(done, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  if (threadIdx.x < 32) tmem_alloc(&slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc(kFmtBF16, 128, static_cast<uint32_t>(n), 0, static_cast<uint32_t>(b_mn));
    const uint32_t s0 = smem_u32(smem);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t sa = s0 + (i & 1) * (16384 + 32768), sb = sa + 16384;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = make_smem_desc(sa + kk * 32, 16, 1024, kSwizzle128B);
        const uint64_t bd = b_mn ? make_smem_desc(sb + kk * 16 * 128, 64 * 128, 1024, kSwizzle128B)
                                 : make_smem_desc(sb + kk * 32, 16, 1024, kSwizzle128B);
        mma_ss<false>(slot, ad, bd, idesc, (i | kk) ? 1u : 0u);
      }
    }
    mma_commit(done);
    mbar_wait(done, 0);
    const long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(slot, 256);
}

}  // namespace
}  // namespace brk

using namespace brk;

// cycles_dev[ctas]: clock64 cycles for iters x 4 MMAs of M = 128, N = n (bf16, K = 16 each)
extern "C" BRK_API int brk_diag_mma_rate(int n, int b_mn, int ctas, int iters, long long* cycles_dev) {
  if (n < 16 || n > 256 || n % 16) return set_error(BRK_ERR_CONTRACT, "diag_mma_rate: bad N");
  const int smem = 2 * (16384 + 32768) + 1024 + 64;
  cudaFuncSetAttribute(mma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_rate_kernel<<<ctas, 128, smem>>>(n, iters, b_mn, cycles_dev);
  cudaError_t err = cudaDeviceSynchronize();
  return err == cudaSuccess ? BRK_OK : set_cuda_error(err, "diag_mma_rate");
}

extern "C" BRK_API int brk_diag_tma_lanes(const void* buf, int rows, int cols, int box_rows, int lanes, int ctas, int iters,
                               float* us, double* bytes) {
  if (lanes < 1 || lanes > 16 || box_rows < 8 || box_rows > 256 || rows % box_rows || cols % 64)
    return set_error(BRK_ERR_CONTRACT, "diag_tma_lanes: bad shape");
  CUtensorMap map;
  const uint64_t dims[2] = {static_cast<uint64_t>(cols), static_cast<uint64_t>(rows)};
  const uint64_t strides[2] = {1, static_cast<uint64_t>(cols)};
  const uint32_t box[2] = {64, static_cast<uint32_t>(box_rows)};
  int rc = encode_tmap(&map, buf, true, 2, dims, strides, box);
  if (rc) return rc;
  const int smem = 2 * lanes * box_rows * 128 + 1024 + 256;
  cudaFuncSetAttribute(tma_bw_lanes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  tma_bw_lanes_kernel<<<ctas, 32, smem>>>(map, iters, lanes, box_rows, rows, cols);
  cudaEventRecord(e0);
  tma_bw_lanes_kernel<<<ctas, 32, smem>>>(map, iters, lanes, box_rows, rows, cols);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  if (err != cudaSuccess) return set_cuda_error(err, "diag_tma_lanes");
  cudaEventElapsedTime(us, e0, e1);
  *us *= 1000.0f;
  *bytes = static_cast<double>(ctas) * iters * lanes * box_rows * 128;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return BRK_OK;
}

BRK_API int brk_diag_tmem_ld(int ctas, int iters, long long* cycles_dev, float* sink_dev) {
  tmem_ld_kernel<<<ctas, 128>>>(iters, cycles_dev, sink_dev);
  cudaError_t err = cudaDeviceSynchronize();
  return err == cudaSuccess ? BRK_OK : set_cuda_error(err, "diag_tmem_ld");
}

extern "C" {

// Returns device-time microseconds of one launch via *us (events), bytes moved in *bytes.
BRK_API int brk_diag_tma_bw(const void* buf, int rows, int cols, int box_rows, int loads_per_slot, int stages,
                            int ctas, int iters, int spin, float* us, double* bytes) {
  const int threads = 32 * (spin > 1 ? spin : 1);
  if (stages < 1 || stages > kMaxStages || box_rows < 8 || box_rows > 256 || rows % box_rows || cols % 64)
    return set_error(BRK_ERR_CONTRACT, "diag_tma_bw: bad shape");
  CUtensorMap map;
  const uint64_t dims[2] = {static_cast<uint64_t>(cols), static_cast<uint64_t>(rows)};
  const uint64_t strides[2] = {1, static_cast<uint64_t>(cols)};
  const uint32_t box[2] = {64, static_cast<uint32_t>(box_rows)};
  int rc = encode_tmap(&map, buf, true, 2, dims, strides, box);
  if (rc) return rc;
  const int slot = box_rows * 128 * loads_per_slot;
  const int smem = stages * slot + 1024 + 256;
  cudaFuncSetAttribute(tma_bw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  tma_bw_kernel<<<ctas, threads, smem>>>(map, iters, stages, slot, box_rows, loads_per_slot, rows, cols, spin);
  cudaEventRecord(e0);
  tma_bw_kernel<<<ctas, threads, smem>>>(map, iters, stages, slot, box_rows, loads_per_slot, rows, cols, spin);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  if (err != cudaSuccess) return set_cuda_error(err, "diag_tma_bw");
  cudaEventElapsedTime(us, e0, e1);
  *us *= 1000.0f;
  *bytes = static_cast<double>(ctas) * iters * slot;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return BRK_OK;
}

}  // extern "C"
