// brk_tma_host.cu — host-side TMA tensor-map encoding without linking libcuda:
// cuTensorMapEncodeTiled is fetched once through cudaGetDriverEntryPoint.
#include <cstdio>
#include <mutex>

#include "brk_internal.h"
#include "brk_tma_host.h"

namespace brk {

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);
EncodeFn g_encode = nullptr;
std::once_flag g_once;
}  // namespace

int encode_tmap(CUtensorMap* out, const void* ptr, bool bf16, int ndims, const uint64_t* dims,
                const uint64_t* strides_elems, const uint32_t* box, bool atom32, const uint32_t* estrides,
                bool sw64) {
  std::call_once(g_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<EncodeFn>(fn);
  });
  if (g_encode == nullptr) return set_error(BRK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const size_t esz = bf16 ? 2 : 4;
  cuuint64_t gdim[5], gstride[4];
  cuuint32_t bdim[5], estride[5];
  for (int d = 0; d < ndims; ++d) {
    gdim[d] = dims[d];
    bdim[d] = box[d];
    estride[d] = estrides != nullptr ? estrides[d] : 1;
    if (d > 0) gstride[d - 1] = strides_elems[d] * esz;
  }
  CUresult r = g_encode(out, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                        ndims, const_cast<void*>(ptr), gdim, gstride, bdim, estride,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        sw64 ? CU_TENSOR_MAP_SWIZZLE_64B
                             : (atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B),
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[256];
    std::snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (CUresult %d, ndims %d)", (int)r, ndims);
    return set_error(BRK_ERR_CONTRACT, buf);
  }
  return BRK_OK;
}

}  // namespace brk

namespace brk {
namespace {
using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeIm2colFn g_encode_im2col = nullptr;
std::once_flag g_once_im2col;
}  // namespace

int encode_tmap_im2col(CUtensorMap* out, const void* ptr, const uint64_t* dims, const uint64_t* strides_elems,
                       const int* lower, const int* upper, uint32_t channels, uint32_t pixels,
                       const uint32_t* estrides, bool f32) {
  std::call_once(g_once_im2col, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode_im2col = reinterpret_cast<EncodeIm2colFn>(fn);
  });
  if (g_encode_im2col == nullptr) return set_error(BRK_ERR_CUDA, "cuTensorMapEncodeIm2col unavailable");
  cuuint64_t gdim[5], gstride[4];
  cuuint32_t es[5];
  for (int d = 0; d < 5; ++d) {
    gdim[d] = dims[d];
    es[d] = estrides[d];
    if (d > 0) gstride[d - 1] = strides_elems[d] * (f32 ? 4 : 2);
  }
  CUresult r = g_encode_im2col(out, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(ptr), gdim, gstride,
                               lower, upper, channels, pixels, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[256];
    std::snprintf(buf, sizeof(buf),
                  "cuTensorMapEncodeIm2col failed (CUresult %d; dims %llu %llu %llu %llu %llu, corners %d,%d,%d / "
                  "%d,%d,%d, pixels %u)",
                  (int)r, (unsigned long long)dims[0], (unsigned long long)dims[1], (unsigned long long)dims[2],
                  (unsigned long long)dims[3], (unsigned long long)dims[4], lower[0], lower[1], lower[2], upper[0],
                  upper[1], upper[2], pixels);
    return set_error(BRK_ERR_CONTRACT, buf);
  }
  return BRK_OK;
}

}  // namespace brk

