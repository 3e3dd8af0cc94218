// brk_tma_host.h — TMA tensor-map encoding helper (host).
#pragma once
#include <cstdint>
#include <cuda.h>

namespace brk {

// dims[0] is innermost; strides_elems[d] (d >= 1) is the element stride of dim d
// (strides_elems[0] is ignored and must be 1).  128B swizzle, zero OOB fill;
// sw64 selects the 64B swizzle (64 B box rows); atom32 selects the 128B swizzle of 32 B chunks (CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B),
// the layout UMMA reads MN-major TF32 operands in (descriptor layout SWIZZLE_128B_BASE32B).
// estrides: per-dimension traversal strides (null: all 1); a box of box[d] elements along d then
// lands as ceil(box[d] / estrides[d]) elements in shared memory
int encode_tmap(CUtensorMap* out, const void* ptr, bool bf16, int ndims, const uint64_t* dims,
                const uint64_t* strides_elems, const uint32_t* box, bool atom32 = false,
                const uint32_t* estrides = nullptr, bool sw64 = false);

// im2col-mode map over a 5-d bf16 (or fp32) tensor (C, W, H, D, N): lower/upper are the
// pixel bounding-box corners of the 3 spatial dims, estrides the traversal
// strides of all 5 dims.  128B swizzle, zero OOB fill.
int encode_tmap_im2col(CUtensorMap* out, const void* ptr, const uint64_t* dims, const uint64_t* strides_elems,
                       const int* lower, const int* upper, uint32_t channels, uint32_t pixels,
                       const uint32_t* estrides, bool f32 = false);

}  // namespace brk
