// brk_tma_host.h — TMA tensor-map encoding helper (host).
#pragma once
#include <cstdint>
#include <cuda.h>

namespace brk {

// dims[0] is innermost; strides_elems[d] (d >= 1) is the element stride of dim d
// (strides_elems[0] is ignored and must be 1).  128B swizzle, zero OOB fill.
int encode_tmap(CUtensorMap* out, const void* ptr, bool bf16, int ndims, const uint64_t* dims,
                const uint64_t* strides_elems, const uint32_t* box);

}  // namespace brk
