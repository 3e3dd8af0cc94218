// brk_layout.cu — device layout transforms of the blocked tensors (the paper's
// "tensor reformatting"; reference tensor.py:143-275:
// block_* / unblock_* / pad_spatial).  Every transform is a relabeling copy:
//
//   dst[i_0, ..., i_{n-1}] = src[sum_d (i_d - lo_d) * sstride_d]   if 0 <= i_d - lo_d < sext_d for all d
//                          = 0                                      otherwise (spatial zero padding)
//
// with dst contiguous in the given shape, plus an optional fp32 <-> bf16
// conversion fused into the copy.  HBM-bound: one read and one write of
// every element.  Coalescing: when the output dimension that is contiguous in
// the SOURCE (sstride 1) is not the output's innermost dimension (the
// NCHW -> NCHWc case: w is contiguous in the source, c in the destination),
// each CTA transposes a 32 x 32 tile of those two dimensions through shared
// memory, so reads and writes are both 128 B-coalesced; otherwise the copy
// runs straight along the innermost dimension.  Grid: a grid-stride loop over
// tiles sized to a multiple of the SM count.
#include <cstdio>
#include <cstring>
#include <cuda_bf16.h>

#include "brk_internal.h"

namespace brk {
namespace {

constexpr int kMaxDims = 8;

struct LayoutDesc {
  int nd;
  int64_t shape[kMaxDims];    // destination shape (contiguous)
  int64_t sstride[kMaxDims];  // source element stride per destination dim
  int64_t lo[kMaxDims];       // padding offset per destination dim
  int64_t sext[kMaxDims];     // source extent per destination dim
  int din;                    // destination dim that is contiguous in the source (-1: none)
  int padded;
};

template <bool kBf16>
__device__ __forceinline__ float load_elem(const void* src, int64_t off) {
  if constexpr (kBf16) return __bfloat162float(static_cast<const __nv_bfloat16*>(src)[off]);
  else return static_cast<const float*>(src)[off];
}
template <bool kBf16>
__device__ __forceinline__ void store_elem(void* dst, int64_t off, float v) {
  if constexpr (kBf16) static_cast<__nv_bfloat16*>(dst)[off] = __float2bfloat16_rn(v);
  else static_cast<float*>(dst)[off] = v;
}

// Straight copy: a CTA walks destination rows (all dims but the innermost), decoding the
// row's source base once (32-bit divisions: every extent < 2^31); its threads stream
// the innermost dimension.
template <bool IB, bool OB>
__global__ void __launch_bounds__(256) layout_copy_kernel(const void* __restrict__ src, void* __restrict__ dst,
                                                          const __grid_constant__ LayoutDesc L, int64_t rows) {
  const int dl = L.nd - 1;
  const int64_t inner = L.shape[dl];
  const int64_t chunks = (inner + 255) / 256;
  for (int64_t w = blockIdx.x; w < rows * chunks; w += gridDim.x) {
    const int64_t row = w / chunks;
    const int64_t i = (w - row * chunks) * 256 + threadIdx.x;
    int64_t r = row, base = 0;
    bool pad = false;
    for (int d = dl - 1; d >= 0; --d) {
      const uint32_t ext = static_cast<uint32_t>(L.shape[d]);
      const int64_t q = r < 0x7fffffff ? static_cast<int64_t>(static_cast<uint32_t>(r) / ext) : r / ext;
      const int64_t s = (r - q * ext) - L.lo[d];
      r = q;
      pad |= L.padded && (s < 0 || s >= L.sext[d]);
      base += s * L.sstride[d];
    }
    if (i < inner) {
      const int64_t s = i - L.lo[dl];
      const bool z = pad || (L.padded && (s < 0 || s >= L.sext[dl]));
      store_elem<OB>(dst, row * inner + i, z ? 0.0f : load_elem<IB>(src, base + s * L.sstride[dl]));
    }
  }
}

// Tiled transpose of (din, dout = nd-1): tile t covers din in [a0, a0+32) and dout in
// [b0, b0+64) for one index of every other dimension.  Reads: lanes along din
// (source-contiguous); writes: lanes along dout (destination-contiguous).  The other
// dimensions' source / destination offsets and padding test are decoded once per tile
// (32-bit divisions); per element only two multiply-adds.
template <bool IB, bool OB>
__global__ void __launch_bounds__(256) layout_tile_kernel(const void* __restrict__ src, void* __restrict__ dst,
                                                          const __grid_constant__ LayoutDesc L, int64_t tiles) {
  constexpr int kA = 32, kB = 64;
  __shared__ float tile[kB][kA + 1];
  const int dn = L.din, dl = L.nd - 1;
  const int64_t na = L.shape[dn], nb = L.shape[dl];
  const uint32_t ta = static_cast<uint32_t>((na + kA - 1) / kA), tb = static_cast<uint32_t>((nb + kB - 1) / kB);
  const int64_t ss_a = L.sstride[dn], ss_b = L.sstride[dl];
  int64_t ds_a = 1;
  for (int d = dl; d > dn; --d) ds_a *= L.shape[d];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    uint32_t r = static_cast<uint32_t>(t);  // tiles < 2^32 (host-checked)
    const int64_t b0 = static_cast<int64_t>(r % tb) * kB;
    r /= tb;
    const int64_t a0 = static_cast<int64_t>(r % ta) * kA;
    r /= ta;
    int64_t sbase = 0, dbase = 0, dstride = 1;
    bool pad = false;
    for (int d = dl; d >= 0; --d) {
      if (d != dn && d != dl) {
        const uint32_t ext = static_cast<uint32_t>(L.shape[d]);
        const uint32_t i = r % ext;
        r /= ext;
        const int64_t s = static_cast<int64_t>(i) - L.lo[d];
        pad |= L.padded && (s < 0 || s >= L.sext[d]);
        sbase += s * L.sstride[d];
        dbase += static_cast<int64_t>(i) * dstride;
      }
      dstride *= L.shape[d];
    }
    const int64_t a = a0 + tx;
    const int64_t sa = a - L.lo[dn];
    const bool a_ok = a < na && !(L.padded && (sa < 0 || sa >= L.sext[dn]));
#pragma unroll
    for (int j = 0; j < kB / 8; ++j) {
      const int64_t b = b0 + ty + 8 * j;
      const int64_t sb = b - L.lo[dl];
      float v = 0.0f;
      if (a_ok && !pad && b < nb && !(L.padded && (sb < 0 || sb >= L.sext[dl])))
        v = load_elem<IB>(src, sbase + sa * ss_a + sb * ss_b);
      tile[ty + 8 * j][tx] = v;
    }
    __syncthreads();
    // store: rows a = a0 + (warp, j), lanes along b (two 32-wide halves of the 64-wide tile)
#pragma unroll
    for (int j = 0; j < kA / 8; ++j) {
      const int64_t aa = a0 + ty + 8 * j;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t b = b0 + h * 32 + tx;
        if (aa < na && b < nb) store_elem<OB>(dst, dbase + aa * ds_a + b, tile[h * 32 + tx][ty + 8 * j]);
      }
    }
    __syncthreads();
  }
}

int grid_for(int64_t work) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t cap = static_cast<int64_t>(sms) * 8;  // 8 resident 256-thread CTAs per SM
  return static_cast<int>(work < cap ? (work > 0 ? work : 1) : cap);
}

}  // namespace
}  // namespace brk

using namespace brk;

extern "C" {

BRK_API int brk_layout_transform(const void* src, void* dst, int ndims, const int64_t* shape,
                                 const int64_t* src_strides, const int64_t* pad_lo, const int64_t* src_extent,
                                 int in_dtype, int out_dtype, void* stream) {
  if (ndims < 1 || ndims > kMaxDims) return set_error(BRK_ERR_CONTRACT, "layout: 1..8 dims");
  if ((in_dtype != BRK_F32 && in_dtype != BRK_BF16) || (out_dtype != BRK_F32 && out_dtype != BRK_BF16))
    return set_error(BRK_ERR_CONTRACT, "layout: dtype must be BRK_F32 or BRK_BF16");
  // coalesce: merge destination dims d, d+1 when the source walks them as one dimension
  LayoutDesc L;
  std::memset(&L, 0, sizeof(L));
  int64_t total = 1;
  for (int d = 0; d < ndims; ++d) {
    if (shape[d] < 0) return set_error(BRK_ERR_CONTRACT, "layout: negative extent");
    total *= shape[d];
    const int64_t lo = pad_lo ? pad_lo[d] : 0;
    const int64_t ext = src_extent ? src_extent[d] : shape[d];
    if (lo < 0 || ext < 0 || lo + ext > shape[d]) return set_error(BRK_ERR_CONTRACT, "layout: bad padding");
    if (lo != 0 || ext != shape[d]) L.padded = 1;
    if (L.nd > 0 && !(lo != 0 || ext != shape[d]) && L.lo[L.nd - 1] == 0 && L.sext[L.nd - 1] == L.shape[L.nd - 1] &&
        L.sstride[L.nd - 1] == src_strides[d] * shape[d]) {
      L.shape[L.nd - 1] *= shape[d];
      L.sext[L.nd - 1] = L.shape[L.nd - 1];
      L.sstride[L.nd - 1] = src_strides[d];
      continue;
    }
    L.shape[L.nd] = shape[d];
    L.sstride[L.nd] = src_strides[d];
    L.lo[L.nd] = lo;
    L.sext[L.nd] = ext;
    ++L.nd;
  }
  if (total == 0) return BRK_OK;
  L.din = -1;
  for (int d = 0; d < L.nd - 1; ++d)
    if (L.sstride[d] == 1 && L.shape[d] > 1) L.din = d;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  g_launches.fetch_add(1);
  const bool ib = in_dtype == BRK_BF16, ob = out_dtype == BRK_BF16;
  if (L.din >= 0 && L.sstride[L.nd - 1] != 1) {
    const int64_t tiles = total / (L.shape[L.din] * L.shape[L.nd - 1]) * ((L.shape[L.din] + 31) / 32) *
                          ((L.shape[L.nd - 1] + 63) / 64);
    if (tiles >= (int64_t(1) << 32)) return set_error(BRK_ERR_CONTRACT, "layout: tensor too large");
    auto k = ib ? (ob ? layout_tile_kernel<true, true> : layout_tile_kernel<true, false>)
                : (ob ? layout_tile_kernel<false, true> : layout_tile_kernel<false, false>);
    k<<<grid_for(tiles), 256, 0, st>>>(src, dst, L, tiles);
  } else {
    const int64_t rows = total / L.shape[L.nd - 1];
    auto k = ib ? (ob ? layout_copy_kernel<true, true> : layout_copy_kernel<true, false>)
                : (ob ? layout_copy_kernel<false, true> : layout_copy_kernel<false, false>);
    k<<<grid_for(rows * ((L.shape[L.nd - 1] + 255) / 256)), 256, 0, st>>>(src, dst, L, rows);
  }
  cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? BRK_OK : set_cuda_error(err, "layout launch");
}

}  // extern "C"
