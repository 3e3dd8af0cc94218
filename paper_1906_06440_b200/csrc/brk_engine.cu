// brk_engine.cu — persistent, warp-specialised tcgen05 BRGEMM engine (see brk_engine.h).
//
// Roles (192 threads):
//   warp 0      TMA producer: walks the batch list (k-steps) of every tile
//               and streams (A_s, B_s) boxes into a kStages smem ring.
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma into a TMEM
//               accumulator that stays resident for the whole batch reduce;
//               tcgen05.commit frees smem stages and publishes finished tiles.
//   warps 2..5  epilogue: tcgen05.ld the accumulator (TMEM lane = output row),
//               fuse alpha/beta, bias, activation, ReLU-mask and the SGD
//               update, and store.  Two TMEM accumulators let the epilogue of
//               tile t overlap the MMAs of tile t+1.
#include <cstdio>

#include "brk_engine.h"
#include "brk_internal.h"
#include "brk_ptx.cuh"

namespace brk {
namespace {

constexpr int kThreads = 192;
constexpr int kTileABytes = kEngineBM * 128;

template <int BN>
struct EngineCfg {
  static constexpr int kTileBBytes = BN * 128;
  static constexpr int kStageBytes = kTileABytes + kTileBBytes;
  static constexpr int kStages = (BN >= 256) ? 4 : 6;
  static constexpr int kTmemCols = 2 * BN;
  static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
};

__device__ __forceinline__ void issue_operand(const CUtensorMap* map, const OperandCoords& oc,
                                              int rowblk, int s, uint8_t* dst, uint64_t* bar) {
  const int q = s / oc.kdiv, r = s - q * oc.kdiv;
  for (int l = 0; l < oc.n_loads; ++l) {
    int32_t c[5];
#pragma unroll
    for (int d = 0; d < 5; ++d) c[d] = oc.rc[d] * rowblk + oc.kq[d] * q + oc.kr[d] * r + oc.lc[d] * l;
    uint8_t* p = dst + l * oc.load_bytes;
    switch (oc.ndims) {
      case 2: { const int32_t cc[2] = {c[0], c[1]}; tma_load<2>(p, map, bar, cc); break; }
      case 3: { const int32_t cc[3] = {c[0], c[1], c[2]}; tma_load<3>(p, map, bar, cc); break; }
      case 4: { const int32_t cc[4] = {c[0], c[1], c[2], c[3]}; tma_load<4>(p, map, bar, cc); break; }
      default: { const int32_t cc[5] = {c[0], c[1], c[2], c[3], c[4]}; tma_load<5>(p, map, bar, cc); break; }
    }
  }
}

// smem descriptor for the MMA sub-step kk (32 bytes of K) of one operand tile
template <bool kTF32>
__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int mn_major, int kk) {
  if (!mn_major) {
    // K-major, 128B swizzle: 8-row groups 1024 B apart; K advance = 32 B.
    return make_smem_desc(base + kk * 32, 16, 1024, kSwizzle128B);
  }
  // MN-major, 128B swizzle: atom = 64 B-elements(128 B) x BK rows; 8 K-rows = 1024 B.
  constexpr uint32_t kRowsPerMma = kTF32 ? 8 : 16;
  constexpr uint32_t kAtomBytes = (kTF32 ? 32 : 64) * 128;  // BK rows x 128 B
  return make_smem_desc(base + kk * kRowsPerMma * 128, kAtomBytes, 1024, kSwizzle128B);
}

template <int BN, bool kTF32>
__global__ void __launch_bounds__(kThreads, 1) engine_kernel(const __grid_constant__ EngineParams p) {
  using Cfg = EngineCfg<BN>;
  constexpr int kStages = Cfg::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * Cfg::kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;  // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id();
  const int lane = threadIdx.x & 31;
  const int num_tiles = p.m_tiles * p.n_tiles;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&p.map_a);
    tma_prefetch_desc(&p.map_b);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t bytes = p.ca.n_loads * p.ca.load_bytes + p.cb.n_loads * p.cb.load_bytes;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int mb = t % p.m_tiles, nb = t / p.m_tiles;
        for (int s = 0; s < p.k_steps; ++s) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::kStageBytes;
          uint8_t* sb = sa + kTileABytes;
          if (p.debug_flags & 2) {
            mbar_arrive(&full[stage]);
          } else {
            mbar_arrive_expect_tx(&full[stage], bytes);
            issue_operand(&p.map_a, p.ca, mb, s, sa, &full[stage]);
            issue_operand(&p.map_b, p.cb, nb, s, sb, &full[stage]);
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = make_idesc(kTF32 ? kFmtTF32 : kFmtBF16, kEngineBM, BN, p.ca.mn_major,
                                      p.cb.mn_major);
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++local) {
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int s = 0; s < p.k_steps; ++s) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (p.debug_flags & 1) {
          if (elect_one()) {
            mbar_arrive(&empty[stage]);
            if (s == p.k_steps - 1) mbar_arrive(&tfull[acc]);
          }
        } else if (elect_one()) {
          const uint32_t sa = smem_u32(smem + stage * Cfg::kStageBytes);
          const uint32_t sb = sa + kTileABytes;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            mma_ss<kTF32>(d_tmem, operand_desc<kTF32>(sa, p.ca.mn_major, kk),
                          operand_desc<kTF32>(sb, p.cb.mn_major, kk), idesc,
                          (s > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&empty[stage]);
          if (s == p.k_steps - 1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int row_in_tile = quarter * 32 + lane;
    int local = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++local) {
      const int mb = t % p.m_tiles, nb = t / p.m_tiles;
      const int acc = local & 1;
      mbar_wait(&tfull[acc], (local >> 1) & 1);
      tc_fence_after();
      const int row = mb * kEngineBM + row_in_tile;
      const bool row_ok = row < p.rows;
      const int64_t roff = (row / p.om.rb) * p.om.rh + (row % p.om.rb) * p.om.rl;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem_base + acc * BN + (static_cast<uint32_t>(quarter * 32) << 16) + c0, v);
        tmem_ld_wait();
        const int col0 = nb * BN + c0;
        if (!row_ok || col0 >= p.cols) continue;
        // 32 columns never straddle an output block when cb % 32 == 0 (host guarantees)
        const int64_t off = roff + (col0 / p.om.cb) * p.om.ch + (col0 % p.om.cb) * p.om.cl;
        float f[32];
        if (p.alpha == 1.0f) {
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]) * p.alpha;
        }
        if (p.out == nullptr) continue;  // diagnostic: mainloop-only timing
        if (p.beta != 0.0f) {
          if (p.out_bf16) {
            const __nv_bfloat16* src = static_cast<const __nv_bfloat16*>(p.out) + off;
#pragma unroll
            for (int j = 0; j < 32; ++j) f[j] += p.beta * __bfloat162float(src[j]);
          } else {
            const float* src = static_cast<const float*>(p.out) + off;
#pragma unroll
            for (int j = 0; j < 32; ++j) f[j] += p.beta * src[j];
          }
        }
        if (p.bias != nullptr) {
          const float4* b4 = reinterpret_cast<const float4*>(p.bias + col0);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 b = __ldg(b4 + q);
            f[q * 4 + 0] += b.x; f[q * 4 + 1] += b.y; f[q * 4 + 2] += b.z; f[q * 4 + 3] += b.w;
          }
        }
        if (p.act == kActRelu) {
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] = fmaxf(f[j], 0.0f);
        } else if (p.act == kActSigmoid) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float e = __expf(-fabsf(f[j]));
            const float r = __fdividef(1.0f, 1.0f + e);
            f[j] = f[j] >= 0.0f ? r : e * r;
          }
        }
        if (p.mask != nullptr) {
          const uint4* mk = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.mask) + off);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 w = mk[q];
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float2 m2 = __bfloat1622float2(h[j]);
              f[q * 8 + 2 * j] = m2.x > 0.0f ? f[q * 8 + 2 * j] : 0.0f;
              f[q * 8 + 2 * j + 1] = m2.y > 0.0f ? f[q * 8 + 2 * j + 1] : 0.0f;
            }
          }
        }
        if (p.out_bf16) {
          uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + off);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 w;
            w.x = pack_bf16x2(f[q * 8 + 0], f[q * 8 + 1]);
            w.y = pack_bf16x2(f[q * 8 + 2], f[q * 8 + 3]);
            w.z = pack_bf16x2(f[q * 8 + 4], f[q * 8 + 5]);
            w.w = pack_bf16x2(f[q * 8 + 6], f[q * 8 + 7]);
            dst[q] = w;
          }
        } else {
          float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.out) + off);
#pragma unroll
          for (int q = 0; q < 8; ++q) dst[q] = make_float4(f[q * 4], f[q * 4 + 1], f[q * 4 + 2], f[q * 4 + 3]);
        }
        if (p.sgd_w != nullptr) {
          uint4* wp = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.sgd_w) + off);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 w = wp[q];
            __nv_bfloat16* h = reinterpret_cast<__nv_bfloat16*>(&w);
#pragma unroll
            for (int j = 0; j < 8; ++j)
              h[j] = __float2bfloat16_rn(__bfloat162float(h[j]) - p.sgd_lr * f[q * 8 + j]);
            wp[q] = w;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, Cfg::kTmemCols);
}

template <int BN, bool kTF32>
int launch_engine_t(const EngineParams& p, int grid, cudaStream_t stream) {
  using Cfg = EngineCfg<BN>;
  auto kern = engine_kernel<BN, kTF32>;
  static int attr_set = 0;  // per instantiation; the attribute is per-context state
  cudaError_t err;
  if (!attr_set) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
    if (err != cudaSuccess) return set_cuda_error(err, "engine smem attribute");
    attr_set = 1;
  }
  kern<<<grid, kThreads, Cfg::kSmem, stream>>>(p);
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_cuda_error(err, "engine launch");
  return BRK_OK;
}

}  // namespace

int engine_sm_count() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

int launch_engine(const EngineParams& p, int bn, int tf32, int max_ctas, cudaStream_t stream) {
  const int tiles = p.m_tiles * p.n_tiles;
  if (tiles <= 0) return BRK_OK;
  int grid = tiles < engine_sm_count() ? tiles : engine_sm_count();
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  if (bn == 256) return tf32 ? launch_engine_t<256, true>(p, grid, stream) : launch_engine_t<256, false>(p, grid, stream);
  if (bn == 128) return tf32 ? launch_engine_t<128, true>(p, grid, stream) : launch_engine_t<128, false>(p, grid, stream);
  if (bn == 64) return tf32 ? launch_engine_t<64, true>(p, grid, stream) : launch_engine_t<64, false>(p, grid, stream);
  return set_error(BRK_ERR_CONTRACT, "engine: BN must be 64, 128 or 256");
}

}  // namespace brk
