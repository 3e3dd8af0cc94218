// brk_lstm_seq.cu — the LSTM cell over a whole sequence as ONE persistent launch
// per direction (reference lstm.py:217-327, paper Alg. 2 / Eqs. 1-6; BPTT as
// restated in oracle/brk_oracle.py:305-350).
//
// The input projections W x_t + b of all steps are one large BRGEMM before the
// loop (brk_gemm_dense), so only the recurrent batch-reduce  sum_j h[n][j] R[.][j]
// sits on the serial path.  Each CTA keeps its slice of the recurrent weights
// resident in shared memory for all T steps and streams the previous step's
// h (bf16) by TMA, one 64-wide K chunk per ring stage; the accumulators live in
// TMEM and the gate / cell-state epilogue is fused (s_t stays in registers).
// There is no grid-wide barrier: K chunk kc of step t is released by a
// per-chunk counter that the CTAs owning those hidden units bump after
// writing their slice of h_t, so step t+1's loads start chunk by chunk.
//
// forward  : CTA c owns hidden units j0 = 8c .. 8c+7 of all four gates
//            (MMA N = 32: rows g*8 + jj of R_cat = [R_i; R_c; R_f; R_o]).
// backward : a cluster of 4 CTAs (one per gate g) owns 32 hidden units; CTA g
//            computes the partial recurrent gradient  dpre_g(t+1) R_g  for them
//            (R_g^T slice resident), the four partials are summed through
//            distributed shared memory and each CTA of the cluster finishes
//            the BPTT element math for a quarter of the minibatch rows.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_bf16.h>

#include "brk_internal.h"
#include "brk_ptx.cuh"
#include "brk_tma_host.h"

namespace brk {
namespace {

// A ring of 4 stages of 32 KB (two 128-row M tiles); each receives only the operand's N valid
// rows (rounded to 8-row swizzle atoms).  The forward chunk stream (16 chunks, ~5 us per step)
// is neither bound by bytes (streaming all 256 rows: same time), nor by the ring depth (6
// stages: 10.4 us per step vs 9.7), nor by the cluster multicast (cluster sizes 1..8 equal,
// BRK_LSTM_CS), nor by serial release polls (polling a producer's chunks of a step together:
// 11.3 us, the first chunk waits for the last).
constexpr int kStagesS = 4;
constexpr int kThreadsS = 9 * 32;    // 4 epilogue, 1 MMA, 4 producer warps (one per stage)
constexpr int kJf = 8;               // forward: hidden units per CTA
constexpr int kJb = 32;              // backward: hidden units per cluster

struct SeqParams {
  CUtensorMap map_a;  // streamed operand, 3-d (cols, N, slots) bf16, box (64, 128, 1)
  CUtensorMap map_w;  // resident operand rows, 2-d (K, rows) bf16, box (64, 8 | 32)
  int T, N, K;
  // forward
  const float* gx;       // [T][N][4][K]  W x_t + b
  const float* s0;       // [N][K] or null
  float* h_out;          // [T][N][K]
  float* s_out;          // [T][N][K]
  float* gates_out;      // [T][N][4][K] activated i, c, f, o
  __nv_bfloat16* h_bf;   // [T+1][N][K]  slot 0 = h0 (filled by the host)
  // backward
  const float* dh;       // [T][N][K]
  const float* gates;    // [T][N][4][K]
  const float* s;        // [T][N][K]
  __nv_bfloat16* dpre;   // [T][N][4][K] (bf16; A operand of the next step and of the weight gradients)
  float* ds0;            // [N][K] dL/ds_{-1}
  unsigned* flags;       // per 64-column chunk release counters (zeroed by the host)
  unsigned long long* ts;  // diagnostics: per-step %globaltimer stamps of CTA 0 [T][8] (or null)
  int slice;               // forward: rows of h each cluster CTA loads and multicasts (multiple of 8)
  int stage_bytes;         // ring stage stride: 32 KB (two 128-row M tiles)
  int stage_tx;            // bytes one stage receives (the N valid rows, whole 8-row atoms)
  int stages;              // ring stages (<= kStagesS: as many as shared memory holds)
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SEQ_TS(step, slot)                                                          \
  do {                                                                              \
    if (p.ts != nullptr && blockIdx.x == 0) p.ts[(step) * 8 + (slot)] = gtime();    \
  } while (0)

__device__ __forceinline__ float sigm_s(float x) {
  const float e = __expf(-fabsf(x));
  const float r = __fdividef(1.0f, 1.0f + e);
  return x >= 0.0f ? r : e * r;
}

// tanh(x) = 1 - 2 / (e^{2x} + 1), saturating correctly at both ends
__device__ __forceinline__ float tanh_f(float x) {
  const float e = __expf(2.0f * x);
  return 1.0f - __fdividef(2.0f, e + 1.0f);
}

// release counters: one per 128 B line (pollers of different chunks hit different L2 lines),
// polled with a short back-off (the MLP step measured polling pressure on shared lines)
#ifndef BRK_LSTM_FLAG_STRIDE
#define BRK_LSTM_FLAG_STRIDE 32
#endif
#ifndef BRK_LSTM_POLL_NS
#define BRK_LSTM_POLL_NS 64
#endif
constexpr int kFlagStride = BRK_LSTM_FLAG_STRIDE;
__device__ __forceinline__ void poll_backoff() {
  if (BRK_LSTM_POLL_NS > 0) __nanosleep(BRK_LSTM_POLL_NS);
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  const int32_t c[3] = {c0, c1, c2};
  tma_load<3>(dst, map, bar, c);
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ uint32_t cluster_nctas() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
// 3-d TMA load multicast to every CTA of the cluster in `mask` (same smem offset,
// complete_tx on the same-offset mbarrier of each destination CTA)
__device__ __forceinline__ void tma_load3_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                             uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
      : "memory");
}
// arrive (when this CTA's prior MMAs complete) on the same-offset barrier of every CTA in `mask`
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

// ------------------------------------------------------------------ forward
__global__ void __launch_bounds__(kThreadsS, 1) lstm_seq_fwd_kernel(const __grid_constant__ SeqParams p) {
  constexpr int kGN = 4 * kJf;  // 32 gate columns
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int KC = p.K / 64;
  uint8_t* ring = smem;
  constexpr int NS = kStagesS;  // (p.stages == kStagesS: checked at launch)
  uint8_t* wsm = smem + NS * p.stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(wsm + KC * kGN * 128);
  uint64_t* empty = full + kStagesS;  // (barrier arrays sized for the maximum)
  uint64_t* tfull = empty + kStagesS;
  uint64_t* tempty = tfull + 1;
  uint64_t* wbar = tempty + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(wbar + 1);
  const int warp = warp_id(), lane = threadIdx.x & 31;
  const int j0 = blockIdx.x * kJf;
  const int n_mt = p.N > 128 ? 2 : 1;
  const int chunk_owners = 64 / kJf;  // CTAs writing one 64-column chunk of h
  // The CTAs of a cluster share each streamed chunk: CTA r loads rows
  // [r*256/cs, (r+1)*256/cs) of the 256-row tile and multicasts them to all.
  const int cs = static_cast<int>(cluster_nctas());
  const int crank = static_cast<int>(cluster_ctarank());
  const uint16_t cmask = static_cast<uint16_t>((1u << cs) - 1u);
  // only the N valid rows (rounded to 8-row swizzle groups per CTA) are streamed, not the
  // whole 256-row tile: the chunk stream is bound by each SM's L2 ingress bandwidth
  const int slice = p.slice;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], cs); }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    mbar_init(wbar, 1);
    fence_barrier_init();
  }
  if (warp == 4) tmem_alloc(tslot, 64);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp >= 5) {
    // ---------------------------------------------------------------- producers
    const int pid = warp - 5;
    if (elect_one()) {
      if (pid == 0) {  // resident R slice: rows g*8+jj of chunk kc <- R_cat[g*K + j0 + jj][64kc ..]
        mbar_arrive_expect_tx(wbar, KC * kGN * 128);
        for (int kc = 0; kc < KC; ++kc)
          for (int g = 0; g < 4; ++g) {
            const int32_t c[2] = {kc * 64, g * p.K + j0};
            tma_load<2>(wsm + kc * kGN * 128 + g * 1024, &p.map_w, wbar, c);
          }
      }
      const int total = p.T * KC;
      for (int gi = pid; pid < NS && gi < total; gi += NS) {
        const int t = gi / KC, kc = gi - t * KC;
        const uint32_t ph = (gi / NS) & 1;
        if (t > 0) {
          while (ld_acquire(&p.flags[kc * kFlagStride]) < static_cast<unsigned>(chunk_owners * t)) poll_backoff();
          fence_proxy_async_global();
        }
        if (kc == 0) SEQ_TS(t, 0);       // chunk 0 of h_{t-1} released
        if (kc == KC - 1) SEQ_TS(t, 1);  // last chunk released
        mbar_wait(&empty[pid], ph ^ 1);  // every CTA of the cluster consumed this stage
        mbar_arrive_expect_tx(&full[pid], static_cast<uint32_t>(slice * cs * 128));
        tma_load3_mc(ring + pid * p.stage_bytes + crank * slice * 128, &p.map_a, &full[pid], kc * 64, crank * slice,
                     t, cmask);
      }
    }
  } else if (warp == 4) {
    // ---------------------------------------------------------------- MMA issuer
    const uint32_t idesc = make_idesc(kFmtBF16, 128, kGN, 0, 0);
    const uint64_t ring_desc = make_smem_desc(smem_u32(ring), 16, 1024, kSwizzle128B);
    const uint64_t w_desc = make_smem_desc(smem_u32(wsm), 16, 1024, kSwizzle128B);
    mbar_wait(wbar, 0);
    for (int t = 0; t < p.T; ++t) {
      mbar_wait(tempty, (t & 1) ^ 1);
      tc_fence_after();
      for (int kc = 0; kc < KC; ++kc) {
        const int gi = t * KC + kc, st = gi % NS;
        mbar_wait(&full[st], (gi / NS) & 1);
        tc_fence_after();
        if (lane == 0 && kc == 0) SEQ_TS(t, 2);       // first chunk landed
        if (lane == 0 && kc == KC - 1) SEQ_TS(t, 3);  // last chunk landed
        if (elect_one()) {  // descriptors advanced by constants (16-byte units), see brk_engine.cu
          const uint64_t ad = ring_desc + static_cast<uint32_t>(st * p.stage_bytes) / 16;
          const uint64_t bd = w_desc + static_cast<uint32_t>(kc * kGN * 128 / 16);
          for (int mt = 0; mt < n_mt; ++mt)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_ss<false>(tmem + mt * kGN, ad + mt * 1024 + kk * 2, bd + kk * 2, idesc, (kc | kk) ? 1u : 0u);
          mma_commit_mc(&empty[st], cmask);  // the stage is free in the whole cluster once all CTAs arrive
          if (kc == KC - 1) mma_commit(tfull);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 0-3)
    // Critical path per step: accumulator -> h_t (bf16) -> chunk release.  The
    // step's input projections are prefetched while the MMAs run, and the fp32
    // h / s / gate stores are issued only after the release.
    float sreg[2][kJf];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int n = mt * 128 + warp * 32 + lane;
#pragma unroll
      for (int jj = 0; jj < kJf; ++jj)
        sreg[mt][jj] = (p.s0 != nullptr && n < p.N) ? p.s0[static_cast<int64_t>(n) * p.K + j0 + jj] : 0.0f;
    }
    for (int t = 0; t < p.T; ++t) {
      float pre[2][4][kJf];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int n = mt * 128 + warp * 32 + lane;
        if (mt < n_mt && n < p.N) {
          const float* gxr = p.gx + (static_cast<int64_t>(t) * p.N + n) * 4 * p.K + j0;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const float4 a = __ldcs(reinterpret_cast<const float4*>(gxr + g * p.K));
            const float4 b = __ldcs(reinterpret_cast<const float4*>(gxr + g * p.K + 4));
            pre[mt][g][0] = a.x; pre[mt][g][1] = a.y; pre[mt][g][2] = a.z; pre[mt][g][3] = a.w;
            pre[mt][g][4] = b.x; pre[mt][g][5] = b.y; pre[mt][g][6] = b.z; pre[mt][g][7] = b.w;
          }
        }
      }
      mbar_wait(tfull, t & 1);
      tc_fence_after();
      if (threadIdx.x == 0) SEQ_TS(t, 4);  // accumulator ready
      float hv[2][kJf];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        if (mt >= n_mt) break;
        uint32_t v[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + mt * kGN, v);
        tmem_ld_wait();
        const int n = mt * 128 + warp * 32 + lane;
        if (n < p.N) {
#pragma unroll
          for (int jj = 0; jj < kJf; ++jj) {
            const float gi = sigm_s(pre[mt][0][jj] + __uint_as_float(v[jj]));
            const float gc = tanh_f(pre[mt][1][jj] + __uint_as_float(v[kJf + jj]));
            const float gf = sigm_s(pre[mt][2][jj] + __uint_as_float(v[2 * kJf + jj]));
            const float go = sigm_s(pre[mt][3][jj] + __uint_as_float(v[3 * kJf + jj]));
            const float sv = gf * sreg[mt][jj] + gi * gc;
            sreg[mt][jj] = sv;
            hv[mt][jj] = go * tanh_f(sv);
            pre[mt][0][jj] = gi; pre[mt][1][jj] = gc; pre[mt][2][jj] = gf; pre[mt][3][jj] = go;
          }
          *reinterpret_cast<uint4*>(p.h_bf + (static_cast<int64_t>(t + 1) * p.N + n) * p.K + j0) =
              make_uint4(pack_bf16x2(hv[mt][0], hv[mt][1]), pack_bf16x2(hv[mt][2], hv[mt][3]),
                         pack_bf16x2(hv[mt][4], hv[mt][5]), pack_bf16x2(hv[mt][6], hv[mt][7]));
        }
      }
      tc_fence_before();
      fence_proxy_async_global();  // h_t (bf16) is read by other CTAs' TMA (async proxy)
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 0) {
        SEQ_TS(t, 5);  // epilogue done
        // release (acq_rel fence + relaxed add) rather than an SC fence + atomic
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&p.flags[(j0 / 64) * kFlagStride]) : "memory");
      }
      // off the critical path: fp32 h, s and the activated gates (BPTT inputs)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int n = mt * 128 + warp * 32 + lane;
        if (mt < n_mt && n < p.N) {
          const int64_t row = static_cast<int64_t>(t) * p.N + n;
          float* go_ = p.gates_out + row * 4 * p.K + j0;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            __stcs(reinterpret_cast<float4*>(go_ + g * p.K),
                   make_float4(pre[mt][g][0], pre[mt][g][1], pre[mt][g][2], pre[mt][g][3]));
            __stcs(reinterpret_cast<float4*>(go_ + g * p.K + 4),
                   make_float4(pre[mt][g][4], pre[mt][g][5], pre[mt][g][6], pre[mt][g][7]));
          }
          float* ho = p.h_out + row * p.K + j0;
          float* so = p.s_out + row * p.K + j0;
          __stcs(reinterpret_cast<float4*>(ho), make_float4(hv[mt][0], hv[mt][1], hv[mt][2], hv[mt][3]));
          __stcs(reinterpret_cast<float4*>(ho + 4), make_float4(hv[mt][4], hv[mt][5], hv[mt][6], hv[mt][7]));
          __stcs(reinterpret_cast<float4*>(so), make_float4(sreg[mt][0], sreg[mt][1], sreg[mt][2], sreg[mt][3]));
          __stcs(reinterpret_cast<float4*>(so + 4), make_float4(sreg[mt][4], sreg[mt][5], sreg[mt][6], sreg[mt][7]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // peers may still multicast into / arrive on this CTA's shared memory
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}

// ------------------------------------------------------------------ forward, CTA pairs
// A CTA pair (cta_group::2, M = 256) owns kUpp = 16 hidden units of all four gates (MMA N = 64
// gate columns, column n = gate * 16 + unit): CTA rank r keeps the B rows of gates 2r, 2r + 1
// resident and streams only its half of the batch rows of h_{t-1} (rows_half, rounded to 8).
// Per chunk and SM that is 11 KB of TMA writes + 16 KB of A and 4 KB of B MMA reads instead of
// 24 + 32 + 8 KB for a single CTA's two 128-row M tiles — the single-CTA chunk stream is bound
// by shared-memory bandwidth (computing only the first M tile: 5.0 -> 3.7 us per step).
constexpr int kUpp = 16;
__global__ void __launch_bounds__(kThreadsS, 1) lstm_seq_fwd_pair_kernel(const __grid_constant__ SeqParams p) {
  constexpr int kGN = 4 * kUpp;   // 64 gate columns per pair
  constexpr int kBRows = kGN / 2; // 32 B rows per CTA
  constexpr int kStageA = 16384;  // one CTA's A stage: 128 rows x 128 B (rows_half of them loaded)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int KC = p.K / 64;
  constexpr int NS = kStagesS;
  uint8_t* ring = smem;
  uint8_t* wsm = smem + NS * kStageA;  // resident B: KC chunks x 32 rows x 128 B
  uint64_t* full = reinterpret_cast<uint64_t*>(wsm + KC * kBRows * 128);
  uint64_t* empty = full + kStagesS;
  uint64_t* tfull = empty + kStagesS;
  uint64_t* tempty = tfull + 1;
  uint64_t* wbar = tempty + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(wbar + 1);
  const int warp = warp_id(), lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int j0 = (blockIdx.x >> 1) * kUpp;  // the pair's first hidden unit
  const int rows_half = p.slice;            // batch rows per CTA (multiple of 8, <= 128)
  const int row_base = static_cast<int>(rank) * rows_half;
  const int chunk_owners = 2 * (64 / kUpp);  // CTAs writing one 64-column chunk of h

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    mbar_init(tempty, 8);  // the 4 epilogue warps of both CTAs (on the leader)
    mbar_init(wbar, 1);
    fence_barrier_init();
  }
  if (warp == 4) tmem_alloc_pair(tslot, 64);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp >= 5) {
    // ---------------------------------------------------------------- producers
    const int pid = warp - 5;
    if (elect_one()) {
      if (pid == 0) {  // resident B rows of gates 2r, 2r + 1: row gg*16 + uu <- R_cat[(2r + gg) K + j0 + uu]
        // (both CTAs' rows complete on the leader's barrier: its MMAs read both)
        if (leader) mbar_arrive_expect_tx(wbar, 2 * KC * kBRows * 128);
        for (int kc = 0; kc < KC; ++kc)
          for (int gg = 0; gg < 2; ++gg) {
            const int32_t c[2] = {kc * 64, (2 * static_cast<int>(rank) + gg) * p.K + j0};
            tma_load_pair<2>(wsm + kc * kBRows * 128 + gg * kUpp * 128, &p.map_w, wbar, c);
          }
      }
      const int total = p.T * KC;
      for (int gi = pid; gi < total; gi += NS) {
        const int t = gi / KC, kc = gi - t * KC;
        const uint32_t ph = (gi / NS) & 1;
        if (t > 0) {
          while (ld_acquire(&p.flags[kc * kFlagStride]) < static_cast<unsigned>(chunk_owners * t)) poll_backoff();
          fence_proxy_async_global();
        }
        if (kc == 0) SEQ_TS(t, 0);
        if (kc == KC - 1) SEQ_TS(t, 1);
        mbar_wait(&empty[pid], ph ^ 1);  // both CTAs' MMAs of the previous round on this stage done
        if (leader) mbar_arrive_expect_tx(&full[pid], static_cast<uint32_t>(2 * rows_half * 128));
        const int32_t c[3] = {kc * 64, row_base, t};
        tma_load_pair<3>(ring + pid * kStageA, &p.map_a, &full[pid], c);
      }
    }
  } else if (warp == 4) {
    // ---------------------------------------------------------------- MMA issuer (leader)
    if (leader) {
      const uint32_t idesc = make_idesc(kFmtBF16, 256, kGN, 0, 0);
      const uint64_t ring_desc = make_smem_desc(smem_u32(ring), 16, 1024, kSwizzle128B);
      const uint64_t w_desc = make_smem_desc(smem_u32(wsm), 16, 1024, kSwizzle128B);
      mbar_wait(wbar, 0);
      for (int t = 0; t < p.T; ++t) {
        mbar_wait(tempty, (t & 1) ^ 1);
        tc_fence_after();
        for (int kc = 0; kc < KC; ++kc) {
          const int gi = t * KC + kc, st = gi % NS;
          mbar_wait(&full[st], (gi / NS) & 1);
          tc_fence_after();
          if (lane == 0 && kc == 0) SEQ_TS(t, 2);
          if (lane == 0 && kc == KC - 1) SEQ_TS(t, 3);
          if (elect_one()) {  // descriptors advanced by constants (16-byte units), see brk_engine.cu
            const uint64_t ad = ring_desc + static_cast<uint32_t>(st * (kStageA / 16));
            const uint64_t bd = w_desc + static_cast<uint32_t>(kc * (kBRows * 128 / 16));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_ss_pair<false>(tmem, ad + kk * 2, bd + kk * 2, idesc, (kc | kk) ? 1u : 0u);
            mma_commit_pair(&empty[st]);
            if (kc == KC - 1) mma_commit_pair(tfull);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 0-3)
    const int li = warp * 32 + lane;  // TMEM lane = this CTA's A row
    const int n = row_base + li;
    const bool ok = li < rows_half && n < p.N;
    const uint32_t tempty_leader = mapa_shared(smem_u32(tempty), 0);
    float sreg[kUpp];
#pragma unroll
    for (int uu = 0; uu < kUpp; ++uu) sreg[uu] = (p.s0 != nullptr && ok) ? p.s0[static_cast<int64_t>(n) * p.K + j0 + uu] : 0.0f;
    for (int t = 0; t < p.T; ++t) {
      float pre[4][kUpp];
      if (ok) {
        const float* gxr = p.gx + (static_cast<int64_t>(t) * p.N + n) * 4 * p.K + j0;
#pragma unroll
        for (int g = 0; g < 4; ++g)
#pragma unroll
          for (int q4 = 0; q4 < kUpp / 4; ++q4) {
            const float4 a = __ldcs(reinterpret_cast<const float4*>(gxr + g * p.K + 4 * q4));
            pre[g][4 * q4] = a.x; pre[g][4 * q4 + 1] = a.y; pre[g][4 * q4 + 2] = a.z; pre[g][4 * q4 + 3] = a.w;
          }
      }
      mbar_wait(tfull, t & 1);
      tc_fence_after();
      if (threadIdx.x == 0) SEQ_TS(t, 4);
      uint32_t v[64];
      tmem_ld64(tmem + (static_cast<uint32_t>(warp * 32) << 16), v);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster_relaxed(tempty_leader);  // accumulator free for step t + 1
      float hv[kUpp];
      if (ok) {
#pragma unroll
        for (int uu = 0; uu < kUpp; ++uu) {
          const float gi = sigm_s(pre[0][uu] + __uint_as_float(v[uu]));
          const float gc = tanh_f(pre[1][uu] + __uint_as_float(v[kUpp + uu]));
          const float gf = sigm_s(pre[2][uu] + __uint_as_float(v[2 * kUpp + uu]));
          const float go = sigm_s(pre[3][uu] + __uint_as_float(v[3 * kUpp + uu]));
          const float sv = gf * sreg[uu] + gi * gc;
          sreg[uu] = sv;
          hv[uu] = go * tanh_f(sv);
          pre[0][uu] = gi; pre[1][uu] = gc; pre[2][uu] = gf; pre[3][uu] = go;
        }
        uint4* hb = reinterpret_cast<uint4*>(p.h_bf + (static_cast<int64_t>(t + 1) * p.N + n) * p.K + j0);
#pragma unroll
        for (int q8 = 0; q8 < kUpp / 8; ++q8)
          hb[q8] = make_uint4(pack_bf16x2(hv[8 * q8], hv[8 * q8 + 1]), pack_bf16x2(hv[8 * q8 + 2], hv[8 * q8 + 3]),
                              pack_bf16x2(hv[8 * q8 + 4], hv[8 * q8 + 5]), pack_bf16x2(hv[8 * q8 + 6], hv[8 * q8 + 7]));
      }
      fence_proxy_async_global();  // h_t (bf16) is read by other CTAs' TMA (async proxy)
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 0) {
        SEQ_TS(t, 5);
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&p.flags[(j0 / 64) * kFlagStride]) : "memory");
      }
      // off the critical path: fp32 h, s and the activated gates (BPTT inputs)
      if (ok) {
        const int64_t row = static_cast<int64_t>(t) * p.N + n;
        float* go_ = p.gates_out + row * 4 * p.K + j0;
#pragma unroll
        for (int g = 0; g < 4; ++g)
#pragma unroll
          for (int q4 = 0; q4 < kUpp / 4; ++q4)
            __stcs(reinterpret_cast<float4*>(go_ + g * p.K + 4 * q4),
                   make_float4(pre[g][4 * q4], pre[g][4 * q4 + 1], pre[g][4 * q4 + 2], pre[g][4 * q4 + 3]));
        float* ho = p.h_out + row * p.K + j0;
        float* so = p.s_out + row * p.K + j0;
#pragma unroll
        for (int q4 = 0; q4 < kUpp / 4; ++q4) {
          __stcs(reinterpret_cast<float4*>(ho + 4 * q4), make_float4(hv[4 * q4], hv[4 * q4 + 1], hv[4 * q4 + 2], hv[4 * q4 + 3]));
          __stcs(reinterpret_cast<float4*>(so + 4 * q4),
                 make_float4(sreg[4 * q4], sreg[4 * q4 + 1], sreg[4 * q4 + 2], sreg[4 * q4 + 3]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 64);
  }
}

// ------------------------------------------------------------------ backward
// Cluster of 4 CTAs: rank g = gate.  Units u0 = 32 * cluster .. +31.
__global__ void __launch_bounds__(kThreadsS, 1) lstm_seq_bwd_kernel(const __grid_constant__ SeqParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int KC = p.K / 64;
  uint8_t* ring = smem;
  constexpr int NS = kStagesS;  // (p.stages == kStagesS: checked at launch)
  uint8_t* wsm = smem + NS * p.stage_bytes;                // R_g^T slice: 32 rows x K
  float* part = reinterpret_cast<float*>(wsm + KC * kJb * 128);  // [256][32] partial dh_rec
  uint64_t* full = reinterpret_cast<uint64_t*>(part + 256 * kJb);
  uint64_t* empty = full + kStagesS;  // (barrier arrays sized for the maximum)
  uint64_t* tfull = empty + kStagesS;
  uint64_t* tempty = tfull + 1;
  uint64_t* wbar = tempty + 1;
  uint64_t* pready = wbar + 1;  // all 16 epilogue warps of the cluster wrote their partials
  uint64_t* pfree = pready + 1;  // all 16 finished reading them
  uint32_t* tslot = reinterpret_cast<uint32_t*>(pfree + 1);
  const int warp = warp_id(), lane = threadIdx.x & 31;
  const int g = static_cast<int>(cluster_ctarank());
  const int u0 = (blockIdx.x >> 2) * kJb;
  const int n_mt = p.N > 128 ? 2 : 1;
  const int chunk_owners = 2 * 4;  // 64-column chunk of dpre = 2 clusters x 4 CTAs (row quarters)

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    mbar_init(wbar, 1);
    mbar_init(pready, 16);
    mbar_init(pfree, 16);
    fence_barrier_init();
  }
  if (warp == 4) tmem_alloc(tslot, 64);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp >= 5) {
    const int pid = warp - 5;
    if (elect_one()) {
      if (pid == 0) {  // R_g^T rows u0 .. u0+31 (RT_cat[g*K + u][k] = R_g[k][u])
        mbar_arrive_expect_tx(wbar, KC * kJb * 128);
        for (int kc = 0; kc < KC; ++kc) {
          const int32_t c[2] = {kc * 64, g * p.K + u0};
          tma_load<2>(wsm + kc * kJb * 128, &p.map_w, wbar, c);
        }
      }
      // steps t = T-2 .. 0 read dpre(t+1) gate g; step T-1 has no recurrent term
      const int steps = p.T - 1;
      const int total = steps * KC;
      for (int gi = pid; pid < NS && gi < total; gi += NS) {
        const int it = gi / KC, kc = gi - it * KC;
        const int tsrc = p.T - 1 - it;  // dpre slot read by this iteration
        const int fidx = g * KC + kc;
        while (ld_acquire(&p.flags[fidx * kFlagStride]) < static_cast<unsigned>(chunk_owners * (it + 1))) poll_backoff();
        fence_proxy_async_global();
        if (kc == 0) SEQ_TS(it, 0);
        if (kc == KC - 1) SEQ_TS(it, 1);
        const uint32_t ph = (gi / NS) & 1;
        mbar_wait(&empty[pid], ph ^ 1);
        mbar_arrive_expect_tx(&full[pid], static_cast<uint32_t>(p.stage_tx));
        tma_load3(ring + pid * p.stage_bytes, &p.map_a, &full[pid], g * p.K + kc * 64, 0, tsrc);
      }
    }
  } else if (warp == 4) {
    const uint32_t idesc = make_idesc(kFmtBF16, 128, kJb, 0, 0);
    const uint64_t ring_desc = make_smem_desc(smem_u32(ring), 16, 1024, kSwizzle128B);
    const uint64_t w_desc = make_smem_desc(smem_u32(wsm), 16, 1024, kSwizzle128B);
    mbar_wait(wbar, 0);
    for (int it = 0; it < p.T - 1; ++it) {
      mbar_wait(tempty, (it & 1) ^ 1);
      tc_fence_after();
      for (int kc = 0; kc < KC; ++kc) {
        const int gi = it * KC + kc, st = gi % NS;
        mbar_wait(&full[st], (gi / NS) & 1);
        tc_fence_after();
        if (lane == 0 && kc == 0) SEQ_TS(it, 2);
        if (lane == 0 && kc == KC - 1) SEQ_TS(it, 3);
        if (elect_one()) {  // descriptors advanced by constants (16-byte units), see brk_engine.cu
          const uint64_t ad = ring_desc + static_cast<uint32_t>(st * p.stage_bytes) / 16;
          const uint64_t bd = w_desc + static_cast<uint32_t>(kc * kJb * 128 / 16);
          for (int mt = 0; mt < n_mt; ++mt)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_ss<false>(tmem + mt * kJb, ad + mt * 1024 + kk * 2, bd + kk * 2, idesc, (kc | kk) ? 1u : 0u);
          mma_commit(&empty[st]);
          if (kc == KC - 1) mma_commit(tfull);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------ epilogue: 128 threads
    // finalize rows r = 64*g + tid/2 (this CTA's quarter), units half = tid%2 (16 units)
    const int tid = threadIdx.x;
    const int rq = 64 * g + (tid >> 1);
    const int uh = (tid & 1) * 16;
    float dsc[16];  // ds_t * f_t carried to step t-1
#pragma unroll
    for (int q = 0; q < 16; ++q) dsc[q] = 0.0f;
    uint32_t part_peer[4], ready_peer[4], free_peer[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      part_peer[r] = mapa_shared(smem_u32(part), r);
      ready_peer[r] = mapa_shared(smem_u32(pready), r);
      free_peer[r] = mapa_shared(smem_u32(pfree), r);
    }
    for (int t = p.T - 1; t >= 0; --t) {
      const int it = p.T - 1 - t;
      const int q = it - 1;  // index of the recurrent step (t < T-1)
      // Everything but the recurrent term is known before the MMAs finish: load
      // this step's gates / states / dh and fold them into per-element factors
      //   ds = (dh + dh_rec) * A + dsc ; dpre_i = ds*CI ; dpre_c = ds*IC ;
      //   dpre_f = ds*SF ; dpre_o = (dh + dh_rec) * B ; dsc <- ds * f
      float fdh[16], fA[16], fB[16], fCI[16], fIC[16], fSF[16], ff[16];
      const bool row_ok = rq < p.N;
      const int64_t row = static_cast<int64_t>(t) * p.N + rq;
      if (row_ok) {
        const float* gr = p.gates + row * 4 * p.K + u0 + uh;
        const float* sr = p.s + row * p.K + u0 + uh;
        const float* spr = t > 0 ? p.s + (row - p.N) * p.K + u0 + uh : (p.s0 ? p.s0 + rq * p.K + u0 + uh : nullptr);
        const float* dhi = p.dh + row * p.K + u0 + uh;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const float4 vi = __ldcs(reinterpret_cast<const float4*>(gr + q4 * 4));
          const float4 vc = __ldcs(reinterpret_cast<const float4*>(gr + p.K + q4 * 4));
          const float4 vf = __ldcs(reinterpret_cast<const float4*>(gr + 2 * p.K + q4 * 4));
          const float4 vo = __ldcs(reinterpret_cast<const float4*>(gr + 3 * p.K + q4 * 4));
          const float4 vs = *reinterpret_cast<const float4*>(sr + q4 * 4);
          const float4 vsp = spr ? *reinterpret_cast<const float4*>(spr + q4 * 4) : make_float4(0, 0, 0, 0);
          const float4 vdh = __ldcs(reinterpret_cast<const float4*>(dhi + q4 * 4));
          const float ai[4] = {vi.x, vi.y, vi.z, vi.w}, ac[4] = {vc.x, vc.y, vc.z, vc.w};
          const float af[4] = {vf.x, vf.y, vf.z, vf.w}, ao[4] = {vo.x, vo.y, vo.z, vo.w};
          const float as[4] = {vs.x, vs.y, vs.z, vs.w}, asp[4] = {vsp.x, vsp.y, vsp.z, vsp.w};
          const float adh[4] = {vdh.x, vdh.y, vdh.z, vdh.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int k = q4 * 4 + e;
            const float ts = tanh_f(as[e]);
            fdh[k] = adh[e];
            fA[k] = ao[e] * (1.0f - ts * ts);
            fB[k] = ts * ao[e] * (1.0f - ao[e]);
            fCI[k] = ac[e] * ai[e] * (1.0f - ai[e]);
            fIC[k] = ai[e] * (1.0f - ac[e] * ac[e]);
            fSF[k] = asp[e] * af[e] * (1.0f - af[e]);
            ff[k] = af[e];
          }
        }
      }
      if (t < p.T - 1) {
        if (q > 0) mbar_wait_acq_cluster(pfree, (q - 1) & 1);  // peers done reading the last partials
        mbar_wait(tfull, q & 1);
        tc_fence_after();
        if (threadIdx.x == 0) SEQ_TS(q, 4);
        // partial dh_rec rows (both M-tiles) -> own smem [256][32]
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          if (mt >= n_mt) break;
          uint32_t v[32];
          tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + mt * kJb, v);
          tmem_ld_wait();
          float4* dst = reinterpret_cast<float4*>(part + (mt * 128 + warp * 32 + lane) * kJb);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            dst[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                 __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(tempty);
#pragma unroll
          for (int r = 0; r < 4; ++r) mbar_arrive_cluster(ready_peer[r]);  // release: partial rows written
        }
        mbar_wait_acq_cluster(pready, q & 1);  // the four gate partials are in the cluster's smem
        if (threadIdx.x == 0) SEQ_TS(q, 5);
      }
      if (row_ok) {
        float dhr[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) dhr[q] = 0.0f;
        if (t < p.T - 1) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const uint32_t base = part_peer[r] + static_cast<uint32_t>((rq * kJb + uh) * 4);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 v4 = ld_dsmem_f4(base + q * 16);
              dhr[4 * q] += v4.x; dhr[4 * q + 1] += v4.y; dhr[4 * q + 2] += v4.z; dhr[4 * q + 3] += v4.w;
            }
          }
        }
        __nv_bfloat16* dp = p.dpre + row * 4 * p.K + u0 + uh;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          float o_i[4], o_c[4], o_f[4], o_o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int k = q4 * 4 + e;
            const float dht = fdh[k] + dhr[k];
            const float ds = dht * fA[k] + dsc[k];
            o_i[e] = ds * fCI[k];
            o_c[e] = ds * fIC[k];
            o_f[e] = ds * fSF[k];
            o_o[e] = dht * fB[k];
            dsc[k] = ds * ff[k];
          }
          *reinterpret_cast<uint2*>(dp + q4 * 4) = make_uint2(pack_bf16x2(o_i[0], o_i[1]), pack_bf16x2(o_i[2], o_i[3]));
          *reinterpret_cast<uint2*>(dp + p.K + q4 * 4) =
              make_uint2(pack_bf16x2(o_c[0], o_c[1]), pack_bf16x2(o_c[2], o_c[3]));
          *reinterpret_cast<uint2*>(dp + 2 * p.K + q4 * 4) =
              make_uint2(pack_bf16x2(o_f[0], o_f[1]), pack_bf16x2(o_f[2], o_f[3]));
          *reinterpret_cast<uint2*>(dp + 3 * p.K + q4 * 4) =
              make_uint2(pack_bf16x2(o_o[0], o_o[1]), pack_bf16x2(o_o[2], o_o[3]));
        }
        if (t == 0 && p.ds0 != nullptr) {
          float* d0 = p.ds0 + static_cast<int64_t>(rq) * p.K + u0 + uh;
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4)
            *reinterpret_cast<float4*>(d0 + 4 * q4) = make_float4(dsc[4 * q4], dsc[4 * q4 + 1], dsc[4 * q4 + 2],
                                                                  dsc[4 * q4 + 3]);
        }
      }
      fence_proxy_async_global();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 0) {
        if (t < p.T - 1) SEQ_TS(it - 1, 6);
        // this CTA wrote rows of its quarter for units u0..u0+31 of all four gates: one release
        // fence, then relaxed adds (rather than an SC fence + atomics)
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
#pragma unroll
        for (int gg = 0; gg < 4; ++gg)
          asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(&p.flags[((gg * p.K + u0) / 64) * kFlagStride])
                       : "memory");
      }
      if (t < p.T - 1) {
        __syncwarp();
        if (lane == 0) {
#pragma unroll
          for (int r = 0; r < 4; ++r) mbar_arrive_cluster(free_peer[r]);  // done reading the partials
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while a peer may still read its shared memory
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}

unsigned long long* g_seq_ts = nullptr;

// CTA-pair forward (lstm_seq_fwd_pair_kernel): K a multiple of 64, N <= 256; BRK_LSTM_PAIR=0
// selects the single-CTA kernel
bool use_fwd_pair(int N, int K) {
  const char* env = std::getenv("BRK_LSTM_PAIR");
  return !(env != nullptr && std::atoi(env) == 0) && K % 64 == 0 && N <= 256 && N >= 1;
}
int smem_fwd_pair(int K) { return kStagesS * 16384 + (K / 64) * (2 * kUpp) * 128 + 256 + 1024; }

int launch_fwd_pair(SeqParams& p, void* h_bf, const void* r_cat, cudaStream_t st) {
  const int N = p.N, K = p.K, T = p.T;
  int rc;
  p.slice = ((N + 1) / 2 + 7) / 8 * 8;  // batch rows per CTA of the pair
  {
    const uint64_t dims[3] = {(uint64_t)K, (uint64_t)N, (uint64_t)(T + 1)};
    const uint64_t strides[3] = {1, (uint64_t)K, (uint64_t)N * K};
    const uint32_t box[3] = {64, static_cast<uint32_t>(p.slice), 1};
    if ((rc = encode_tmap(&p.map_a, h_bf, true, 3, dims, strides, box))) return rc;
  }
  {
    const uint64_t dims[2] = {(uint64_t)K, (uint64_t)(4 * K)};
    const uint64_t strides[2] = {1, (uint64_t)K};
    const uint32_t box[2] = {64, static_cast<uint32_t>(kUpp)};
    if ((rc = encode_tmap(&p.map_w, r_cat, true, 2, dims, strides, box))) return rc;
  }
  const int smem = smem_fwd_pair(K);
  if (smem > 232448) return set_error(BRK_ERR_CONTRACT, "lstm seq fwd: K too large for the resident slice");
  cudaError_t err = cudaFuncSetAttribute(lstm_seq_fwd_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (err != cudaSuccess) return set_cuda_error(err, "lstm seq fwd pair smem");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * (K / kUpp));
  cfg.blockDim = dim3(kThreadsS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // the pairs wait on each other's chunks: the whole grid must be co-resident
  int max_clusters = 0;
  err = cudaOccupancyMaxActiveClusters(&max_clusters, lstm_seq_fwd_pair_kernel, &cfg);
  if (err != cudaSuccess) return set_cuda_error(err, "lstm seq fwd pair occupancy");
  if (max_clusters < K / kUpp) return set_error(BRK_ERR_CONTRACT, "lstm seq fwd pair: grid cannot be co-resident");
  err = cudaMemsetAsync(p.flags, 0, static_cast<size_t>(4 * (K / 64) + 4) * kFlagStride * sizeof(unsigned), st);
  if (err != cudaSuccess) return set_cuda_error(err, "lstm seq flags");
  g_launches.fetch_add(1);
  err = cudaLaunchKernelEx(&cfg, lstm_seq_fwd_pair_kernel, p);
  return err == cudaSuccess ? BRK_OK : set_cuda_error(err, "lstm seq fwd pair launch");
}


// streamed rows per stage: N rounded up to whole 8-row swizzle atoms (forward: cs slices of
// `slice` rows, slice = ceil(N / cs) rounded to 8)
int rows_pad(int N) { return (N + 7) / 8 * 8; }
// everything but the ring, and the ring depth that fits beside it (>= 3, else 0)
int fixed_fwd(int K) { return (K / 64) * 4 * kJf * 128 + 256 + 1024; }
int fixed_bwd(int K) { return (K / 64) * kJb * 128 + 256 * kJb * 4 + 256 + 1024; }
int ring_stages(int fixed, int stage_bytes) {
  const int n = std::min(kStagesS, (232448 - fixed) / stage_bytes);
  return n >= 3 ? n : 0;
}

int check_seq(int T, int N, int K) {
  char buf[200];
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // (worst case of the forward stage: 8 slices of ceil(N / 8) rows rounded to 8)
  if (T <= 0 || N <= 0 || N > 256 || K <= 0 || K % 64 || K / kJf > sms ||
      ring_stages(fixed_fwd(K), std::max(32768, 8 * rows_pad((N + 7) / 8) * 128)) == 0 ||
      ring_stages(fixed_bwd(K), 32768) == 0) {
    std::snprintf(buf, sizeof(buf),
                  "lstm sequence kernels need 1 <= N <= 256, K %% 64 == 0, K/8 <= %d SMs, K <= 1024 "
                  "(T=%d N=%d K=%d)", sms, T, N, K);
    return set_error(BRK_ERR_CONTRACT, buf);
  }
  return BRK_OK;
}

}  // namespace
}  // namespace brk

using namespace brk;

extern "C" {

// Diagnostic: subsequent sequence launches record per-step %globaltimer stamps of CTA 0 ([T][8]); NULL disables.
BRK_API void brk_diag_lstm_timestamps(unsigned long long* ts) { g_seq_ts = ts; }

BRK_API size_t brk_lstm_seq_flags_bytes(int K) {
  return static_cast<size_t>(4 * (K / 64) + 4) * kFlagStride * sizeof(unsigned);
}

BRK_API int brk_lstm_seq_fwd(const float* gx, const void* r_cat, const float* s0, void* h_bf, float* h_out,
                             float* s_out, float* gates_out, unsigned* flags, int T, int N, int K, void* stream) {
  int rc = check_seq(T, N, K);
  if (rc) return rc;
  SeqParams p;
  std::memset(&p, 0, sizeof(p));
  p.T = T; p.N = N; p.K = K;
  p.gx = gx; p.s0 = s0; p.h_out = h_out; p.s_out = s_out; p.gates_out = gates_out;
  p.h_bf = static_cast<__nv_bfloat16*>(h_bf);
  p.flags = flags;
  p.ts = g_seq_ts;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (use_fwd_pair(N, K)) return launch_fwd_pair(p, h_bf, r_cat, st);
  // stages are 32 KB slots (cs slices of ceil(N / cs) rows rounded to 8 never exceed 256 rows)
  const int smem = kStagesS * 32768 + fixed_fwd(K);
  cudaError_t err = cudaFuncSetAttribute(lstm_seq_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (err != cudaSuccess) return set_cuda_error(err, "lstm seq fwd smem");
  cudaFuncSetAttribute(lstm_seq_fwd_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(K / kJf);
  cfg.blockDim = dim3(kThreadsS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // largest cluster (<= 8, dividing the grid) whose clusters are all co-resident:
  // the CTAs wait on each other's chunks, so the whole grid must be resident
  const char* cs_env = std::getenv("BRK_LSTM_CS");  // tuning: largest cluster size to try
  int cs = cs_env != nullptr ? std::max(1, std::min(8, std::atoi(cs_env))) : 8;
  for (; cs >= 1; cs /= 2) {
    if ((K / kJf) % cs) continue;
    attr[0].val.clusterDim.x = cs;
    int max_clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&max_clusters, lstm_seq_fwd_kernel, &cfg) == cudaSuccess &&
        max_clusters * cs >= K / kJf)
      break;
    cudaGetLastError();
  }
  if (cs < 1) return set_error(BRK_ERR_CONTRACT, "lstm seq fwd: grid cannot be co-resident");
  {
    const uint64_t dims[3] = {(uint64_t)K, (uint64_t)N, (uint64_t)(T + 1)};
    const uint64_t strides[3] = {1, (uint64_t)K, (uint64_t)N * K};
    const char* full_env = std::getenv("BRK_LSTM_FULL_TILE");  // diagnostics: stream all 256 rows
    p.slice = (full_env != nullptr && std::atoi(full_env) != 0) ? 256 / cs : ((N + cs - 1) / cs + 7) / 8 * 8;
    p.stage_bytes = std::max(32768, p.slice * cs * 128);
    p.stage_tx = p.slice * cs * 128;
    p.stages = ring_stages(fixed_fwd(K), p.stage_bytes);
    if (p.stages != kStagesS || p.stage_bytes != 32768)
      return set_error(BRK_ERR_CONTRACT, "lstm seq fwd: ring does not fit");
    const uint32_t box[3] = {64, static_cast<uint32_t>(p.slice), 1};
    if ((rc = encode_tmap(&p.map_a, h_bf, true, 3, dims, strides, box))) return rc;
  }
  {
    const uint64_t dims[2] = {(uint64_t)K, (uint64_t)(4 * K)};
    const uint64_t strides[2] = {1, (uint64_t)K};
    const uint32_t box[2] = {64, 8};
    if ((rc = encode_tmap(&p.map_w, r_cat, true, 2, dims, strides, box))) return rc;
  }
  err = cudaMemsetAsync(flags, 0, brk_lstm_seq_flags_bytes(K), st);
  if (err != cudaSuccess) return set_cuda_error(err, "lstm seq flags");
  g_launches.fetch_add(1);
  err = cudaLaunchKernelEx(&cfg, lstm_seq_fwd_kernel, p);
  return err == cudaSuccess ? BRK_OK : set_cuda_error(err, "lstm seq fwd launch");
}

BRK_API int brk_lstm_seq_bwd(const float* dh, const float* gates, const float* s, const float* s0,
                             const void* rt_cat, void* dpre, float* ds0, unsigned* flags, int T, int N, int K,
                             void* stream) {
  int rc = check_seq(T, N, K);
  if (rc) return rc;
  if (K % kJb) return set_error(BRK_ERR_CONTRACT, "lstm seq bwd: K must be a multiple of 32");
  SeqParams p;
  std::memset(&p, 0, sizeof(p));
  p.T = T; p.N = N; p.K = K;
  p.dh = dh; p.gates = gates; p.s = s; p.s0 = s0;
  p.dpre = static_cast<__nv_bfloat16*>(dpre);
  p.ds0 = ds0;
  p.flags = flags;
  p.ts = g_seq_ts;
  {
    const uint64_t dims[3] = {(uint64_t)(4 * K), (uint64_t)N, (uint64_t)T};
    const uint64_t strides[3] = {1, (uint64_t)(4 * K), (uint64_t)N * 4 * K};
    p.stage_bytes = 32768;
    p.stage_tx = rows_pad(N) * 128;
    p.stages = ring_stages(fixed_bwd(K), p.stage_bytes);
    if (p.stages != kStagesS) return set_error(BRK_ERR_CONTRACT, "lstm seq bwd: ring does not fit");
    const uint32_t box[3] = {64, static_cast<uint32_t>(rows_pad(N)), 1};
    if ((rc = encode_tmap(&p.map_a, dpre, true, 3, dims, strides, box))) return rc;
  }
  {
    const uint64_t dims[2] = {(uint64_t)K, (uint64_t)(4 * K)};
    const uint64_t strides[2] = {1, (uint64_t)K};
    const uint32_t box[2] = {64, 32};
    if ((rc = encode_tmap(&p.map_w, rt_cat, true, 2, dims, strides, box))) return rc;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t err = cudaMemsetAsync(flags, 0, brk_lstm_seq_flags_bytes(K), st);
  if (err != cudaSuccess) return set_cuda_error(err, "lstm seq flags");
  const int smem = p.stages * p.stage_bytes + fixed_bwd(K);
  err = cudaFuncSetAttribute(lstm_seq_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (err != cudaSuccess) return set_cuda_error(err, "lstm seq bwd smem");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(4 * (K / kJb));
  cfg.blockDim = dim3(kThreadsS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 4;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int max_clusters = 0;
  err = cudaOccupancyMaxActiveClusters(&max_clusters, lstm_seq_bwd_kernel, &cfg);
  if (err != cudaSuccess) return set_cuda_error(err, "lstm seq bwd occupancy");
  if (max_clusters < K / kJb) {
    char buf[160];
    std::snprintf(buf, sizeof(buf), "lstm seq bwd: %d co-resident 4-CTA clusters needed, device offers %d",
                  K / kJb, max_clusters);
    return set_error(BRK_ERR_CONTRACT, buf);
  }
  g_launches.fetch_add(1);
  err = cudaLaunchKernelEx(&cfg, lstm_seq_bwd_kernel, p);
  return err == cudaSuccess ? BRK_OK : set_cuda_error(err, "lstm seq bwd launch");
}

}  // extern "C"
