// brk_mlp.cu — the whole MLP training step (BASELINE config 2: L x FC(C) + bias
// + ReLU, fwd / bwd-data / weight update + SGD) as ONE lean persistent
// tcgen05 launch.  See brk_mlp.h.
//
// Roles (512 threads, one CTA per SM, CTA pairs = clusters of 2):
//   warps 0..7   epilogue: warp w drains TMEM lane quarter w % 4 (32 rows) and
//                column half w / 4 (64 columns = one 64-wide output block) of the
//                CTA's 128 x 128 accumulator with ONE tcgen05.ld (x64), frees the
//                accumulator, runs its problem kind's epilogue into a 32 x 128 B
//                staging tile (128B swizzle, the TMA box layout) and stores it
//                with one TMA store; side operands (dy, ReLU mask, old weights)
//                were TMA-loaded into the warp's second staging tile before the
//                accumulator was ready.
//   warp 8       MMA issuer (leader CTA): tcgen05.mma cta_group::2, M = 256, N = 128.
//   warps 9..14  TMA producers, one ring stage each (a TMA-issuing warp keeps about
//                one box in flight, brk_diag_tma_bw).
// Scheduling (tile order, dependency counters, 64-column chunk releases) is the
// grouped engine's (brk_sched.cuh), so the host builds the same GroupSched.
#include <algorithm>
#include <vector>
#include <cstdio>
#include <cstring>
#include <cstdlib>

#include "brk_internal.h"
#include "brk_mlp.h"
#include "brk_ptx.cuh"
#include "brk_sched.cuh"

namespace brk {
namespace {

constexpr int kEpiWarps = 8;
constexpr int kMmaWarp = kEpiWarps;
constexpr int kThreads = 16 * 32;
constexpr int kABytes = 128 * 128;  // per CTA per k-step: 128 rows x 128 B (64 bf16 / 32 fp32)
constexpr int kBBytes = 64 * 128;   // per CTA per k-step: 64 rows (N / 2) x 128 B
constexpr int kStageBytes = kABytes + kBBytes;
constexpr uint32_t kTxBytes = 2 * kStageBytes;  // both CTAs' boxes complete on the leader's barrier
constexpr int kEpiTile = 4096;                  // 32 rows x 128 B
constexpr int kBarBytes = 256;
constexpr int kBN = 128;
// bf16: 6 ring stages, 2 staging tiles per epilogue warp (+ bias broadcast area); TF32 (fp32
// outputs and side operands are two 32-column boxes each): 4 stages, 4 tiles, bias by shuffles
template <bool kTF32>
struct MlpCfg {
  static constexpr int kStages = kTF32 ? 4 : 6;
  static constexpr int kProducers = kStages;
  static constexpr int kTiles = kTF32 ? 4 : 2;
  static constexpr int kEpiBytes = kEpiWarps * kTiles * kEpiTile;
  static constexpr int kBiasBytes = kTF32 ? 0 : kEpiWarps * 256;
  static constexpr int kSmem = kStages * kStageBytes + kEpiBytes + kBiasBytes + kBarBytes + 1024;
  static_assert(kSmem <= 232448, "shared memory budget");
};

__device__ __forceinline__ uint32_t relu_pack(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint32_t bf16_pack(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a)
               : "memory");
  return v;
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a)
               : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// dep_mode 2 wait (brk_sched.cuh wait_chunk) with the MLP kernel's polling options (flags):
// bit 2 relaxed probes and one acquire fence once the count is reached (slower: 75.9 vs
// 68.4 us per step), bits 4/5 back-off 16 ns / none instead of 64 ns
__device__ __forceinline__ void mlp_wait_chunk(const GroupSched* gs, int prob, int mb, int rank, int s, int flags) {
  const bool relaxed = (flags & 4) != 0;
  const unsigned sleep_ns = (flags & 32) ? 0u : ((flags & 16) ? 16u : 64u);
  for (int d = 0; d < kMaxDeps; ++d) {
    const int q = gs->dep_prob[prob][d];
    if (q < 0 || gs->dep_mode[prob][d] != 2) continue;
    const unsigned* c = gs->chunk_counters + ((q * gs->chunk_mb + mb) * 2 + rank) * gs->chunk_n + s;
    unsigned v;
    long long spins = 0;
    do {
      if (relaxed) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
      else asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
      if (++spins > (1ll << 31)) __trap();  // a dependency that never completes is a bug: fail loudly
      if (v < static_cast<unsigned>(gs->chunk_target) && sleep_ns) __nanosleep(sleep_ns);
    } while (v < static_cast<unsigned>(gs->chunk_target));
  }
  if (relaxed) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");  // the TMA reads follow
}

// smem operand descriptor of MMA sub-step kk (32 bytes of K) — 128B swizzle.  MN-major: bf16
// atoms of 64 K-rows x 128 B (8-row groups 1024 B apart); TF32 the 32 B-chunk swizzle with
// atoms of 32 K-rows (4-row groups 512 B apart), 8 K-rows per MMA (as brk_engine.cu)
template <bool kTF32>
__device__ __forceinline__ uint64_t op_desc(uint32_t base, int mn_major, int kk) {
  if (!mn_major) return make_smem_desc(base + kk * 32, 16, 1024, kSwizzle128B);
  if constexpr (kTF32) return make_smem_desc(base + kk * 8 * 128, 32 * 128, 512, kSwizzle128B32);
  return make_smem_desc(base + kk * 16 * 128, 64 * 128, 1024, kSwizzle128B);
}

// k-step s of row block `row` -> box coordinates (see MlpProb)
template <int kDims>
__device__ __forceinline__ void op_coords(const int32_t* rc, const int32_t* k0, const int32_t* k1, int row, int d0,
                                          int d1, int32_t (&c)[kDims]) {
#pragma unroll
  for (int d = 0; d < kDims; ++d) c[d] = rc[d] * row + k0[d] * d0 + k1[d] * d1;
}

// fp32 column sums over the 32 rows of two staged 32-column fp32 boxes (columns 0-31 in ta,
// 32-63 in tb): lane l sums columns 2l, 2l + 1 and stores them (generic stores; the caller
// fences them before the whole-tile release)
__device__ __forceinline__ void tile_colsum_f32(uint32_t ta, uint32_t tb, int lane, float* gdst) {
  const uint32_t tile = lane < 16 ? ta : tb;
  const uint32_t c32 = (static_cast<uint32_t>(lane) * 2u) & 31u;
  const uint32_t j = c32 >> 2, wd = (c32 & 3u) << 2;
  float s0 = 0.0f, s1 = 0.0f;
#pragma unroll 8
  for (uint32_t r = 0; r < 32; ++r) {
    float2 x;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x.x), "=f"(x.y)
                 : "r"(tile + r * 128 + (((j ^ (r & 7u)) << 4) | wd)) : "memory");
    s0 += x.x;
    s1 += x.y;
  }
  *reinterpret_cast<float2*>(gdst + 2 * lane) = make_float2(s0, s1);
}

// Work unit u -> (problem, row block, column tile).  kPairs CTA pairs per cluster take
// adjacent column tiles of one row block (they share the A operand by multicast).
template <int kPairs>
__device__ __forceinline__ void locate(const GroupSched* gs, const MlpProb* P, int u, int pair, int& prob, int& mb,
                                       int& nb) {
  prob = 0;
  while (prob + 1 < gs->n_probs && u >= gs->tile_begin[prob + 1]) ++prob;
  const int rel = u - gs->tile_begin[prob];
  const int per_row = P[prob].n_tiles / kPairs;
  nb = (rel % per_row) * kPairs + pair;
  mb = rel / per_row;
}

// Column sums over the 32 rows of a staged bf16 tile: lane l sums columns 2l, 2l + 1
// (32-bit word l % 4 of 16 B chunk l / 4, which sits at chunk (l / 4) ^ (r % 8) of row r),
// into 64 floats of shared memory at `dst`; lane 0 then writes them to global by a bulk copy
// (async proxy: its completion orders them before the relaxed counter release).
__device__ __forceinline__ void tile_colsum(uint32_t tile, int lane, uint32_t dst, float* gdst) {
  const uint32_t j = static_cast<uint32_t>(lane) >> 2, wd = (static_cast<uint32_t>(lane) & 3u) << 2;
  float s0 = 0.0f, s1 = 0.0f;
#pragma unroll 8
  for (uint32_t r = 0; r < 32; ++r) {
    const uint32_t x = lds32(tile + r * 128 + (((j ^ (r & 7u)) << 4) | wd));
    s0 += __uint_as_float(x << 16);
    s1 += __uint_as_float(x & 0xffff0000u);
  }
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(dst + lane * 8), "f"(s0), "f"(s1) : "memory");
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 256;" ::"l"(gdst), "r"(dst) : "memory");
    bulk_commit();
  }
}

#ifdef BRK_DIAG
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define MLP_TT(tile, slot)                                                                   \
  do {                                                                                       \
    if (G.debug_ts != nullptr && (tile) < 16) G.debug_ts[(blockIdx.x * 16 + (tile)) * 8 + (slot)] = gtimer(); \
  } while (0)
#else
#define MLP_TT(tile, slot) \
  do {                     \
  } while (0)
#endif

// kCS = 2: one CTA pair per cluster.  kCS = 4: two pairs per cluster on adjacent column tiles
// of the same row block; the pair whose index matches the k-step's parity loads the A box and
// multicasts it into both pairs (L2 reads per k-step 96 -> 64 KB per cluster... per pair 48 -> 32).
template <int kCS, bool kTF32>
__global__ void __launch_bounds__(kThreads, 1) mlp_step_kernel(const __grid_constant__ MlpGroup G) {
  constexpr int kPairs = kCS / 2;
  using Cfg = MlpCfg<kTF32>;
  constexpr int kStages = Cfg::kStages;
  constexpr int kProducers = Cfg::kProducers;
  constexpr int kEpiBytes = Cfg::kEpiBytes;
  constexpr int kBiasBytes = Cfg::kBiasBytes;
  constexpr int kDims = kTF32 ? 5 : 4;
  const MlpProb* P = G.probs;
  const GroupSched* gs = &G.sched;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi = smem + kStages * kStageBytes;
  float* bias_area = reinterpret_cast<float*>(epi + kEpiBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(epi + kEpiBytes + kBiasBytes);  // (bias area: bf16 only)
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;   // [2]
  uint64_t* tempty = tfull + 2;        // [2]
  uint64_t* ebar = tempty + 2;         // [kEpiWarps]: epilogue side-operand loads
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ebar + kEpiWarps);
  uint32_t* deps_seq = tmem_slot + 1;
  uint32_t* exit_flag = tmem_slot + 2;

  const int warp = warp_id();
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank & 1u;  // rank within the CTA pair
  const int pair = static_cast<int>(crank >> 1);
  const bool leader = rank == 0;
  const int unit0 = static_cast<int>(blockIdx.x) / kCS;
  const int n_units = static_cast<int>(gridDim.x) / kCS;
  const int num_work = gs->tile_begin[gs->n_probs];
  // this cluster's work units: the host's list schedule (G.list) or round robin
  const bool listed = kCS == 2 && G.list_len > 0;
  const int it_begin = listed ? G.list_off[unit0] : unit0;
  const int it_end = listed ? G.list_off[unit0 + 1] : num_work;
  const int it_step = listed ? 1 : n_units;

  if (warp == kMmaWarp + 1 && lane == 0) {
    for (int q = 0; q < gs->n_probs; ++q) {
      tma_prefetch_desc(&P[q].map_a);
      tma_prefetch_desc(&P[q].map_b);
    }
    *deps_seq = 0u;
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kPairs);  // a stage is free once every pair of the cluster consumed it
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * kEpiWarps);
    }
    for (int w = 0; w < kEpiWarps; ++w) mbar_init(&ebar[w], 1);
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc_pair(tmem_slot, 2 * kBN);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();

  if (warp > kMmaWarp) {
    // ---------------------------------------------------------------- producers
    const int pid = warp - kMmaWarp - 1;
    if (pid < kProducers && elect_one()) {
      pdl_wait();
      int g = 0;
      uint32_t ordinal = 0;
      for (int it = it_begin; it < it_end; it += it_step) {
        const int u = listed ? G.list[it] : it;
        int prob, mb, nb;
        locate<kPairs>(gs, P, u, pair, prob, mb, nb);
        const MlpProb& p = P[prob];
        ++ordinal;
        const bool chunked = has_dep_mode(gs, prob, true);
        bool published = !chunked;
        bool deps_pending = !chunked || has_dep_mode(gs, prob, false);
        if (pid == 0) {
          wait_deps(gs, P, prob, mb, 2);
          if (!chunked) {
            publish_deps(deps_seq, ordinal);
            MLP_TT(static_cast<int>(ordinal) - 1, 0);
          }
          deps_pending = false;
        } else if (deps_pending && !p.b_first) {
          wait_published(deps_seq, ordinal, true);
          deps_pending = false;
        }
        const int arow = mb * 2 + static_cast<int>(rank);
        const int brow = nb * 2 + static_cast<int>(rank);
        const int n_steps = p.k_steps;
        // rotate the batch-list start per tile (concurrent tiles read different blocks)
        // k-step order: natural (tiles sharing a row block read the same A box at about the same
        // time: L2 dedup, 69.5 -> 68.6 us); flags bit 0: the per-pass engine's rotation; bit 6
        // (affinity lists): a chained tile starts with the chunks its own pair wrote last
        const int rot = (G.flags & 1) ? (mb * 7 + (nb - pair) * 3) % n_steps
                                      : ((G.flags & 64) && chunked ? (2 * nb) % n_steps : 0);
        for (int s0 = (pid - g % kProducers + kProducers) % kProducers; s0 < n_steps; s0 += kProducers) {
          const int gg = g + s0;
          const int stage = gg % kStages;
          const uint32_t phase = (gg / kStages) & 1;
          const int s = s0 + rot < n_steps ? s0 + rot : s0 + rot - n_steps;
          if (chunked) {  // before the ring wait: the poll latency overlaps the slot becoming free
            // (a TF32 k-step is 32 columns: half of a 64-column chunk)
            mlp_wait_chunk(gs, prob, mb, static_cast<int>(rank), kTF32 ? s >> 1 : s, G.flags);
            if (pid == 0 && !published) {
              publish_deps(deps_seq, ordinal);
              MLP_TT(static_cast<int>(ordinal) - 1, 0);
              published = true;
            }
          }
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * kStageBytes;
          if (leader) mbar_arrive_expect_tx(&full[stage], kTxBytes);
          const int d0 = kTF32 ? (s & 1) : s, d1 = kTF32 ? (s >> 1) : 0;
          int32_t ca[kDims], cb[kDims];
          op_coords<kDims>(p.a_rc, p.a_k0, p.a_k1, arow, d0, d1, ca);
          op_coords<kDims>(p.b_rc, p.b_k0, p.b_k1, brow, d0, d1, cb);
          if (deps_pending) {  // B (weights) does not wait for the tile's dependencies
            tma_load_pair<kDims>(sa + kABytes, &p.map_b, &full[stage], cb);
            wait_published(deps_seq, ordinal, true);
            deps_pending = false;
          } else {
            tma_load_pair<kDims>(sa + kABytes, &p.map_b, &full[stage], cb);
          }
          if constexpr (kPairs == 1) {
            tma_load_pair<kDims>(sa, &p.map_a, &full[stage], ca);
          } else if ((s & 1) == pair) {  // A into this CTA and its counterpart in the other pair
            if constexpr (kDims == 4)
              tma_load_pair_mc4(sa, &p.map_a, &full[stage], ca, static_cast<uint16_t>((1u << rank) | (4u << rank)));
          }
        }
        if (!published && pid == 0) {
          wait_chunk(gs, prob, mb, static_cast<int>(rank), 0);
          publish_deps(deps_seq, ordinal);
        }
        g += n_steps;
      }
    }
  } else if (warp == kMmaWarp) {
    // ---------------------------------------------------------------- MMA issuer (leader CTA)
    // descriptors built once per tile and advanced by constants (brk_engine.cu)
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      const uint32_t s0 = smem_u32(smem);
      constexpr uint32_t kMnInc = (kTF32 ? 8 : 16) * 128 / 16;
      for (int it = it_begin; it < it_end; it += it_step, ++local) {
        const int u = listed ? G.list[it] : it;
        int prob, mb, nb;
        locate<kPairs>(gs, P, u, pair, prob, mb, nb);
        const MlpProb& p = P[prob];
        const int a_mn = p.a_mn, b_mn = p.b_mn, n_steps = p.k_steps;
        const uint32_t idesc = make_idesc(kTF32 ? kFmtTF32 : kFmtBF16, 256, kBN, a_mn, b_mn);
        const uint64_t a0 = op_desc<kTF32>(s0, a_mn, 0), b0 = op_desc<kTF32>(s0 + kABytes, b_mn, 0);
        const uint32_t a_inc = a_mn ? kMnInc : 2u, b_inc = b_mn ? kMnInc : 2u;
        const int acc = local & 1;
        mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kBN;
        for (int s = 0; s < n_steps; ++s) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (s == 0 && lane == 0) MLP_TT(local, 1);
          const uint64_t so = static_cast<uint64_t>(stage * (kStageBytes / 16));
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_ss_pair<kTF32>(d_tmem, a0 + so + kk * a_inc, b0 + so + kk * b_inc, idesc, (s | kk) ? 1u : 0u);
            if constexpr (kPairs == 1) {
              mma_commit_pair(&empty[stage]);
              if (s == n_steps - 1) mma_commit_pair(&tfull[acc]);
            } else {  // the stage was filled by both pairs' producers: free it in all four CTAs
              mma_commit_pair_mask(&empty[stage], 0xF);
              if (s == n_steps - 1) mma_commit_pair_mask(&tfull[acc], static_cast<uint16_t>(3u << (2 * pair)));
            }
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) MLP_TT(local, 2);
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 0..7)
    pdl_wait();
    const int quarter = warp & 3, half = warp >> 2;
    const uint32_t st0 = smem_u32(epi + warp * Cfg::kTiles * kEpiTile), st1 = st0 + kEpiTile;
    const uint32_t lrow = static_cast<uint32_t>(lane) * 128;
    const uint32_t lsw = static_cast<uint32_t>(lane & 7);
    const uint32_t bias_s = smem_u32(bias_area + warp * 64);
    const uint32_t tempty_leader = mapa_shared(smem_u32(&tempty[0]), static_cast<uint32_t>(2 * pair));
    uint32_t ephase = 0;
    int local = 0;
    for (int it = it_begin; it < it_end; it += it_step, ++local) {
      const int u = listed ? G.list[it] : it;
      int prob, mb, nb;
      locate<kPairs>(gs, P, u, pair, prob, mb, nb);
      const MlpProb& p = P[prob];
      const int kind = p.kind;
#ifdef BRK_DIAG
      if (threadIdx.x == 0 && G.debug_ts != nullptr && local < 16) G.debug_ts[gridDim.x * 128 + blockIdx.x * 16 + local] = u;
#endif
      const int acc = local & 1;
      const int row0 = mb * 256 + static_cast<int>(rank) * 128 + quarter * 32;  // this warp's first row
      const int colblk = nb * 2 + half;                                          // its 64-column output block
      const bool upd = kind == kMlpUpd;
      // side operand by TMA, issued before the accumulator wait (dy is an input; the ReLU mask
      // and the weights may be written earlier in this launch: acquire the tile's dependencies)
      if (p.has_in) {
        if (kind != kMlpFwdTop) wait_published(deps_seq, static_cast<uint32_t>(local + 1), true);
        if (lane == 0) {
          // bf16: one 64-column box into the warp's second tile; fp32: two 32-column boxes into
          // its third and fourth
          constexpr int kBoxes = kTF32 ? 2 : 1;
          mbar_arrive_expect_tx(&ebar[warp], kBoxes * kEpiTile);
#pragma unroll
          for (int b = 0; b < kBoxes; ++b) {
            const int32_t c[4] = {32 * b, row0 & 63, upd ? row0 >> 6 : colblk, upd ? colblk : row0 >> 6};
            tma_load<4>(epi + (warp * Cfg::kTiles + (kTF32 ? 2 + b : 1)) * kEpiTile, &p.map_in, &ebar[warp], c);
          }
        }
      } else if (p.db_partials != nullptr) {
        wait_published(deps_seq, static_cast<uint32_t>(local + 1), false);
      }
      // this warp's 64 bias values: bf16 -> smem (read back as broadcasts), TF32 -> registers
      // (broadcast by shuffles)
      float bias0 = 0.0f, bias1 = 0.0f;
      if (kind <= kMlpFwdTop) {
        bias0 = __ldg(p.bias + colblk * 64 + lane);
        bias1 = __ldg(p.bias + colblk * 64 + 32 + lane);
        if constexpr (!kTF32) {
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(bias_s + lane * 4), "f"(bias0) : "memory");
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(bias_s + 128 + lane * 4), "f"(bias1) : "memory");
        }
      }
      mbar_wait(&tfull[acc], (local >> 1) & 1);
      tc_fence_after();
      uint32_t v[64];
      tmem_ld64(tmem_base + acc * kBN + (static_cast<uint32_t>(quarter * 32) << 16) + half * 64, v);
      tmem_ld_wait();
      if (threadIdx.x == 0) MLP_TT(local, 4);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster_relaxed(tempty_leader + acc * 8);  // accumulator free
      if (p.has_in) {
        mbar_wait(&ebar[warp], ephase);
        ephase ^= 1;
      }
      const int32_t ao[4] = {0, row0 & 63, colblk, row0 >> 6};  // activation-layout box
      float* colsum_dst = p.colsum_ws != nullptr ? p.colsum_ws + (row0 >> 5) * p.cols + colblk * 64 : nullptr;
      // lane 0, right after the chunk's TMA stores are committed: wait for their completion and
      // release the warp's 32 rows x 64 columns to dependent tiles (before the column sums).
      // The data left through TMA stores whose bulk-group completion means they are performed
      // in L2, and this thread wrote nothing else the consumers read (they acquire the counter,
      // fence the async proxy and read by TMA from L2).  A release reduction would add a
      // gpu-scope MEMBAR per warp and tile on the critical path (65.1 vs 68.4 us per step;
      // flags bit 3 restores it); determinism under thousands of back-to-back steps is a GPU
      // test (test_gpu_mlp.py).
      auto release_chunk_mlp = [&]() {
        if (threadIdx.x == 0) MLP_TT(local, 5);
        bulk_wait0();
        if (threadIdx.x == 0) MLP_TT(local, 6);
        if (!(G.flags & 2)) asm volatile("fence.proxy.async.global;" ::: "memory");
        if (gs->chunk_counters != nullptr) {
          unsigned* cc = gs->chunk_counters + ((prob * gs->chunk_mb + mb) * 2 + rank) * gs->chunk_n + colblk;
          if (G.flags & 8) red_release_add(cc, 1u);
          else asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cc) : "memory");
        }
        if (threadIdx.x == 0) MLP_TT(local, 7);
      };
      if constexpr (kTF32) {
        // fp32 storage: a warp's 32 x 64 block is two 32-column boxes.  Tiles: t[0], t[1] the
        // primary output (y / dx / dW); t[2], t[3] the side operand, overwritten in place by the
        // second output (dz of the top layer, dz of bwd-data, the new weights)
        const uint32_t t[4] = {st0, st0 + kEpiTile, st0 + 2 * kEpiTile, st0 + 3 * kEpiTile};
        const int32_t wr = row0 & 63, wb = row0 >> 6;
        if (kind <= kMlpFwdTop) {
          const bool top = kind == kMlpFwdTop;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              float x[4];
#pragma unroll
              for (int e = 0; e < 4; ++e)
                x[e] = fmaxf(__uint_as_float(v[32 * hh + 4 * c + e]) +
                                 __shfl_sync(0xffffffffu, hh ? bias1 : bias0, 4 * c + e), 0.0f);
              const uint32_t off = lrow + ((static_cast<uint32_t>(c) ^ lsw) << 4);
              sts128(t[hh] + off, __float_as_uint(x[0]), __float_as_uint(x[1]), __float_as_uint(x[2]),
                     __float_as_uint(x[3]));
              if (top) {  // dz = dy * (y > 0)
                const float4 d = lds_f4(t[2 + hh] + off);
                sts128(t[2 + hh] + off, x[0] > 0.0f ? __float_as_uint(d.x) : 0u, x[1] > 0.0f ? __float_as_uint(d.y) : 0u,
                       x[2] > 0.0f ? __float_as_uint(d.z) : 0u, x[3] > 0.0f ? __float_as_uint(d.w) : 0u);
              }
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              tma_store4(&p.map_out, t[hh], 32 * hh, wr, colblk, wb);
              if (top) tma_store4(&p.map_aux, t[2 + hh], 32 * hh, wr, colblk, wb);
            }
            bulk_commit();
            release_chunk_mlp();
          }
          if (top) tile_colsum_f32(t[2], t[3], lane, colsum_dst);
        } else if (kind <= kMlpBwdPlain) {
          // dz = acc * (mask > 0), in place over the mask (bwd-data of layers > 1); dx = acc
          const bool masked = kind == kMlpBwd;
          const int o = masked ? 2 : 0;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const uint32_t off = lrow + ((static_cast<uint32_t>(c) ^ lsw) << 4);
              uint32_t x[4] = {v[32 * hh + 4 * c], v[32 * hh + 4 * c + 1], v[32 * hh + 4 * c + 2],
                               v[32 * hh + 4 * c + 3]};
              if (masked) {
                const float4 m = lds_f4(t[2 + hh] + off);
                x[0] = m.x > 0.0f ? x[0] : 0u;
                x[1] = m.y > 0.0f ? x[1] : 0u;
                x[2] = m.z > 0.0f ? x[2] : 0u;
                x[3] = m.w > 0.0f ? x[3] : 0u;
              }
              sts128(t[o + hh] + off, x[0], x[1], x[2], x[3]);
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store4(&p.map_out, t[o], 0, wr, colblk, wb);
            tma_store4(&p.map_out, t[o + 1], 32, wr, colblk, wb);
            bulk_commit();
            release_chunk_mlp();
          }
          if (colsum_dst != nullptr) tile_colsum_f32(t[2], t[3], lane, colsum_dst);
        } else {
          // dW (fp32) from t[0], t[1]; w_next = w - lr dW in place over the old weights (t[2], t[3])
          const float lr = p.lr;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const uint32_t off = lrow + ((static_cast<uint32_t>(c) ^ lsw) << 4);
              const int b = 32 * hh + 4 * c;
              sts128(t[hh] + off, v[b], v[b + 1], v[b + 2], v[b + 3]);
              if (p.has_aux) {
                const float4 w = lds_f4(t[2 + hh] + off);
                sts128(t[2 + hh] + off, __float_as_uint(w.x - lr * __uint_as_float(v[b])),
                       __float_as_uint(w.y - lr * __uint_as_float(v[b + 1])),
                       __float_as_uint(w.z - lr * __uint_as_float(v[b + 2])),
                       __float_as_uint(w.w - lr * __uint_as_float(v[b + 3])));
              }
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              tma_store4(&p.map_out, t[hh], 32 * hh, wr, wb, colblk);
              if (p.has_aux) tma_store4(&p.map_aux, t[2 + hh], 32 * hh, wr, wb, colblk);
            }
            bulk_commit();
          }
        }
        if (colsum_dst != nullptr) __threadfence();  // generic column-sum stores before the tile release
      } else {
        if (kind <= kMlpFwdTop) {
          // y = relu(acc + bias) -> st0; top layer: dz = dy * (y > 0) in place in st1
          const bool top = kind == kMlpFwdTop;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 bl = lds_f4(bias_s + j * 32), bh = lds_f4(bias_s + j * 32 + 16);
            const uint32_t x = relu_pack(__uint_as_float(v[8 * j]) + bl.x, __uint_as_float(v[8 * j + 1]) + bl.y);
            const uint32_t y = relu_pack(__uint_as_float(v[8 * j + 2]) + bl.z, __uint_as_float(v[8 * j + 3]) + bl.w);
            const uint32_t z = relu_pack(__uint_as_float(v[8 * j + 4]) + bh.x, __uint_as_float(v[8 * j + 5]) + bh.y);
            const uint32_t w = relu_pack(__uint_as_float(v[8 * j + 6]) + bh.z, __uint_as_float(v[8 * j + 7]) + bh.w);
            const uint32_t off = lrow + ((static_cast<uint32_t>(j) ^ lsw) << 4);
            sts128(st0 + off, x, y, z, w);
            if (top) {  // relu outputs are >= +0: y > 0 <=> the bf16 bits as int16 > 0
              const uint4 d = lds128(st1 + off);
              sts128(st1 + off, d.x & __vcmpgts2(x, 0u), d.y & __vcmpgts2(y, 0u), d.z & __vcmpgts2(z, 0u),
                     d.w & __vcmpgts2(w, 0u));
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store4(&p.map_out, st0, ao[0], ao[1], ao[2], ao[3]);
            if (top) tma_store4(&p.map_aux, st1, ao[0], ao[1], ao[2], ao[3]);
            bulk_commit();
            release_chunk_mlp();
          }
          if (top) tile_colsum(st1, lane, bias_s, colsum_dst);  // (the bias values are consumed)
        } else if (kind <= kMlpBwdPlain) {
          // dz = bf16(acc) * (mask > 0) (mask: the previous layer's ReLU output, >= +0)
          const bool masked = kind == kMlpBwd;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            uint32_t x = bf16_pack(__uint_as_float(v[8 * j]), __uint_as_float(v[8 * j + 1]));
            uint32_t y = bf16_pack(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3]));
            uint32_t z = bf16_pack(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5]));
            uint32_t w = bf16_pack(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7]));
            const uint32_t off = lrow + ((static_cast<uint32_t>(j) ^ lsw) << 4);
            if (masked) {
              const uint4 m = lds128(st1 + off);
              x &= __vcmpgts2(m.x, 0u);
              y &= __vcmpgts2(m.y, 0u);
              z &= __vcmpgts2(m.z, 0u);
              w &= __vcmpgts2(m.w, 0u);
            }
            sts128(st0 + off, x, y, z, w);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store4(&p.map_out, st0, ao[0], ao[1], ao[2], ao[3]);
            bulk_commit();
            release_chunk_mlp();
          }
          if (colsum_dst != nullptr) tile_colsum(st0, lane, bias_s, colsum_dst);
        } else {
          // weight update: dW (fp32, two 32-column boxes through st0); w_next = w - lr dW (st1)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            if (hh == 1) {
              if (lane == 0) bulk_wait_read0();  // st0 free again
              __syncwarp();
            }
#pragma unroll
            for (int c = 0; c < 8; ++c)
              sts128(st0 + lrow + ((static_cast<uint32_t>(c) ^ lsw) << 4), v[32 * hh + 4 * c], v[32 * hh + 4 * c + 1],
                     v[32 * hh + 4 * c + 2], v[32 * hh + 4 * c + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store4(&p.map_out, st0, 32 * hh, row0 & 63, row0 >> 6, colblk);
              bulk_commit();
            }
            if (hh == 0 && p.has_aux) {
              const float lr = p.lr;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const uint32_t off = lrow + ((static_cast<uint32_t>(j) ^ lsw) << 4);
                const uint4 wq = lds128(st1 + off);
                const uint32_t wv[4] = {wq.x, wq.y, wq.z, wq.w};
                uint32_t o[4];
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  o[e] = bf16_pack(__uint_as_float(wv[e] << 16) - lr * __uint_as_float(v[8 * j + 2 * e]),
                                   __uint_as_float(wv[e] & 0xffff0000u) - lr * __uint_as_float(v[8 * j + 2 * e + 1]));
                sts128(st1 + off, o[0], o[1], o[2], o[3]);
              }
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store4(&p.map_aux, st1, 0, row0 & 63, row0 >> 6, colblk);
                bulk_commit();
              }
            }
          }
        }
      }
      if (upd && threadIdx.x == 0) MLP_TT(local, 5);
      if (lane == 0) bulk_wait0();  // (update kind: dW / new weights complete)
      if (upd && threadIdx.x == 0) MLP_TT(local, 6);
      // bias gradient of the layer from the column-sum partials (row-block-0 tiles of the update)
      if (upd && p.db_partials != nullptr && mb == 0 && rank == 0) {
        const int t = threadIdx.x, c = t & (kBN - 1), grp = t >> 7;  // 2 groups x 128 columns
        const int col = nb * kBN + c;
        const int per = (p.db_parts + 1) / 2, q0 = grp * per, q1 = min(p.db_parts, q0 + per);
        float s = 0.0f;
        for (int q = q0; q < q1; q += 8) {
          float x[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) x[e] = q + e < q1 ? __ldcg(p.db_partials + (q + e) * p.cols + col) : 0.0f;
#pragma unroll
          for (int e = 0; e < 8; ++e) s += x[e];
        }
        // group 1 parks its sums in its own warps' first staging tile (their stores have completed:
        // lane 0 waited above); group 0 reads thread t + 128's slot
        __syncwarp();
        const uint32_t red_mine = smem_u32(epi) + (t >> 5) * Cfg::kTiles * kEpiTile + (t & 31) * 4;
        const uint32_t red_peer = smem_u32(epi) + ((t + 128) >> 5) * Cfg::kTiles * kEpiTile + (t & 31) * 4;
        if (grp == 1) asm volatile("st.shared.f32 [%0], %1;" ::"r"(red_mine), "f"(s) : "memory");
        bar_sync(2, kEpiWarps * 32);
        if (grp == 0) {
          float o;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(o) : "r"(red_peer) : "memory");
          s += o;
          p.db_out[col] = s;
          if (p.bias_sgd != nullptr) p.bias_sgd[col] -= p.lr * s;
        }
        bar_sync(2, kEpiWarps * 32);  // the staging tiles are reused by the next tile
      }
      // whole-tile release (row-block / whole-problem counters: weight updates, in-place SGD)
      // (every warp's outputs, column sums included, left through bulk copies that lane 0
      //  waited on: relaxed increments, as for the chunk counters; flags bit 3: release)
      bar_sync(1, kEpiWarps * 32);
      if (threadIdx.x == 0) {
        unsigned* c0 = gs->counters + prob * kCounterStride;
        if (G.flags & 8) {
          red_release_add(c0 + mb, 1u);
          red_release_add(c0 + kCounterStride - 1, 1u);
        } else {
          asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(c0 + mb) : "memory");
          asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(c0 + kCounterStride - 1) : "memory");
        }
        MLP_TT(local, 3);
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 2 * kBN);
  }
  // every CTA is done with the counters: the last one out re-zeroes them for the next launch
  unsigned* exit_ctr = gs->counters + gs->n_probs * kCounterStride;
  if (threadIdx.x == 0) {
    __threadfence();
    *exit_flag = atomicAdd(exit_ctr, 1u) == gridDim.x - 1 ? 1u : 0u;
  }
  __syncthreads();
  if (*exit_flag) {
    __threadfence();
    for (int i = threadIdx.x; i <= gs->n_probs * kCounterStride; i += blockDim.x) gs->counters[i] = 0u;
    if (gs->chunk_counters != nullptr) {
      const int nc = gs->n_probs * gs->chunk_mb * 2 * gs->chunk_n;
      for (int i = threadIdx.x; i < nc; i += blockDim.x) gs->chunk_counters[i] = 0u;
    }
  }
}

}  // namespace

int engine_sm_count();

namespace {
template <int kCS, bool kTF32>
int launch_mlp_t(MlpGroup& G, cudaStream_t stream) {
  auto kern = mlp_step_kernel<kCS, kTF32>;
  constexpr int kSmem = MlpCfg<kTF32>::kSmem;
  static int attr_set = 0;
  cudaError_t err;
  if (!attr_set) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (err != cudaSuccess) return set_cuda_error(err, "mlp smem attribute");
    if (kCS > 2) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr_set = 1;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = kCS;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  // tiles spin on counters of earlier problems: every CTA must be resident at once, so the
  // grid is as many clusters as the device holds together (a persistent grid of any size works)
  static int resident = -1;
  if (resident < 0) {
    cfg.gridDim = dim3((engine_sm_count() / kCS) * kCS);
    err = cudaOccupancyMaxActiveClusters(&resident, kern, &cfg);
    if (err != cudaSuccess) return set_cuda_error(err, "mlp occupancy");
  }
  const int clusters = std::min(engine_sm_count() / kCS, resident);
  if (clusters < 1) return set_error(BRK_ERR_CONTRACT, "mlp step: no cluster fits on the device");
  cfg.gridDim = dim3(clusters * kCS);
  if (kCS == 2 && G.list_len > 0) mlp_list_schedule(G, clusters);  // for the pairs launched
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.numAttrs = 2;
  err = cudaLaunchKernelEx(&cfg, kern, G);
  if (err != cudaSuccess) return set_cuda_error(err, "mlp step launch");
  return BRK_OK;
}
}  // namespace

// Greedy list schedule of the step's work units over the CTA pairs, from a simple timing model
// of one B200 (profiles/r02/mlp_lean_timeline.txt): a unit's mainloop takes k_steps x 0.175 us
// (operand delivery bound), its epilogue ~1.4 us (bwd / top-layer kinds more), and a consumer's
// mainloop starts ~1.3 us after the release it waits for.  Units are taken in the global order
// (dependencies point backwards); each goes to the pair where it can start first, so the long
// weight-update units do not sit in front of the bwd-data chain on the pairs it needs.
void mlp_list_schedule(MlpGroup& G, int pairs) {
  const GroupSched& gs = G.sched;
  const int W = gs.tile_begin[gs.n_probs];
  G.list_len = 0;
  if (W > kMaxListUnits || pairs > kMaxListPairs || pairs < 1) return;
  // the schedule depends only on the problem structure: reuse the last one when it matches
  std::vector<int32_t> key = {pairs, gs.n_probs, G.flags};
  if (const char* env = std::getenv("BRK_MLP_SCHED"))
    for (const char* c = env; *c; ++c) key.push_back(*c);
  for (int q = 0; q < gs.n_probs; ++q) {
    key.insert(key.end(), {gs.tile_begin[q + 1], G.probs[q].k_steps, G.probs[q].kind, G.probs[q].n_tiles});
    for (int d = 0; d < kMaxDeps; ++d) key.insert(key.end(), {gs.dep_prob[q][d], gs.dep_mode[q][d]});
  }
  static std::vector<int32_t> last_key;
  static std::vector<int16_t> last_list, last_off;
  if (key == last_key) {
    std::copy(last_off.begin(), last_off.end(), G.list_off);
    std::copy(last_list.begin(), last_list.end(), G.list);
    G.list_len = static_cast<int32_t>(last_list.size());
    return;
  }
  double kStep = 0.175, kHandoff = 1.3, epi_scale = 1.0;
  if (const char* env = std::getenv("BRK_MLP_SCHED"))  // tuning: "step_us:handoff_us:epilogue_scale"
    std::sscanf(env, "%lf:%lf:%lf", &kStep, &kHandoff, &epi_scale);
  double epi[5] = {1.4, 2.1, 1.7, 1.2, 2.5};  // by MlpKind
  for (double& e : epi) e *= epi_scale;
  std::vector<double> row_done(static_cast<size_t>(gs.n_probs) * 64, 0.0), prob_done(gs.n_probs, 0.0);
  std::vector<double> free_at(pairs, 0.0);
  std::vector<std::vector<int16_t>> lists(pairs);
  for (int q = 0; q < gs.n_probs; ++q) {
    const MlpProb& p = G.probs[q];
    for (int u = gs.tile_begin[q]; u < gs.tile_begin[q + 1]; ++u) {
      const int rel = u - gs.tile_begin[q];
      const int mb = rel / p.n_tiles;
      double ready = 0.0;
      for (int d = 0; d < kMaxDeps; ++d) {
        const int s = gs.dep_prob[q][d];
        if (s < 0) continue;
        const double t = gs.dep_mode[q][d] == 1 ? prob_done[s] : row_done[static_cast<size_t>(s) * 64 + mb];
        ready = std::max(ready, t + kHandoff);
      }
      int best = 0;
      double best_start = 1e30;
      const bool chained = G.probs[q].kind != kMlpUpd;
      if ((G.flags & 64) && chained && p.m_tiles * p.n_tiles <= pairs) {
        // affinity: tile t of every chained pass on pair t (its first k-steps read the chunks
        // that pair wrote in the previous pass)
        best = rel;
        best_start = std::max(free_at[best], ready);
      } else {
        for (int c = 0; c < pairs; ++c) {
          const double st = std::max(free_at[c], ready);
          if (st < best_start - 1e-9) { best_start = st; best = c; }
        }
      }
      const double main_end = best_start + p.k_steps * kStep;
      free_at[best] = main_end;
      const double done = main_end + epi[p.kind];
      double& rd = row_done[static_cast<size_t>(q) * 64 + mb];
      rd = std::max(rd, done);
      prob_done[q] = std::max(prob_done[q], done);
      lists[best].push_back(static_cast<int16_t>(u));
    }
  }
  int n = 0;
  for (int c = 0; c < pairs; ++c) {
    G.list_off[c] = static_cast<int16_t>(n);
    for (int16_t u : lists[c]) G.list[n++] = u;
  }
  G.list_off[pairs] = static_cast<int16_t>(n);
  G.list_len = n;
  last_key = key;
  last_off.assign(G.list_off, G.list_off + pairs + 1);
  last_list.assign(G.list, G.list + n);
}

int launch_mlp_group(const MlpGroup& Gin, cudaStream_t stream) {
  const GroupSched& gs = Gin.sched;
  if (gs.n_probs < 1 || gs.n_probs > kMaxProbs || gs.counters == nullptr)
    return set_error(BRK_ERR_CONTRACT, "mlp group: 1..12 problems and a counter buffer");
  bool even = true;
  for (int q = 0; q < gs.n_probs; ++q) {
    const MlpProb& p = Gin.probs[q];
    if (gs.tile_begin[q + 1] - gs.tile_begin[q] != p.m_tiles * p.n_tiles || p.k_steps < 1)
      return set_error(BRK_ERR_CONTRACT, "mlp group: tile_begin does not match the problem's tiles");
    if (p.m_tiles > kCounterStride - 1) return set_error(BRK_ERR_CONTRACT, "mlp group: > 64 row blocks");
    for (int d = 0; d < kMaxDeps; ++d)
      if (gs.dep_prob[q][d] >= q) return set_error(BRK_ERR_CONTRACT, "mlp group: dependencies must point back");
    even = even && p.n_tiles % 2 == 0;
  }
  static MlpGroup G;
  G = Gin;
  if (Gin.tf32) return launch_mlp_t<2, true>(G, stream);
  if (Gin.cluster != 4 || !even) return launch_mlp_t<2, false>(G, stream);
  // two pairs per cluster: work units are pairs of adjacent column tiles
  for (int q = 0; q < gs.n_probs; ++q)
    G.sched.tile_begin[q + 1] = G.sched.tile_begin[q] + G.probs[q].m_tiles * G.probs[q].n_tiles / 2;
  return launch_mlp_t<4, false>(G, stream);
}

}  // namespace brk

// Diagnostics / host test of the list scheduler (no GPU): the chain-first MLP step structure
// of brk_mlp_step for L layers of width C and batch N (256 x 128 tiles), scheduled over `pairs`
// CTA pairs.  Writes the pair lists (units[offsets[c] .. offsets[c+1]) for pair c), the unit
// count per problem (tiles[q]) and each problem's dependency (dep[q], -1: none) and returns the
// number of units (0: the schedule was not built).
extern "C" BRK_API int brk_diag_mlp_schedule(int L, int N, int C, int pairs, int16_t* units, int16_t* offsets,
                                             int* tiles, int* dep) {
  using namespace brk;
  if (L < 1 || 3 * L > kMaxProbs || N % 256 || C % 256 || pairs < 1 || pairs > kMaxListPairs) return 0;
  static MlpGroup G;
  std::memset(&G, 0, sizeof(G));
  GroupSched& gs = G.sched;
  int q = 0;
  auto add = [&](int kind, int m_tiles, int n_tiles, int k_steps, int d, int mode) {
    MlpProb& p = G.probs[q];
    p.kind = kind;
    p.m_tiles = m_tiles;
    p.n_tiles = n_tiles;
    p.k_steps = k_steps;
    for (int j = 0; j < kMaxDeps; ++j) gs.dep_prob[q][j] = -1;
    gs.dep_prob[q][0] = d;
    gs.dep_mode[q][0] = mode;
    gs.tile_begin[q + 1] = gs.tile_begin[q] + m_tiles * n_tiles;
    return q++;
  };
  int fwd[8], bwd[8];
  for (int l = 0; l < L; ++l) fwd[l] = add(l == L - 1 ? kMlpFwdTop : kMlpFwd, N / 256, C / 128, C / 64, l ? fwd[l - 1] : -1, 2);
  for (int l = L; l >= 2; --l) bwd[l] = add(kMlpBwd, N / 256, C / 128, C / 64, l == L ? fwd[L - 1] : bwd[l + 1], 2);
  for (int l = L; l >= 1; --l) add(kMlpUpd, C / 256, C / 128, N / 64, l == L ? fwd[L - 1] : bwd[l + 1], 1);
  add(kMlpBwdPlain, N / 256, C / 128, C / 64, L >= 2 ? bwd[2] : fwd[L - 1], 2);
  gs.n_probs = q;
  mlp_list_schedule(G, pairs);
  if (G.list_len == 0) return 0;
  for (int i = 0; i <= pairs; ++i) offsets[i] = G.list_off[i];
  for (int i = 0; i < G.list_len; ++i) units[i] = G.list[i];
  for (int i = 0; i < q; ++i) {
    tiles[i] = gs.tile_begin[i + 1] - gs.tile_begin[i];
    dep[i] = gs.dep_prob[i][0];
  }
  return G.list_len;
}
