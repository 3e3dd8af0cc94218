// brk_sched.cuh — device side of the grouped (multi-problem) persistent launches:
// dependency counters between the problems of one launch (see GroupSched in
// brk_engine.h).  Shared by the generic grouped engine and the fused MLP step.
#pragma once
#include <cstdint>

#include "brk_engine.h"
#include "brk_ptx.cuh"

namespace brk {
namespace {

#ifndef BRK_POLL_SLEEP
#define BRK_POLL_SLEEP 128
#endif
constexpr unsigned kPollSleepNs = BRK_POLL_SLEEP;

// Grouped launches: block until the tiles this tile consumes are complete.  One
// thread per CTA polls the global counters (producer 0) and publishes the tile
// ordinal in shared memory; the other producers and the epilogue wait on that
// (polling pressure on the counters' L2 lines slowed the whole step down).
__device__ __forceinline__ void publish_deps(uint32_t* seq, uint32_t ordinal) {
  asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(smem_u32(seq)), "r"(ordinal) : "memory");
}
__device__ __forceinline__ void wait_published(const uint32_t* seq, uint32_t ordinal, bool async_reads) {
  uint32_t v;
  long long spins = 0;
  do {
    asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(seq)) : "memory");
    if (++spins > (1ll << 31)) __trap();
  } while (static_cast<int32_t>(v - ordinal) < 0);
  if (async_reads) asm volatile("fence.proxy.async.global;" ::: "memory");  // TMA reads follow
}
template <class Prob>
__device__ __forceinline__ void wait_deps(const GroupSched* gs, const Prob* P, int prob, int mb, int halves) {
  for (int d = 0; d < kMaxDeps; ++d) {
    const int q = gs->dep_prob[prob][d];
    if (q < 0 || gs->dep_mode[prob][d] == 2) continue;  // chunk deps: per k-step (wait_chunk)
    const bool whole = gs->dep_mode[prob][d] != 0;
    const unsigned* c = gs->counters + q * kCounterStride + (whole ? kCounterStride - 1 : mb);
    const unsigned need = static_cast<unsigned>(halves * (whole ? P[q].m_tiles * P[q].n_tiles : P[q].n_tiles));
    unsigned v;
    long long spins = 0;
    do {
      // acquiring probes: measured to observe the producer's release sooner than relaxed
      // polling followed by a fence (profiles/r01b_summary.md)
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
      if (++spins > (1ll << 31)) __trap();  // a dependency that never completes is a bug: fail loudly
      if (v < need) __nanosleep(kPollSleepNs);  // back off: fewer probes on the counter's L2 line
    } while (v < need);
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");  // the producer's TMA reads follow
}

__device__ __forceinline__ bool has_dep_mode(const GroupSched* gs, int prob, bool chunk) {
  bool any = false;
#pragma unroll
  for (int d = 0; d < kMaxDeps; ++d)
    any |= gs->dep_prob[prob][d] >= 0 && ((gs->dep_mode[prob][d] == 2) == chunk);
  return any;
}
// dep_mode 2: block until the 64-column chunk s (rows of row block mb, CTA rank r) of every
// chunk dependency is stored, then order the TMA reads after it.
__device__ __forceinline__ void wait_chunk(const GroupSched* gs, int prob, int mb, int rank, int s) {
  for (int d = 0; d < kMaxDeps; ++d) {
    const int q = gs->dep_prob[prob][d];
    if (q < 0 || gs->dep_mode[prob][d] != 2) continue;
    const unsigned* c = gs->chunk_counters + ((q * gs->chunk_mb + mb) * 2 + rank) * gs->chunk_n + s;
    unsigned v;
    long long spins = 0;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
      if (++spins > (1ll << 31)) __trap();
      if (v < static_cast<unsigned>(gs->chunk_target)) __nanosleep(64);
    } while (v < static_cast<unsigned>(gs->chunk_target));
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// One epilogue warp's part of a 64-column chunk is stored: make it visible to the TMA reads
// of dependent tiles (generic -> async proxy, then a release add).
__device__ __forceinline__ void release_chunk(const GroupSched* gs, int prob, int mb, int rank, int chunk, int lane) {
  if (gs == nullptr || gs->chunk_counters == nullptr) return;
  asm volatile("fence.proxy.async.global;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    atomicAdd(gs->chunk_counters + ((prob * gs->chunk_mb + mb) * 2 + rank) * gs->chunk_n + chunk, 1u);
  }
}

}  // namespace
}  // namespace brk
