// peer.cuh -- SURVEY.md 8(f) F4: the all-reduce of the step-A7 result fused
// into the sieve kernel over NVLink peer memory.
//
// The paper's flow ends every node's sieve with a gather of its result
// (Fig. 6; read as SPEC.md:296).  For the pi/sum path the
// gathered result is two u64 per GPU, so the "collective" is 16 bytes: an
// NCCL all-reduce costs a separate launch and ~10 us of protocol for it.  Here
// the kernel's last CTA -- which already reduces the per-CTA partials --
// publishes its (count, sum) straight into every peer's slab through P2P
// stores and then sums the slots the peers wrote into its own slab.
//
// Slab (one per rank, kPeerSlabBytes, zeroed before the first use): two
// parities x kMaxPeers slots x {count, sum, epoch, 0} (u64).  Launch e (the
// e-th fused launch, identical on every rank: SPMD) uses parity e & 1.  Rank q
// writes slot [e & 1][q] of every rank's slab: data with relaxed sys-scope
// stores, then the epoch with a release store.  A reader acquires the epoch
// of every slot [e & 1][*] of its own slab, then reads the data.
// Double buffering makes slot reuse safe: rank q can publish e + 2 into the
// same parity only after finishing e + 1, which needed every rank's e + 1
// publication, which each rank makes only after it has read all of e.
// A wait longer than timeout_ns (a peer that never launched) ends with the
// sentinel result (2^64-1, 2^64-1) instead of a hung GPU.  peer_publish alone
// (sieve_peer_publish_async) makes a rank's share visible without waiting,
// so that no two kernels ever wait on each other (the cross-process test on
// one GPU).
#pragma once
#include <cstdint>

namespace sv {

constexpr int kMaxPeers = 64;
constexpr size_t kPeerSlabBytes = 2ull * kMaxPeers * 4 * sizeof(uint64_t);

__device__ __forceinline__ void st_relaxed_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One thread: this rank's (c, s) into slot [epoch & 1][rank] of every slab.
static __device__ __forceinline__ void peer_publish(unsigned long long *const *peers, uint32_t world,
                                                    uint32_t rank, uint64_t epoch,
                                                    unsigned long long c, unsigned long long s) {
  const uint32_t base = (uint32_t)(epoch & 1u) * kMaxPeers;
  for (uint32_t q = 0; q < world; ++q) {
    unsigned long long *slot = peers[q] + 4 * (base + rank);
    st_relaxed_sys(slot, c);
    st_relaxed_sys(slot + 1, s);
    st_release_sys(slot + 2, epoch);
  }
}

// One thread.  (c, s): this rank's result; returns the sums over all ranks
// (mod 2^64), or (2^64-1, 2^64-1) on timeout.
static __device__ __forceinline__ ulonglong2 peer_allreduce(unsigned long long *const *peers,
                                                         uint32_t world, uint32_t rank,
                                                         uint64_t epoch, uint64_t timeout_ns,
                                                         unsigned long long c,
                                                         unsigned long long s) {
  peer_publish(peers, world, rank, epoch, c, s);
  const uint32_t base = (uint32_t)(epoch & 1u) * kMaxPeers;
  const unsigned long long *mine = peers[rank];
  const unsigned long long t0 = global_ns();
  ulonglong2 tot = make_ulonglong2(0, 0);
  for (uint32_t q = 0; q < world; ++q) {
    const unsigned long long *slot = mine + 4 * (base + q);
    while (ld_acquire_sys(slot + 2) != epoch) {
      if (global_ns() - t0 > timeout_ns) return make_ulonglong2(~0ull, ~0ull);
      __nanosleep(32);
    }
    tot.x += ld_relaxed_sys(slot);
    tot.y += ld_relaxed_sys(slot + 1);
  }
  return tot;
}

}  // namespace sv
