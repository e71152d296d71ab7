// peer.cu -- SURVEY.md 8(f) F4: the fused all-reduce (peer.cuh) for a rank
// with no sieve work (an empty block of a small range): one thread publishes
// the block's (count, sum) -- (1, 2) when the block holds only 2 -- and
// waits for the peers like the sieve kernel's last CTA would.
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"
#include "peer.cuh"

namespace sv {
namespace {

__global__ void k_peer_only(unsigned long long *const *peers, uint32_t world, uint32_t rank,
                            uint64_t epoch, uint64_t timeout_ns, uint64_t count, uint64_t sum,
                            uint64_t *result) {
  const ulonglong2 t = peer_allreduce(peers, world, rank, epoch, timeout_ns, count, sum);
  result[0] = t.x;
  result[1] = t.y;
}

}  // namespace

cudaError_t launch_peer_only(unsigned long long *const *peers, uint32_t world, uint32_t rank,
                             uint64_t epoch, uint64_t timeout_ns, uint64_t count, uint64_t sum,
                             uint64_t *result, cudaStream_t s) {
  k_peer_only<<<1, 1, 0, s>>>(peers, world, rank, epoch, timeout_ns, count, sum, result);
  return cudaGetLastError();
}

}  // namespace sv
