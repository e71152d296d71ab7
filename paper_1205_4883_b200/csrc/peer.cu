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
                            uint64_t *result, bool wait) {
  if (!wait) {  // publish only
    peer_publish(peers, world, rank, epoch, count, sum);
    return;
  }
  const ulonglong2 t = peer_allreduce(peers, world, rank, epoch, timeout_ns, count, sum);
  result[0] = t.x;
  result[1] = t.y;
}

}  // namespace

cudaError_t launch_peer_only(unsigned long long *const *peers, uint32_t world, uint32_t rank,
                             uint64_t epoch, uint64_t timeout_ns, uint64_t count, uint64_t sum,
                             uint64_t *result, cudaStream_t s, bool wait) {
  k_peer_only<<<1, 1, 0, s>>>(peers, world, rank, epoch, timeout_ns, count, sum, result, wait);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K0 ("R_atom = conflict-free shared atomicOr lanes per
// clock per SM, measured by K0 on the box in the same run"): one CTA of 1024
// threads per SM; every warp issues 16 red.shared.or per iteration at
// [R + imm] addresses, lane l always in bank l (word l + 32 k), so the loop
// measures the shared-memory atomic pipe, not the integer ALUs.  Cycles from
// clock64 inside the kernel (max over CTAs): the rate per SM-clock does not
// depend on the clock the GPU happened to run at.
namespace {
constexpr int kK0Words = 32 * 1024;  // 128 KiB
constexpr int kK0Iters = 2048;

__global__ void __launch_bounds__(1024) k_k0_atomics(unsigned long long *cycles, uint32_t *sink) {
  extern __shared__ uint32_t w[];
  for (int i = threadIdx.x; i < kK0Words; i += blockDim.x) w[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  // lanes in distinct banks; warps spread over rows so that they do not share words
  uint32_t a = (uint32_t)__cvta_generic_to_shared(w) + 4u * (lane + 32u * ((warp * 37u) % 32u));  // < 4 KiB + 16 x 8 KiB
  const uint32_t m = 1u << lane;
  const unsigned long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < kK0Iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
      asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a + (uint32_t)u * 8192u), "r"(m) : "memory");
    a = (it & 1) ? a - 128u : a + 128u;
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) atomicMax(cycles, t1 - t0);
  uint32_t acc = 0;
  for (int i = threadIdx.x; i < kK0Words; i += blockDim.x) acc ^= w[i];
  if (acc == 0x12345678u) sink[0] = acc;
}
}  // namespace

cudaError_t k0_smem_atomic_rate(int nsm, double *lanes_per_clk_per_sm, double *sm_ghz) {
  unsigned long long *cyc = nullptr;
  uint32_t *sink = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaError_t err = cudaFuncSetAttribute(k_k0_atomics, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kK0Words * 4);
  if (!err) err = cudaMalloc(&cyc, 8);
  if (!err) err = cudaMalloc(&sink, 4);
  if (!err) err = cudaEventCreate(&e0);
  if (!err) err = cudaEventCreate(&e1);
  for (int rep = 0; rep < 3 && !err; ++rep) {  // the first run warms up (module load, clocks)
    err = cudaMemset(cyc, 0, 8);
    if (!err) err = cudaEventRecord(e0);
    if (!err) {
      k_k0_atomics<<<nsm, 1024, kK0Words * 4>>>(cyc, sink);
      err = cudaGetLastError();
    }
    if (!err) err = cudaEventRecord(e1);
    if (!err) err = cudaEventSynchronize(e1);
    unsigned long long c = 0;
    float ms = 0;
    if (!err) err = cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    if (!err) err = cudaEventElapsedTime(&ms, e0, e1);
    if (!err && c) {
      *lanes_per_clk_per_sm = 32.0 * 32.0 * 16.0 * kK0Iters / (double)c;  // lanes x warps x atomics
      *sm_ghz = (double)c / (ms * 1e6);
    }
  }
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (cyc) cudaFree(cyc);
  if (sink) cudaFree(sink);
  return err;
}

}  // namespace sv
