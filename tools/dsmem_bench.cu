// Distributed shared memory atomic throughput (diagnostics for SURVEY.md 8(f)
// F3): a cluster of CL CTAs, every warp issues conflict-free 32-lane
// red.shared::cluster.or.b32 to (a) its own CTA's shared memory through the
// cluster window and (b) its partner CTA's shared memory.  Prints warp
// instructions per clock per SM.
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int WORDS = 32 * 1024;  // 128 KB per CTA

__device__ __forceinline__ void red_cluster_or(uint32_t caddr, uint32_t m) {
  asm volatile("red.shared::cluster.or.b32 [%0], %1;" ::"r"(caddr), "r"(m) : "memory");
}

template <int REMOTE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(1024) k(int iters, unsigned long long *cyc) {
  extern __shared__ uint32_t seg[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < WORDS; i += blockDim.x) seg[i] = 0;
  cl.sync();
  const uint32_t rank = cl.block_rank();
  uint32_t *dst = REMOTE == 1 ? cl.map_shared_rank(seg, rank ^ 1u) : seg;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint32_t *p = dst + lane + 32 * ((warp * 37) % 64);
  const uint32_t m = 1u << lane;
  unsigned long long t0 = clock64();
  if (REMOTE == 2) {
    // explicit shared::cluster window address of the partner's word (mapa)
    uint32_t local = (uint32_t)__cvta_generic_to_shared(seg + lane + 32 * ((warp * 37) % 64));
    uint32_t caddr;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(caddr) : "r"(local), "r"(rank ^ 1u));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int u = 0; u < 16; ++u) red_cluster_or(caddr + u * 4096, m);
      caddr += (it & 1) ? -128 : 128;
    }
  } else {
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) atomicOr(p + u * 1024, m);
    p += (it & 1) ? -32 : 32;
  }
  }
  cl.sync();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) atomicMax(cyc, t1 - t0);
}

int main() {
  unsigned long long *d;
  cudaMalloc(&d, 8);
  for (int remote = 0; remote < 3; ++remote) {
    auto f = remote == 2 ? k<2> : remote ? k<1> : k<0>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, WORDS * 4);
    const int iters = 2000;
    cudaMemset(d, 0, 8);
    f<<<148, 1024, WORDS * 4>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double instr = 32.0 * iters * 16;  // warp instructions per CTA (one CTA per SM)
    printf("{\"remote\": %d, \"err\": \"%s\", \"cycles\": %llu, \"warp_atoms_per_clk_per_sm\": %.3f}\n",
           remote, cudaGetErrorString(e), c, instr / (double)c);
  }
  return 0;
}
