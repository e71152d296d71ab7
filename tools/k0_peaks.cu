// K0 microbenchmarks (standalone): shared-memory atomicOr / store rates and
// HBM write bandwidth on the B200 this runs on.  Prints one JSON line.
// Rates are per SM per SM-clock (cycles measured in-kernel with clock64),
// so they do not depend on the clock the GPU happened to run at.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int SMEM_WORDS = 48 * 1024;  // 192 KB

// mode 0: conflict-free ATOMS.OR (lane l -> bank l)
// mode 1: random-address ATOMS.OR
// mode 2: random-address STS.U8
// mode 3: conflict-free STS.32
// mode 4: warp-strided "sieve-like" ATOMS.OR: lanes at j + l*p, p odd in [33, 2000)
// mode 5: random-address LDS+STS (non-atomic RMW, for reference only)
template <int MODE>
__global__ void __launch_bounds__(1024) k_smem(int iters, unsigned long long *cycles, uint32_t *sink) {
  extern __shared__ uint32_t seg[];
  for (int i = threadIdx.x; i < SMEM_WORDS; i += blockDim.x) seg[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x * 7919u;
  uint32_t p = 33 + 2 * ((warp * 37 + blockIdx.x) % 980);
  uint32_t j = (lane * p + warp * 977u) % (SMEM_WORDS * 32);
  unsigned long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (MODE == 0) {
        uint32_t w = (lane + 32 * ((warp + it * 8 + u) & 1023)) % SMEM_WORDS;
        atomicOr(&seg[w], 1u << ((it + u) & 31));
      } else if (MODE == 1) {
        x = x * 1664525u + 1013904223u;
        atomicOr(&seg[(x >> 8) % SMEM_WORDS], 1u << (x & 31));
      } else if (MODE == 2) {
        x = x * 1664525u + 1013904223u;
        reinterpret_cast<volatile unsigned char *>(seg)[(x >> 4) % (SMEM_WORDS * 4)] = 1;
      } else if (MODE == 3) {
        uint32_t w = (lane + 32 * ((warp + it * 8 + u) & 1023)) % SMEM_WORDS;
        reinterpret_cast<volatile uint32_t *>(seg)[w] = it;
      } else if (MODE == 4) {
        atomicOr(&seg[j >> 5], 1u << (j & 31));
        j += 32 * p;
        if (j >= SMEM_WORDS * 32) j -= SMEM_WORDS * 32;
      } else if (MODE == 5) {
        x = x * 1664525u + 1013904223u;
        volatile uint32_t *v = seg;
        uint32_t a = (x >> 8) % SMEM_WORDS;
        v[a] = v[a] | (1u << (x & 31));
      }
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) atomicMax(cycles, t1 - t0);
  uint32_t acc = 0;
  for (int i = threadIdx.x; i < SMEM_WORDS; i += blockDim.x) acc ^= seg[i];
  if (acc == 0x12345678u) sink[0] = acc;
}

__global__ void k_write(uint4 *out, size_t n16) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  uint4 v = make_uint4(i, i, i, i);
  for (; i < n16; i += stride) out[i] = v;
}

template <int MODE>
int run(const char *name, int nsm, int iters, unsigned long long *dcyc, uint32_t *sink) {
  CK(cudaFuncSetAttribute(k_smem<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_WORDS * 4));
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaMemset(dcyc, 0, 8));
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k_smem<MODE><<<nsm, 1024, SMEM_WORDS * 4>>>(iters, dcyc, sink);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long cyc; CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost));
    double ops_per_sm = 1024.0 * iters * 8;
    if (rep == 1)
      printf("\"%s\": {\"lanes_per_clk_per_sm\": %.3f, \"ms\": %.3f, \"cycles\": %llu, \"eff_ghz\": %.3f},\n",
             name, ops_per_sm / cyc, ms, cyc, cyc / (ms * 1e6));
  }
  return 0;
}

int main() {
  int dev = 0, nsm = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  unsigned long long *dcyc; uint32_t *sink;
  CK(cudaMalloc(&dcyc, 8)); CK(cudaMalloc(&sink, 4));
  printf("{\"sms\": %d,\n", nsm);
  int iters = 4096;
  run<0>("atoms_or_conflict_free", nsm, iters, dcyc, sink);
  run<1>("atoms_or_random", nsm, iters, dcyc, sink);
  run<2>("sts_u8_random", nsm, iters, dcyc, sink);
  run<3>("sts_32_conflict_free", nsm, iters, dcyc, sink);
  run<4>("atoms_or_warp_strided_prime", nsm, iters, dcyc, sink);
  run<5>("lds_sts_rmw_random", nsm, iters, dcyc, sink);
  // HBM write
  size_t bytes = (size_t)4 << 30;
  uint4 *buf; CK(cudaMalloc(&buf, bytes));
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k_write<<<nsm * 8, 512>>>(buf, bytes / 16);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  printf("\"stg128_write_gbs\": %.1f}\n", bytes / (best * 1e6));
  return 0;
}
