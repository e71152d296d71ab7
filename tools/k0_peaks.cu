// K0 microbenchmarks (standalone): shared-memory atomicOr / load / store
// instruction rates and HBM write bandwidth on the B200 this runs on.  Prints
// one JSON object.  Rates are per SM per SM-clock (cycles from clock64 inside
// the kernel), so they do not depend on the clock the GPU happened to run at.
//
// The shared-memory loops issue 16 accesses per iteration at [R + imm]
// addresses (one IADD per 16 accesses), so they measure the LSU/shared pipe,
// not the integer ALUs.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int SMEM_WORDS = 48 * 1024;  // 192 KB

// MODE 0: ATOMS.OR, 32 lanes in 32 distinct banks
// MODE 1: ATOMS.OR, 2-way bank conflict (lane pairs share a bank)
// MODE 2: ATOMS.OR, 4-way bank conflict
// MODE 3: STS.32, 32 distinct banks
// MODE 4: LDS.32, 32 distinct banks
// MODE 5: ATOMS.OR, 16 active lanes, distinct banks
// MODE 6: ATOMS.OR, random addresses (LCG per lane; ALU-heavy)
template <int MODE>
__global__ void __launch_bounds__(1024) k_smem(int iters, unsigned long long *cycles, uint32_t *sink) {
  extern __shared__ uint32_t seg[];
  for (int i = threadIdx.x; i < SMEM_WORDS; i += blockDim.x) seg[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t bank = lane;
  if (MODE == 1) bank = lane >> 1;
  if (MODE == 2) bank = lane >> 2;
  // word = bank + 32 * row; rows spread per lane so that conflicting lanes hit different words
  uint32_t row = (warp * 37 + lane * 7) % 64;
  uint32_t *p = seg + bank + 32 * row;
  const uint32_t m = 1u << (lane & 31);
  uint32_t acc = 0, x = 0x9E3779B9u * (threadIdx.x + 1);
  const bool active = MODE != 5 || lane < 16;
  unsigned long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    if (MODE == 6) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        x = x * 1664525u + 1013904223u;
        atomicOr(&seg[x >> 17], m);  // x>>17 < 32768 words
      }
    } else if (active) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        if (MODE == 3) reinterpret_cast<volatile uint32_t *>(p)[u * 1024] = it;
        else if (MODE == 4) acc += reinterpret_cast<volatile uint32_t *>(p)[u * 1024];
        else atomicOr(p + u * 1024, m);
      }
    }
    p += (it & 1) ? -32 : 32;
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) atomicMax(cycles, t1 - t0);
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
int run(const char *name, int nsm, int iters, unsigned long long *dcyc, uint32_t *sink, bool last = false) {
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
    const double lanes = (MODE == 5 ? 16.0 : 32.0) * 32 /*warps*/ * iters * 16;
    const double instr = 32.0 * iters * 16;
    if (rep == 1)
      printf("\"%s\": {\"lanes_per_clk_per_sm\": %.3f, \"warp_instr_per_clk_per_sm\": %.3f, \"ms\": %.3f, \"eff_ghz\": %.3f},\n",
             name, lanes / cyc, instr / cyc, ms, cyc / (ms * 1e6));
  }
  return 0;
}

int main() {
  int nsm = 0;
  CK(cudaSetDevice(0));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  unsigned long long *dcyc; uint32_t *sink;
  CK(cudaMalloc(&dcyc, 8)); CK(cudaMalloc(&sink, 4));
  printf("{\"sms\": %d,\n", nsm);
  const int iters = 2048;
  run<0>("atoms_or_conflict_free", nsm, iters, dcyc, sink);
  run<1>("atoms_or_2way", nsm, iters, dcyc, sink);
  run<2>("atoms_or_4way", nsm, iters, dcyc, sink);
  run<3>("sts32_conflict_free", nsm, iters, dcyc, sink);
  run<4>("lds32_conflict_free", nsm, iters, dcyc, sink);
  run<5>("atoms_or_16_lanes", nsm, iters, dcyc, sink);
  run<6>("atoms_or_random", nsm, iters, dcyc, sink);
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
