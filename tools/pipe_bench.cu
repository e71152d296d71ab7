// Pipe-throughput microbenchmark (diagnostics): warp instructions per clock
// per SM for the integer ops the sieve's marking loops use.  8 independent
// chains per thread, 32 warps per SM, 148 x 2 CTAs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(uint32_t *out, uint32_t iters, uint32_t m) {
  uint32_t x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 7 + i;
  for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("lop3.b32 %0, %0, %1, 127, 0xB8;" : "+r"(x[i]) : "r"(m));
      if (OP == 1) asm volatile("shf.l.wrap.b32 %0, %0, %0, %1;" : "+r"(x[i]) : "r"(m));
      if (OP == 2) asm volatile("mad.lo.u32 %0, %0, %1, %1;" : "+r"(x[i]) : "r"(m));
      if (OP == 3) asm volatile("mad.hi.u32 %0, %0, %1, %1;" : "+r"(x[i]) : "r"(m));
      if (OP == 4) asm volatile("add.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(m));
      if (OP == 5) asm volatile("min.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(m));
      if (OP == 6) asm volatile("{ .reg .pred q; setp.lt.u32 q, %0, %1; @q add.u32 %0, %0, 1; }" : "+r"(x[i]) : "r"(m));
      if (OP == 7) asm volatile("shr.b32 %0, %0, 5;" : "+r"(x[i]));
      if (OP == 8) asm volatile("popc.b32 %0, %0;" : "+r"(x[i]));
      if (OP == 9) asm volatile("shfl.sync.bfly.b32 %0, %0, 1, 31, -1;" : "+r"(x[i]));
      if (OP == 10) asm volatile("{ .reg .u32 t; popc.b32 t, %0; add.u32 %0, %0, t; }" : "+r"(x[i]));
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 0x12345678u) out[0] = s;
}

int main() {
  uint32_t *out;
  cudaMalloc(&out, 4);
  const char *names[] = {"lop3", "shf.l.wrap", "mad.lo", "mad.hi", "add", "min", "setp+@p add", "shr", "popc", "shfl.bfly", "popc+add"};
  int nsm = 148, clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const uint32_t iters = 1 << 14;
  for (int op = 0; op < 11; ++op) {
    void (*f)(uint32_t *, uint32_t, uint32_t) =
        op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : op == 3 ? k<3> : op == 4 ? k<4> : op == 5 ? k<5> : op == 6 ? k<6> : op == 7 ? k<7> : op == 8 ? k<8> : op == 9 ? k<9> : k<10>;
    f<<<nsm * 2, 512>>>(out, 16, 3u);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    f<<<nsm * 2, 512>>>(out, iters, 3u);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double warp_instr = (double)nsm * 2 * 16 * iters * 8;  // per chip
    const double per_sm_per_clk = warp_instr / nsm / (ms * 1e-3 * 1.965e9);
    printf("{\"op\": \"%s\", \"warp_instr_per_clk_per_sm\": %.3f, \"ms\": %.3f}\n", names[op], per_sm_per_clk, ms);
  }
  return 0;
}
