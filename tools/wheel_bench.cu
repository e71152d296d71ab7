// Wheel-init microbenchmark (diagnostics): cycles per 32 segment words of a
// 208 KiB shared-memory segment built as the OR of 4 periodic tables (the
// wheel of kernels.cu, periods 1155, 221, 437, 899), 1024 threads, one CTA
// per SM:
//   W1 one word per lane: 4 LDS.32 + 1 STS.32 per word, indices mod P per word
//   W3 three tables + the primes 29 and 31 by shifts (timing stand-in)
//   W2 two consecutive words per lane: 4 LDS.64 + 1 STS.64 per 2 words
//      (every table stored twice, the second copy shifted by one word, so that
//      the lane's pair is 8-byte aligned in one of them)
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

constexpr uint32_t kWords = 51200;  // 200 KiB: room for the doubled tables
constexpr uint32_t P0 = 1155, P1 = 221, P2 = 437, P3 = 899;
constexpr uint32_t OFF0 = 0, OFF1 = OFF0 + P0 + 64, OFF2 = OFF1 + P1 + 64, OFF3 = OFF2 + P2 + 64, TAB = OFF3 + P3 + 64;

template <uint32_t P>
__device__ __forceinline__ uint32_t step(uint32_t i, uint32_t d) { const uint32_t t = i + d; return t >= P ? t - P : t; }

template <int V>
__global__ void __launch_bounds__(1024, 1) k(const uint32_t *gtab, uint32_t *out, unsigned long long *cyc, int reps, uint32_t x0) {
  extern __shared__ __align__(128) uint32_t sm[];
  uint32_t *seg = sm, *tab = sm + kWords;         // tab: TAB words (+ TAB shifted copy for W2)
  const uint32_t nt = blockDim.x, t = threadIdx.x;
  for (uint32_t i = t; i < (V == 2 ? 2 * TAB : TAB); i += nt) tab[i] = gtab[i % TAB + (i >= TAB)];
  __syncthreads();
  unsigned long long tot = 0;
  for (int rep = 0; rep < reps; ++rep) {
    const long long c0 = clock64();
    if (V == 1) {
      uint32_t i0 = (x0 + t) % P0, i1 = (x0 + t) % P1, i2 = (x0 + t) % P2, i3 = (x0 + t) % P3;
      const uint32_t d0 = nt % P0, d1 = nt % P1, d2 = nt % P2, d3 = nt % P3;
#pragma unroll 4
      for (uint32_t w = t; w < kWords; w += nt) {
        seg[w] = tab[OFF0 + i0] | tab[OFF1 + i1] | tab[OFF2 + i2] | tab[OFF3 + i3];
        i0 = step<P0>(i0, d0); i1 = step<P1>(i1, d1); i2 = step<P2>(i2, d2); i3 = step<P3>(i3, d3);
      }
    } else if (V == 3) {
      // groups 0..2 from the tables, the primes 29 and 31 of group 3 arithmetically: the
      // word's bits for p are (bits 0, p of M_p) << i_p, i_p advancing by a constant mod p
      uint32_t i0 = (x0 + t) % P0, i1 = (x0 + t) % P1, i2 = (x0 + t) % P2;
      uint32_t j29 = (x0 + t) % 29u, j31 = (x0 + t) % 31u;
      const uint32_t d0 = nt % P0, d1 = nt % P1, d2 = nt % P2;
      const uint32_t e29 = 29u - nt % 29u, e31 = 31u - nt % 31u;
#pragma unroll 4
      for (uint32_t w = t; w < kWords; w += nt) {
        seg[w] = tab[OFF0 + i0] | tab[OFF1 + i1] | tab[OFF2 + i2] | (0x20000001u << j29) | (0x80000001u << j31);
        i0 = step<P0>(i0, d0); i1 = step<P1>(i1, d1); i2 = step<P2>(i2, d2);
        j29 = step<29>(j29, e29); j31 = step<31>(j31, e31);
      }
    } else {
      // lane pair of words 2t', 2t'+1 (t' = t): index x = (x0 + 2t) mod P; an odd x reads the
      // shifted copy at x - 1 (8-byte aligned there)
      uint32_t i0 = (x0 + 2 * t) % P0, i1 = (x0 + 2 * t) % P1, i2 = (x0 + 2 * t) % P2, i3 = (x0 + 2 * t) % P3;
      const uint32_t d0 = (2 * nt) % P0, d1 = (2 * nt) % P1, d2 = (2 * nt) % P2, d3 = (2 * nt) % P3;
      const uint2 *t2 = reinterpret_cast<const uint2 *>(tab);
      uint2 *s2 = reinterpret_cast<uint2 *>(seg);
#pragma unroll 4
      for (uint32_t w = t; w < kWords / 2; w += nt) {
        // element index of word x in copy c: c * TAB + x - c (the copy holds word x at x - 1 + TAB)
        const uint2 a = t2[(((OFF0 + i0) & 1) * TAB + OFF0 + i0 - ((OFF0 + i0) & 1)) >> 1];
        const uint2 b = t2[(((OFF1 + i1) & 1) * TAB + OFF1 + i1 - ((OFF1 + i1) & 1)) >> 1];
        const uint2 c = t2[(((OFF2 + i2) & 1) * TAB + OFF2 + i2 - ((OFF2 + i2) & 1)) >> 1];
        const uint2 d = t2[(((OFF3 + i3) & 1) * TAB + OFF3 + i3 - ((OFF3 + i3) & 1)) >> 1];
        s2[w] = make_uint2(a.x | b.x | c.x | d.x, a.y | b.y | c.y | d.y);
        i0 = step<P0>(i0, d0); i1 = step<P1>(i1, d1); i2 = step<P2>(i2, d2); i3 = step<P3>(i3, d3);
      }
    }
    __syncthreads();
    tot += clock64() - c0;
  }
  if (t == 0) atomicAdd(cyc, tot);
  if (blockIdx.x == 0) for (uint32_t w = t; w < kWords; w += nt) out[w] = seg[w];
}

int main() {
  // tables: word x of group g = pseudo-random, extended by 64 words (wrap-free windows)
  std::vector<uint32_t> h(TAB + 1);
  uint32_t offs[4] = {OFF0, OFF1, OFF2, OFF3}, per[4] = {P0, P1, P2, P3};
  uint64_t st = 99;
  for (int g = 0; g < 4; ++g)
    for (uint32_t x = 0; x < per[g]; ++x) {
      st = st * 6364136223846793005ull + 1442695040888963407ull;
      h[offs[g] + x] = (uint32_t)(st >> 40) & (1u << (x % 32));
    }
  for (int g = 0; g < 4; ++g)
    for (uint32_t x = per[g]; x < per[g] + 64; ++x) h[offs[g] + x] = h[offs[g] + x % per[g]];
  h[TAB] = 0;
  // the shifted copy: element TAB + y holds word y + 1 ... built on the device from gtab[i % TAB + 1]
  uint32_t *dt, *dout; unsigned long long *dc;
  cudaMalloc(&dt, (TAB + 1) * 4); cudaMalloc(&dout, kWords * 4); cudaMalloc(&dc, 8);
  cudaMemcpy(dt, h.data(), (TAB + 1) * 4, cudaMemcpyHostToDevice);
  const uint32_t x0 = 12345;
  std::vector<uint32_t> ref(kWords), got(kWords);
  for (uint32_t w = 0; w < kWords; ++w) {
    uint32_t v = 0;
    for (int g = 0; g < 4; ++g) v |= h[offs[g] + (x0 + w) % per[g]];
    ref[w] = v;
  }
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  void (*ks[3])(const uint32_t *, uint32_t *, unsigned long long *, int, uint32_t) = {k<1>, k<2>, k<3>};
  const char *names[3] = {"W1 one word per lane (LDS.32 x4 + STS.32)", "W2 two words per lane (LDS.64 x4 + STS.64)", "W3 three tables + 29, 31 by shifts (LDS.32 x3 + STS.32)"};
  for (int v = 0; v < 3; ++v) {
    const int smem = (kWords + 2 * TAB) * 4;
    cudaFuncSetAttribute(ks[v], cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaMemset(dc, 0, 8);
    ks[v]<<<nsm, 1024, smem>>>(dt, dout, dc, 50, x0);
    cudaError_t e = cudaGetLastError();
    if (!e) e = cudaDeviceSynchronize();
    if (e) { printf("%s\n", cudaGetErrorString(e)); return 1; }
    unsigned long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(got.data(), dout, kWords * 4, cudaMemcpyDeviceToHost);
    printf("{\"variant\": \"%s\", \"cycles_per_32_words\": %.3f, \"segment_cycles\": %.0f, \"ok\": %s}\n", names[v],
           (double)c / nsm / 50 / (kWords / 32), (double)c / nsm / 50,
           v == 2 ? "\"n/a (timing stand-in: 29, 31 not the table pattern)\"" : got == ref ? "true" : "false");
  }
  return 0;
}
