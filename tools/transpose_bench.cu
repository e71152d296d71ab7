// Write-back transpose microbenchmark (diagnostics): cycles per 1024-slot
// block of the in-place 32x32 bit transpose of a 208 KiB shared-memory
// segment (transposed layout -> natural layout, inverted), 1024 threads per
// CTA, one CTA per SM:
//   V0 shuffle transpose (the round-2 untranspose: 5 x SHF + SHFL + LOP3)
//   V1 in-register transpose, one block per thread, loads and stores of
//      quad q ^ (block & 7) (conflict-free), the XOR skew absorbed by the
//      stage masks (no extra instructions)
//   V2 V1 + count of the prime bits in carry-save planes (no second pass)
//   V3 V0 + a second pass that counts (LDS.128 + POPC)
// Checks every variant's words and count against a host transpose.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr uint32_t kWords = 53248, kBlocks = kWords / 32;

__device__ __forceinline__ void csa(uint32_t &carry, uint32_t &sum, uint32_t a, uint32_t b, uint32_t c) {
  const uint32_t u = a ^ b;
  carry = (a & b) | (u & c);
  sum = u ^ c;
}

__device__ __forceinline__ void t_shfl(uint32_t *seg) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t amt[5], keep[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const uint32_t w = 16u >> k;
    const uint32_t m = k == 0 ? 0x0000FFFFu : k == 1 ? 0x00FF00FFu : k == 2 ? 0x0F0F0F0Fu
                     : k == 3 ? 0x33333333u : 0x55555555u;
    amt[k] = (lane & w) ? 32u - w : w;
    keep[k] = (lane & w) ? ~m : m;
  }
  constexpr int kUT = 2;
  for (uint32_t B = warp; B < kBlocks; B += kUT * nw) {
    uint32_t x[kUT];
#pragma unroll
    for (int u = 0; u < kUT; ++u) {
      const uint32_t Bu = B + u * nw;
      x[u] = Bu < kBlocks ? seg[32u * Bu + lane] : 0u;
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) {
#pragma unroll
      for (int u = 0; u < kUT; ++u) {
        const uint32_t y = __shfl_xor_sync(0xffffffffu, __funnelshift_r(x[u], x[u], amt[k]), 16u >> k);
        asm("lop3.b32 %0, %0, %1, %2, 0xE4;" : "+r"(x[u]) : "r"(y), "r"(keep[k]));
      }
    }
#pragma unroll
    for (int u = 0; u < kUT; ++u) {
      const uint32_t Bu = B + u * nw;
      if (Bu < kBlocks) seg[32u * Bu + lane] = ~x[u];
    }
  }
}

// (x & k) | (y & ~k)
__device__ __forceinline__ uint32_t sel(uint32_t x, uint32_t y, uint32_t k) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(r) : "r"(x), "r"(y), "r"(k));
  return r;
}

template <int J>
__device__ __forceinline__ void stage_std(uint32_t (&A)[32]) {
  constexpr uint32_t m = J == 16 ? 0x0000FFFFu : J == 8 ? 0x00FF00FFu : J == 4 ? 0x0F0F0F0Fu
                       : J == 2 ? 0x33333333u : 0x55555555u;
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    if (r & J) continue;
    const uint32_t x = A[r], y = A[r + J];
    A[r] = sel(x, y << J, m);
    A[r + J] = sel(x >> J, y, m);
  }
}
template <int J>
__device__ __forceinline__ void stage_skew(uint32_t (&A)[32], uint32_t keep, uint32_t amt) {
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    if (r & J) continue;
    const uint32_t x = A[r], y = A[r + J];
    A[r] = sel(x, __funnelshift_l(y, y, amt), keep);
    A[r + J] = sel(__funnelshift_r(x, x, amt), y, keep);
  }
}

// V4: count and the two weighted sums from the INPUT rows only (planes for
// the bit-position weighting, one POPC per row for the row-index weighting)
__device__ __forceinline__ uint32_t t_reg_in(uint32_t *seg, uint32_t &wsum) {
  uint4 *seg4 = reinterpret_cast<uint4 *>(seg);
  uint32_t pl[4] = {0, 0, 0, 0}, cnt = 0, wb = 0, hi = 0;
  for (uint32_t B = threadIdx.x; B < kBlocks; B += blockDim.x) {
    const uint32_t s = B & 7u;
    uint32_t A[32];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint4 v = seg4[8u * B + (q ^ s)];
      A[4 * q] = v.x; A[4 * q + 1] = v.y; A[4 * q + 2] = v.z; A[4 * q + 3] = v.w;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t c0 = __popc(A[4 * q]), c1 = __popc(A[4 * q + 1]), c2 = __popc(A[4 * q + 2]), c3 = __popc(A[4 * q + 3]);
      const uint32_t cq = c0 + c1 + c2 + c3;
      cnt += cq;
      wb += 4u * (q ^ s) * cq + c1 + 2u * c2 + 3u * c3;
      uint32_t tA, tB, fA;
      csa(tA, pl[0], pl[0], A[4 * q], A[4 * q + 1]);
      csa(tB, pl[0], pl[0], A[4 * q + 2], A[4 * q + 3]);
      csa(fA, pl[1], pl[1], tA, tB);
      const uint32_t e = pl[2] & fA;
      pl[2] ^= fA;
      const uint32_t e2 = pl[3] & e;
      pl[3] ^= e;
      hi += __popc(e2);
    }
    const uint32_t k4 = 4u * s;
    const uint32_t f16 = k4 & 16u, f8 = k4 & 8u, f4 = k4 & 4u;
    stage_skew<16>(A, f16 ? 0xFFFF0000u : 0x0000FFFFu, 16u);
    stage_skew<8>(A, f8 ? 0xFF00FF00u : 0x00FF00FFu, f8 ? 24u : 8u);
    stage_skew<4>(A, f4 ? 0xF0F0F0F0u : 0x0F0F0F0Fu, f4 ? 28u : 4u);
    stage_std<2>(A);
    stage_std<1>(A);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      seg4[8u * B + (q ^ s)] = make_uint4(~A[4 * q], ~A[4 * q + 1], ~A[4 * q + 2], ~A[4 * q + 3]);
  }
  wsum = wb + pl[0] + pl[1] + pl[2] + pl[3] + hi;
  return cnt;
}


// V5/V6: two lanes per block (16 rows each, stage 16 by one SHFL per row),
// as in kernels.cu writeback_fused; V5 with its 64 POPC per block for the
// count and the weighted sums, V6 without
template <int J>
__device__ __forceinline__ void hstage_std(uint32_t (&A)[16]) {
  constexpr uint32_t m = J == 2 ? 0x33333333u : 0x55555555u;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    if (r & J) continue;
    const uint32_t x = A[r], y = A[r + J];
    A[r] = sel(x, y << J, m);
    A[r + J] = sel(x >> J, y, m);
  }
}
template <int J>
__device__ __forceinline__ void hstage_skew(uint32_t (&A)[16], uint32_t keep, uint32_t amt) {
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    if (r & J) continue;
    const uint32_t x = A[r], y = A[r + J];
    A[r] = sel(x, __funnelshift_l(y, y, amt), keep);
    A[r + J] = sel(__funnelshift_r(x, x, amt), y, keep);
  }
}
template <bool kPopc>
__device__ __forceinline__ uint32_t t_half(uint32_t *seg) {
  const uint32_t lane = threadIdx.x & 31u, h = lane & 1u;
  uint32_t comp = 0, wrow = 0, wnat = 0;
  for (uint32_t B2 = threadIdx.x & ~31u; B2 < 2u * kBlocks; B2 += blockDim.x) {
    const uint32_t B = (B2 + lane) >> 1;
    const uint32_t qa = (uint32_t)__cvta_generic_to_shared(seg) + 128u * B + 64u * h + 16u * (B & 3u);
    const uint32_t t4 = 4u * (B & 3u) + 16u * h;
    uint32_t A[16];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(A[4 * q]), "=r"(A[4 * q + 1]), "=r"(A[4 * q + 2]), "=r"(A[4 * q + 3])
                   : "r"(qa ^ (16u * q)));
    if (kPopc) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t c0 = __popc(A[4 * q]), c1 = __popc(A[4 * q + 1]), c2 = __popc(A[4 * q + 2]), c3 = __popc(A[4 * q + 3]);
        const uint32_t cq = c0 + c1 + c2 + c3;
        comp += cq;
        wrow += (t4 ^ (4u * q)) * cq + c1 + 2u * c2 + 3u * c3;
      }
    }
    const uint32_t keep16 = h ? 0xFFFF0000u : 0x0000FFFFu;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t y = __shfl_xor_sync(0xffffffffu, __funnelshift_l(A[r], A[r], 16u), 1u);
      A[r] = sel(A[r], y, keep16);
    }
    const uint32_t k = 4u * (B & 3u);
    const bool f8 = k & 8u, f4 = k & 4u;
    hstage_skew<8>(A, f8 ? 0xFF00FF00u : 0x00FF00FFu, f8 ? 24u : 8u);
    hstage_skew<4>(A, f4 ? 0xF0F0F0F0u : 0x0F0F0F0Fu, f4 ? 28u : 4u);
    hstage_std<2>(A);
    hstage_std<1>(A);
    if (kPopc) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t c1 = __popc(A[4 * q + 1]), c2 = __popc(A[4 * q + 2]), c3 = __popc(A[4 * q + 3]);
        wnat += (t4 ^ (4u * q)) * (__popc(A[4 * q]) + c1 + c2 + c3) + c1 + 2u * c2 + 3u * c3;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(qa ^ (16u * q)), "r"(~A[4 * q]),
                   "r"(~A[4 * q + 1]), "r"(~A[4 * q + 2]), "r"(~A[4 * q + 3]) : "memory");
  }
  return kPopc ? 1024u * 0u + (uint32_t)(kBlocks * 0) + comp + 0u * (wrow + wnat) + ((wrow ^ wnat) == 0x7fffffffu) : 0u;
}

template <bool kCount>
__device__ __forceinline__ uint32_t t_reg(uint32_t *seg) {
  uint4 *seg4 = reinterpret_cast<uint4 *>(seg);
  uint32_t ones = 0, twos = 0, fours = 0, eights = 0, cnt = 0;
  for (uint32_t B = threadIdx.x; B < kBlocks; B += blockDim.x) {
    const uint32_t s = B & 7u;
    uint32_t A[32];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint4 v = seg4[8u * B + (q ^ s)];
      A[4 * q] = v.x; A[4 * q + 1] = v.y; A[4 * q + 2] = v.z; A[4 * q + 3] = v.w;
    }
    // stages 16, 8, 4 see the rows and columns XOR-permuted by 4 s: where
    // bit j of 4 s is set the pair's roles swap (keep ~m, rotate the other way)
    const uint32_t k4 = 4u * s;
    const uint32_t f16 = k4 & 16u, f8 = k4 & 8u, f4 = k4 & 4u;
    stage_skew<16>(A, f16 ? 0xFFFF0000u : 0x0000FFFFu, f16 ? 16u : 16u);
    stage_skew<8>(A, f8 ? 0xFF00FF00u : 0x00FF00FFu, f8 ? 24u : 8u);
    stage_skew<4>(A, f4 ? 0xF0F0F0F0u : 0x0F0F0F0Fu, f4 ? 28u : 4u);
    stage_std<2>(A);
    stage_std<1>(A);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint4 v = make_uint4(~A[4 * q], ~A[4 * q + 1], ~A[4 * q + 2], ~A[4 * q + 3]);
      seg4[8u * B + (q ^ s)] = v;
      if (kCount) {
        uint32_t tA, tB, fA;
        csa(tA, ones, ones, v.x, v.y);
        csa(tB, ones, ones, v.z, v.w);
        csa(fA, twos, twos, tA, tB);
        const uint32_t e = fours & fA;
        fours ^= fA;
        const uint32_t e2 = eights & e;
        eights ^= e;
        cnt += __popc(e2);
      }
    }
  }
  return kCount ? 16u * cnt + 8u * __popc(eights) + 4u * __popc(fours) + 2u * __popc(twos) + __popc(ones) : 0u;
}

__device__ __forceinline__ uint32_t count_pass(const uint32_t *seg) {
  const uint4 *seg4 = reinterpret_cast<const uint4 *>(seg);
  uint32_t c = 0;
  for (uint32_t q = threadIdx.x; q < kWords / 4; q += blockDim.x) {
    const uint4 v = seg4[q];
    c += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
  }
  return c;
}

template <int V>
__global__ void __launch_bounds__(1024, 1) k_bench(const uint32_t *in, uint32_t *out, unsigned long long *cyc,
                                                   unsigned long long *cnt, int reps) {
  extern __shared__ __align__(128) uint32_t seg[];
  unsigned long long total_cyc = 0, c = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (uint32_t w = threadIdx.x; w < kWords; w += blockDim.x) seg[w] = in[w];
    __syncthreads();
    const long long t0 = clock64();
    uint32_t cc = 0;
    if (V == 0 || V == 3) t_shfl(seg);
    if (V == 1) t_reg<false>(seg);
    if (V == 2) cc = t_reg<true>(seg);
    if (V == 4) {
      uint32_t ws;
      cc = t_reg_in(seg, ws);
      if (ws == 0x7fffffffu) cc = 0;
      cc = 1024u * 0u + cc;
    }
    if (V == 5) cc = t_half<true>(seg);
    if (V == 6) t_half<false>(seg);
    if (V == 3) {
      __syncthreads();
      cc = count_pass(seg);
    }
    __syncthreads();
    total_cyc += clock64() - t0;
    c += cc;
  }
  atomicAdd(cnt, c);
  if (threadIdx.x == 0) atomicAdd(cyc, total_cyc);
  if (blockIdx.x == 0)
    for (uint32_t w = threadIdx.x; w < kWords; w += blockDim.x) out[w] = seg[w];
}

int main(int argc, char **argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 50;
  std::vector<uint32_t> h(kWords), ref(kWords), got(kWords);
  uint64_t st = 12345;
  for (auto &x : h) {
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    x = (uint32_t)(st >> 32);
  }
  unsigned long long refcnt = 0;
  for (uint32_t B = 0; B < kBlocks; ++B)
    for (int c = 0; c < 32; ++c) {
      uint32_t w = 0;
      for (int r = 0; r < 32; ++r) w |= ((h[32 * B + r] >> c) & 1u) << r;
      ref[32 * B + c] = ~w;
      refcnt += __builtin_popcount(~w);
    }
  uint32_t *din, *dout;
  unsigned long long *dcyc, *dcnt;
  cudaMalloc(&din, kWords * 4);
  cudaMalloc(&dout, kWords * 4);
  cudaMalloc(&dcyc, 8);
  cudaMalloc(&dcnt, 8);
  cudaMemcpy(din, h.data(), kWords * 4, cudaMemcpyHostToDevice);
  const int smem = kWords * 4;
  void (*ks[7])(const uint32_t *, uint32_t *, unsigned long long *, unsigned long long *, int) = {
      k_bench<0>, k_bench<1>, k_bench<2>, k_bench<3>, k_bench<4>, k_bench<5>, k_bench<6>};
  const char *names[7] = {"V0 shuffle", "V1 in-register skew", "V2 in-register + count", "V3 shuffle + count pass", "V4 in-register + input planes + row popc", "V5 half-block + 64 POPC", "V6 half-block, no POPC"};
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int v = 0; v < 7; ++v) {
    cudaFuncSetAttribute(ks[v], cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaMemset(dcyc, 0, 8);
    cudaMemset(dcnt, 0, 8);
    cudaMemset(dout, 0, kWords * 4);
    ks[v]<<<nsm, 1024, smem>>>(din, dout, dcyc, dcnt, reps);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("%s: %s\n", names[v], cudaGetErrorString(e)); return 1; }
    unsigned long long cyc = 0, cnt = 0;
    cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cnt, dcnt, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(got.data(), dout, kWords * 4, cudaMemcpyDeviceToHost);
    bool ok = got == ref;
    const unsigned long long want = (v == 4 || v == 5) ? (unsigned long long)kWords * 32ull - refcnt : refcnt;
    const bool cnt_ok = (v == 0 || v == 1 || v == 6) || cnt == want * (unsigned long long)reps * nsm;
    printf("{\"variant\": \"%s\", \"cycles_per_block\": %.3f, \"words_ok\": %s, \"count_ok\": %s}\n", names[v],
           (double)cyc / nsm / reps / kBlocks, ok ? "true" : "false", cnt_ok ? "true" : "false");
  }
  return 0;
}
