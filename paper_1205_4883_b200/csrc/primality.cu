// primality.cu -- sm_100a kernels for the paper's second algorithm pair
// (SURVEY.md 8(f) F2): Alg. 2 "modulo(a,b,c): exponentiating by squaring to
// (a^b) mod c" and Alg. 3 "Fermat(p, iterations)"
// (PAPER.md:220-234), batched one candidate per thread; plus a deterministic
// Miller-Rabin test (bases 2..37, exact for every 64-bit n), the "improved
// primality test" the paper names, used as an on-GPU
// verifier of sieve outputs.
//
// Modular products: 64 x 64 -> 128-bit, reduced by Montgomery multiplication
// (R = 2^64) for odd moduli -- three 64-bit multiply(-high)s and no division;
// even moduli (only reachable through sieve_modpow, or p = 2) use a 128-bit
// remainder.  Alg. 2's loop is kept exactly: x = 1, y = a; while b > 0:
// if b & 1, x = x y mod c; y = y y mod c; b >>= 1.
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"

namespace sv {
namespace {

struct Mont {
  uint64_t c;     // odd modulus
  uint64_t cinv;  // -c^-1 mod 2^64
  uint64_t r2;    // R^2 mod c (R = 2^64)
};

__device__ __forceinline__ uint64_t mont_reduce(uint64_t lo, uint64_t hi, const Mont &M) {
  // (hi:lo + m c) / 2^64 with m = lo cinv mod 2^64; the sum's low word is 0
  const uint64_t m = lo * M.cinv;
  const uint64_t mclo = m * M.c, mchi = __umul64hi(m, M.c);
  const uint64_t s = lo + mclo;
  const uint64_t carry = s < lo ? 1u : 0u;
  uint64_t u = hi + mchi;
  const bool over = u < hi;  // hi + mchi overflowed 2^64
  u += carry;
  const bool over2 = u < carry;
  // true value is u + 2^64 (over | over2); it is < 2c, so one subtraction
  if (over || over2 || u >= M.c) u -= M.c;
  return u;
}

__device__ __forceinline__ uint64_t mont_mul(uint64_t a, uint64_t b, const Mont &M) {
  return mont_reduce(a * b, __umul64hi(a, b), M);
}

__device__ __forceinline__ Mont mont_setup(uint64_t c) {
  Mont M;
  M.c = c;
  uint64_t x = c;                        // c^-1 mod 2^64 by Newton: 3 -> 6 -> ... -> 96 bits
  for (int i = 0; i < 5; ++i) x *= 2 - c * x;
  M.cinv = 0 - x;
  // R mod c = (2^64 - c) mod c; R^2 mod c by 64 doublings of R mod c
  const uint64_t r1 = (0 - c) % c;
  uint64_t r = r1;
  for (int i = 0; i < 64; ++i) {
    const uint64_t t = r << 1;
    r = (t < r || t >= c) ? t - c : t;   // 2r mod c (r < c < 2^64)
  }
  M.r2 = r;
  return M;
}

__device__ __forceinline__ uint64_t to_mont(uint64_t a, const Mont &M) { return mont_mul(a % M.c, M.r2, M); }
__device__ __forceinline__ uint64_t from_mont(uint64_t a, const Mont &M) { return mont_reduce(a, 0, M); }

// 128-bit remainder for even moduli (a b) mod c
__device__ __forceinline__ uint64_t mulmod_wide(uint64_t a, uint64_t b, uint64_t c) {
  const unsigned __int128 t = (unsigned __int128)a * b;
  return (uint64_t)(t % c);
}

// Alg. 2 with Montgomery products (odd c >= 3)
__device__ uint64_t modpow_odd(uint64_t a, uint64_t b, const Mont &M) {
  uint64_t x = to_mont(1, M), y = to_mont(a, M);
  while (b > 0) {
    if (b & 1u) x = mont_mul(x, y, M);
    y = mont_mul(y, y, M);
    b >>= 1;
  }
  return from_mont(x, M);
}

// Alg. 2 for any c >= 1
__device__ uint64_t modpow_any(uint64_t a, uint64_t b, uint64_t c) {
  if (c == 1) return 0;
  if (c & 1u) return modpow_odd(a, b, mont_setup(c));
  uint64_t x = 1, y = a % c;
  while (b > 0) {
    if (b & 1u) x = mulmod_wide(x, y, c);
    y = mulmod_wide(y, y, c);
    b >>= 1;
  }
  return x % c;
}

__global__ void k_modpow(const uint64_t *__restrict__ a, const uint64_t *__restrict__ b,
                         const uint64_t *__restrict__ c, uint64_t n, uint64_t *__restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = c[i] == 0 ? ~0ull : modpow_any(a[i], b[i], c[i]);
}

// Alg. 3: Fermat(p, iterations); the t-th base is draws[i it + t] mod (p-1) + 1
__global__ void k_fermat(const uint64_t *__restrict__ p, uint64_t n, const uint64_t *__restrict__ draws,
                         uint32_t iters, uint8_t *__restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t q = p[i];
    uint8_t verdict = 1;
    if (q <= 1) {
      verdict = 0;  // p = 1: Alg. 3's guard; p = 0: domain error, reported as false
    } else if (q & 1u) {
      const Mont M = mont_setup(q);
      const uint64_t one = to_mont(1, M);
      for (uint32_t t = 0; t < iters; ++t) {
        const uint64_t a = draws[i * iters + t] % (q - 1) + 1;
        // modulo(a, p-1, p) != 1 ?  (compared in Montgomery form)
        uint64_t x = one, y = to_mont(a, M), e = q - 1;
        while (e > 0) {
          if (e & 1u) x = mont_mul(x, y, M);
          y = mont_mul(y, y, M);
          e >>= 1;
        }
        if (x != one) { verdict = 0; break; }
      }
    } else {
      for (uint32_t t = 0; t < iters; ++t) {
        const uint64_t a = draws[i * iters + t] % (q - 1) + 1;
        if (modpow_any(a, q - 1, q) != 1) { verdict = 0; break; }
      }
    }
    out[i] = verdict;
  }
}

// deterministic Miller-Rabin: the first 12 primes as bases decide every n < 3.3e24
__global__ void k_is_prime(const uint64_t *__restrict__ nums, uint64_t n, uint8_t *__restrict__ out) {
  const uint32_t bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = nums[i];
    uint8_t verdict = 1;
    if (v < 2) {
      verdict = 0;
    } else {
      bool decided = false;
      for (int k = 0; k < 12; ++k) {
        if (v == bases[k]) { decided = true; break; }
        if (v % bases[k] == 0) { verdict = 0; decided = true; break; }
      }
      if (!decided) {
        uint64_t d = v - 1;
        int s = 0;
        while (!(d & 1u)) { d >>= 1; ++s; }
        const Mont M = mont_setup(v);
        const uint64_t one = to_mont(1, M), minus1 = to_mont(v - 1, M);
        for (int k = 0; k < 12 && verdict; ++k) {
          uint64_t x = one, y = to_mont(bases[k], M), e = d;
          while (e > 0) {
            if (e & 1u) x = mont_mul(x, y, M);
            y = mont_mul(y, y, M);
            e >>= 1;
          }
          if (x == one || x == minus1) continue;
          bool witness = true;
          for (int r = 1; r < s; ++r) {
            x = mont_mul(x, x, M);
            if (x == minus1) { witness = false; break; }
          }
          if (witness) verdict = 0;
        }
      }
    }
    out[i] = verdict;
  }
}

int grid_of(uint64_t n) {
  const uint64_t b = (n + 255) / 256;
  return (int)(b < 148 * 16 ? (b ? b : 1) : 148 * 16);
}

}  // namespace

cudaError_t launch_modpow(const uint64_t *a, const uint64_t *b, const uint64_t *c, uint64_t n,
                          uint64_t *out, cudaStream_t s) {
  k_modpow<<<grid_of(n), 256, 0, s>>>(a, b, c, n, out);
  return cudaGetLastError();
}

cudaError_t launch_fermat(const uint64_t *p, uint64_t n, const uint64_t *draws, uint32_t iters,
                          uint8_t *out, cudaStream_t s) {
  k_fermat<<<grid_of(n), 256, 0, s>>>(p, n, draws, iters, out);
  return cudaGetLastError();
}

cudaError_t launch_is_prime(const uint64_t *nums, uint64_t n, uint8_t *out, cudaStream_t s) {
  k_is_prime<<<grid_of(n), 256, 0, s>>>(nums, n, out);
  return cudaGetLastError();
}

}  // namespace sv
