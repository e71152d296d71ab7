// kernels.cu -- the sm_100a kernels of the segmented sieve of Eratosthenes.
//
// Steps:
//   A2  k_base_primes : odd primes <= r (sliced over CTAs, decoupled look-back),
//                       or base_phase inside the sieve launch (fused A2)
//   A3  wheel init    : segment <- OR of periodic composite patterns of 3..w
//   A4  marking       : shared-memory atomicOr of the odd multiples of each
//                       base prime w < p <= r, starting at max(p^2, first
//                       odd multiple >= segment start)  (PAPER.md:131,
//                       "iteratively marking as composite the multiples of
//                       each prime"; SPEC.md:158 start rule), conflict-free
//                       in the bank-transposed segment layout (internal.h)
//   A5  large primes  : primes with < kWarpHits hits per segment are marked
//                       lane-per-prime straight from their first hit, so a
//                       segment a prime skips costs one Barrett reduction
//   A6  count + sum   : popc of the inverted words, weighted popcs for the sum
//   A7  bitmap        : writeback_fused: in-register transpose of each block,
//                       count/sum from registers, prime words back to shared
//                       memory, one TMA bulk copy per warp to HBM
//   A8  list          : per-segment counts -> scan -> ballot/scan compaction
//   A10 batch         : the same segment kernel over (interval, segment) items
//
// Bit j of a call's odd-only grid <-> the odd integer o0 + 2j (o0 = lo|1).
// In shared memory a set bit means "composite" (the paper's marking); the
// write-back inverts it so that the bitmap has 1 = prime (reading R5), and
// transposes each 1024-slot block back to the natural bit order.
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "internal.h"
#include "peer.cuh"

namespace sv {

constexpr uint32_t kNone = 0xFFFFFFFFu;

// ---------------------------------------------------------------------------
// Bounds-check build (internal.h SIEVE_CHECK_BOUNDS): violations are counted
// per class, never trapped; the product build compiles every check out.
// ---------------------------------------------------------------------------
__device__ unsigned long long g_violations[kVioClasses];
#if SIEVE_CHECK_BOUNDS
// the CTA's segment words in the shared window: [s_chk_lo, s_chk_hi) bytes
__shared__ uint32_t s_chk_lo, s_chk_hi;
#define SV_CHECK(cond, cls)                                             \
  do {                                                                  \
    if (!(cond)) atomicAdd(&g_violations[cls], 1ull);                   \
  } while (0)
#else
#define SV_CHECK(cond, cls) \
  do {                      \
  } while (0)
#endif

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
// Offset (in odd slots from a) of the first odd multiple m of p with
// m >= max(a, p*p); kNone when p*p >= seg_end.  a is odd, m = a + 2*j.
// a mod p by Barrett reduction with recip = floor((2^64-1)/p): the quotient
// estimate is floor(a/p) or one less, so one conditional subtraction is exact
// for any a < 2^64.
// Branch-free, so that the loads of p and recip issue together (an early
// return on p^2 would make the recip load wait for the p load).
__device__ __forceinline__ uint32_t first_hit(uint64_t a, uint64_t seg_end, uint32_t p,
                                              uint64_t recip) {
  const uint64_t pp = (uint64_t)p * p;
  const uint64_t q = __umul64hi(a, recip);
  uint32_t r = (uint32_t)(a - q * (uint64_t)p);
  r = min(r, r - p);              // r in [0, 2p) -> [0, p)
  uint32_t d = r ? p - r : 0u;    // a + d == 0 (mod p)
  d += (d & 1u) ? p : 0u;         // a odd: the odd multiple is a + d with d even
  uint32_t j = d >> 1;
  j = (a + 2ull * j < pp) ? (uint32_t)((pp - a) >> 1) : j;
  return pp >= seg_end ? kNone : j;
}

// first_hit when p^2 <= a (the segment lies above p^2): the first odd multiple
// a + 2 j of p, r = a mod p by the same Barrett step, j = (((r & 1) ? p : 2 p)
// - r) / 2 mod p (a odd: r odd leaves p - r even).  No clamp, no 64-bit compare.
__device__ __forceinline__ uint32_t first_hit_above(uint64_t a, uint32_t p, uint64_t recip) {
  uint32_t r = (uint32_t)a - (uint32_t)__umul64hi(a, recip) * p;
  r = min(r, r - p);  // a mod p
  const uint32_t j = (((r & 1u) ? p : 2u * p) - r) >> 1;
  return min(j, j - p);  // r = 0: j = p -> 0
}

// first_hit_above with one 32-bit multiply-high instead of the 64 x 64 one,
// for a < 2^(32+t) and p > 2^t (t uniform, sh = 32 - t, a_sh = a >> t,
// na_lo = -a mod 2^32): M = recip >> sh = floor(2^(32+t)/p) < 2^32 (recip =
// floor(2^64/p) for odd p, and floors nest), q = hi32(a_sh M) is floor(a/p)
// less 0, 1 or 2 (each truncation costs under one unit), so d = (q + 3) p - a
// is -a mod p plus 0, p or 2 p, in (0, 3p] (p < 2^30: no wrap).  The odd
// multiple a + 2 j' with 2 j' = d or d + p (whichever is even) has j' in
// (0, 2p]; two conditional subtractions give j in [0, p).
__device__ __forceinline__ uint32_t first_hit_scaled(uint32_t a_sh, uint32_t na_lo, uint32_t sh,
                                                     uint32_t p, uint64_t recip) {
  const uint32_t M = __funnelshift_rc((uint32_t)recip, (uint32_t)(recip >> 32), sh);
  const uint32_t d = (__umulhi(a_sh, M) + 3u) * p + na_lo;
  uint32_t j2;  // d + (d & 1) p as one lop3 + one imad (a select costs two more)
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(j2) : "r"(d & 1u), "r"(p), "r"(d));
  uint32_t j = j2 >> 1;
  j = min(j, j - p);
  return min(j, j - p);
}

// first_hit_scaled with M = floor(2^(32+t)/p) given (the packed plain-pass
// table holds floor(2^44/p); M = that >> (12 - t) for t <= 12).
__device__ __forceinline__ uint32_t first_hit_m(uint32_t a_sh, uint32_t na_lo, uint32_t p, uint32_t M) {
  const uint32_t d = (__umulhi(a_sh, M) + 3u) * p + na_lo;
  uint32_t j2;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(j2) : "r"(d & 1u), "r"(p), "r"(d));
  uint32_t j = j2 >> 1;
  j = min(j, j - p);
  return min(j, j - p);
}

// floor((2^64-1)/p) for an odd p >= 3, without a 64-bit integer division:
// a double quotient (within 2^12 of the result), then the exact remainder
// T = (2^64-1) - q p (|T| < 2^40, so mod-2^64 arithmetic gives it as a signed
// number) corrects q by floor(T / p), with a final +-1 guard on the rounding.
__device__ __forceinline__ uint64_t recip_of(uint32_t p) {
  // floor((2^64 - 1) / p), p >= 3: a double estimate q (within ~2^12 of the
  // quotient: one reciprocal, no division), then exact integer correction
  // of the remainder T = (2^64 - 1) - q p (|T| < 2^45: read as signed)
  const double r = __drcp_rn((double)p);
  uint64_t q = __double2ull_rz(1.8446744073709552e19 * r);
  int64_t T = (int64_t)(~0ull - q * (uint64_t)p);
  const int64_t d = (int64_t)floor((double)T * r);
  q += (uint64_t)d;
  T -= d * (int64_t)p;
  while (T < 0) { --q; T += p; }
  while (T >= (int64_t)p) { ++q; T -= p; }
  return q;
}

__device__ __forceinline__ uint32_t upper_bound_u32(const uint32_t *v, uint32_t n, uint64_t x) {
  uint32_t lo = 0, hi = n;  // first index with v[idx] > x
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if ((uint64_t)__ldg(v + mid) <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// sum of the bit indices of the set bits of w
__device__ __forceinline__ uint32_t bit_index_sum(uint32_t w) {
  return __popc(w & 0xAAAAAAAAu) + 2u * __popc(w & 0xCCCCCCCCu) + 4u * __popc(w & 0xF0F0F0F0u) +
         8u * __popc(w & 0xFF00FF00u) + 16u * __popc(w & 0xFFFF0000u);
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// Segment phases.  The segment is held in the bank-transposed layout of
// internal.h: slot j <-> word 32 (j >> 10) + (j & 31), bit (j >> 5) & 31.
// ---------------------------------------------------------------------------

// shared-memory OR without return (ATOMS.OR RZ) at a 32-bit shared-window
// byte address: the segment base is 128-byte aligned and kept in a register,
// so that the address arithmetic below needs no generic->shared conversion
__device__ __forceinline__ void red_or(uint32_t saddr, uint32_t mask) {
#if SIEVE_CHECK_BOUNDS
  SV_CHECK(saddr >= s_chk_lo && saddr < s_chk_hi && __popc(mask) == 1, kVioSmemMark);
#endif
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(saddr), "r"(mask) : "memory");
}

// byte address (shared window) and bit mask of slot j in the transposed
// segment from J = 4 j + 32 sb: (J >> 5) & ~127 | J & 127 as ONE lop3, and
// 1 << ((J >> 7) & 31)
__device__ __forceinline__ uint32_t j_addr(uint32_t J) {
  uint32_t d;
  asm("lop3.b32 %0, %1, 127, %2, 0xB8;" : "=r"(d) : "r"(J >> 5), "r"(J));  // (a & ~b) | (c & b)
  return d;
}
__device__ __forceinline__ uint32_t j_mask(uint32_t J) { return __funnelshift_l(0u, 1u, J >> 7); }

// byte offset and bit mask of slot j in the transposed segment
__device__ __forceinline__ uint32_t t_addr(uint32_t j) {
  return ((j >> 3) & ~127u) | ((j & 31u) << 2);
}
__device__ __forceinline__ uint32_t t_mask(uint32_t j) { return __funnelshift_l(0u, 1u, j >> 5); }
__device__ __forceinline__ uint32_t rotl(uint32_t x, uint32_t s) { return __funnelshift_l(x, x, s); }

// A3: wheel pre-sieve of one segment into seg (composite = 1), plus the
// fix-ups (1 is not prime; wheel primes in range are prime) and the tail
// (slots >= valid are set composite).  Thread t builds words t, t+nt, ...;
// word T (bank b = T & 31, block B = T >> 5) of group g is the table word
// TT_g[(X0 + 1024 B + b) mod P_g]: the 32 lanes of a warp read 32 consecutive
// table words (conflict-free), and the index of a thread advances by
// 32 nt (mod P_g) per word.  Whole 1024-slot blocks are written, so that the
// epilogue can read whole blocks.
template <int G>
struct WheelGroup {
  static constexpr uint32_t P = group_period(G);
  static constexpr uint32_t OFF = group_offset(G);
};

// OR the table words of groups G..NG-1 for the current segment word and
// advance their indices (compile-time recursion: constant moduli).  Indices
// are byte offsets ig = 4 y; the step d4 = 4 (32 nt mod P) is applied mod 4P
// as ig' = umin(ig + d4, ig - e4), e4 = 4P - d4 (ig - e4 wraps above every
// valid offset when ig < e4): one add and one add+min per group and word.
template <int G, int NG>
__device__ __forceinline__ uint32_t wheel_word(const char *tabb, uint32_t (&ig)[NG],
                                               const uint32_t (&d4)[NG], const uint32_t (&e4)[NG]) {
  if constexpr (G == NG) {
    return 0u;
  } else {
    const uint32_t v = *reinterpret_cast<const uint32_t *>(tabb + 4u * WheelGroup<G>::OFF + ig[G]);
#if SIEVE_WHEEL_DIAG == 1  // diagnostics build only: no index update (wrong pattern, in bounds)
    (void)d4; (void)e4;
#else
    const uint32_t t = ig[G] - e4[G];
    ig[G] = min(ig[G] + d4[G], t);
#endif
    return v | wheel_word<G + 1, NG>(tabb, ig, d4, e4);
  }
}

template <int G, int NG>
__device__ __forceinline__ void wheel_setup(uint32_t (&ig)[NG], uint32_t (&d4)[NG], uint32_t (&e4)[NG],
                                            uint64_t X0, uint32_t tid, uint32_t nt) {
  if constexpr (G < NG) {
    constexpr uint32_t P = WheelGroup<G>::P;
    ig[G] = 4u * (uint32_t)((X0 % P + 1024u * (tid >> 5) + (tid & 31u)) % P);
    d4[G] = 4u * ((32u * nt) % P);
    e4[G] = 4u * P - d4[G];
    wheel_setup<G + 1, NG>(ig, d4, e4, X0, tid, nt);
  }
}

// (count mode unrolls the word loop: SIEVE_WHEEL_UNROLL, same-box A/B)
constexpr int kWheelUnroll = SIEVE_WHEEL_UNROLL;
template <int NG, int UNR = 1>
__device__ __forceinline__ void wheel_init(uint32_t *seg, const uint32_t *tab, uint64_t o0,
                                           uint64_t bit0, uint32_t valid, uint64_t a) {
  const uint32_t nt = blockDim.x, tid = threadIdx.x;
  const uint32_t nwords = ((valid + 1023u) >> 10) << 5;
  uint32_t ig[NG], d4[NG], e4[NG];
  wheel_setup<0, NG>(ig, d4, e4, ((o0 - 1) >> 1) + bit0, tid, nt);
  const char *tabb = reinterpret_cast<const char *>(tab);
  // fast path: words of whole blocks with no fix-up (block 0 holds the
  // integers <= w when a <= w) and no tail slot
  const uint32_t wfast_lo = a <= wheel_bound(NG) ? 32u : 0u;
  const uint32_t wfast_hi = (valid >> 10) << 5;
  uint32_t w = tid;
  if (wfast_lo == 0) {
#pragma unroll UNR
    for (; w < wfast_hi; w += nt) {
      SV_CHECK(4u * w + (uint32_t)__cvta_generic_to_shared(seg) < s_chk_hi, kVioScratch);
      seg[w] = wheel_word<0, NG>(tabb, ig, d4, e4);
    }
  }
  for (; w < nwords; w += nt) {
    uint32_t v = wheel_word<0, NG>(tabb, ig, d4, e4);
    const uint32_t b = w & 31u, j0 = ((w >> 5) << 10) + b;  // slot of the word's bit 0
    if (w < 32u) {  // bit 0 <-> n = a + 2b (a <= w: n <= 2w+63, bits >= 1 are > w)
      const uint64_t n = a + 2ull * b;
      if (n == 1u) v |= 1u;  // 1 is not prime (reading R2)
      else if (n < 64 && ((kOddPrimesBelow64 >> n) & 1ull) && n <= wheel_bound(NG)) v &= ~1u;
    }
    // valid bits i: j0 + 32 i < valid
    const int k = j0 < valid ? (int)((valid - j0 + 31u) >> 5) : 0;
    if (k < 32) v = k <= 0 ? 0xFFFFFFFFu : (v | (0xFFFFFFFFu << k));
    SV_CHECK(4u * w + (uint32_t)__cvta_generic_to_shared(seg) < s_chk_hi, kVioScratch);
    seg[w] = v;
  }
}

struct PrimeRegions {
  uint32_t start;  // first marking prime (after the wheel primes)
  uint32_t unit;   // first prime with fewer than kUnitHits hits per full segment
  uint32_t cls;    // first prime with fewer than kClassHits hits per full segment
  uint32_t warp;   // first prime with fewer than kWarpHits hits per full segment
  uint32_t few;    // first prime with fewer than kC15Hits hits per full segment
  uint32_t two;    // first prime with at most 2 hits in any segment (p > S / 2)
  uint32_t big;    // first bucket prime (fewer than kBucketHits hits; = end without buckets)
  uint32_t end;    // first prime > r
};

// Multiples of 3 are composite from the wheel (every wheel includes 3), so a
// prime p's hit n = p m with 3 | m need not be marked: one hit in three.
// Counting hits k = 0, 1, ... from the segment's first hit n0 = a + 2 j0 =
// p m0, hit k is p (m0 + 2k), a multiple of 3 iff k = m0 (mod 3), and
// m0 = n0 p (mod 3) (p^-1 = p mod 3).  a3 = a mod 3.
__device__ __forceinline__ uint32_t skip_residue(uint32_t a3, uint32_t j0, uint32_t p) {
  return ((a3 + 2u * j0) * (p % 3u)) % 3u;
}
// 5 is in every wheel too: hit k is a multiple of 5 iff k = 2 m0 (mod 5),
// m0 = n0 p^-1 (mod 5); a5 = a mod 5, p^-1 mod 5 from the nibble table
// 1 -> 1, 2 -> 3, 3 -> 2, 4 -> 4.
__device__ __forceinline__ uint32_t skip_residue5(uint32_t a5, uint32_t j0, uint32_t p) {
  const uint32_t inv = (0x42310u >> (4u * (p % 5u))) & 7u;
  return ((a5 + 2u * j0) * 2u * inv) % 5u;
}
// the 8 kept hit offsets of a period of 15 (k mod 15 not = r3 mod 3 and not
// = r5 mod 5), ascending, as nibbles of one word: table entry 5 r3 + r5
__device__ __forceinline__ uint32_t kept15(uint32_t r3, uint32_t r5) {
  uint32_t keep = ~((0x1249u << r3) | (0x421u << r5)) & 0x7FFFu, w = 0;
  for (int i = 0; i < 8; ++i) {
    w |= (uint32_t)(__ffs(keep) - 1) << (4 * i);
    keep &= keep - 1u;
  }
  return w;
}
// the two kept offsets {0, 1, 2} \ {skip} of a period of three steps
__device__ __forceinline__ uint32_t keep_lo(uint32_t skip) { return skip == 0u ? 1u : 0u; }
__device__ __forceinline__ uint32_t keep_hi(uint32_t skip) { return skip == 2u ? 1u : 2u; }

// Mark bit `mask` of the words at byte offsets A + t step < alim of the
// segment, t = 0, 1, ... except t = skip (mod 3): the hits of one residue
// class mod 1024 that are not multiples of 3 (2 instructions per mark: the
// address add and the atomic, plus a guard per 4 marks).
__device__ __forceinline__ void mark_run(uint32_t A, uint32_t alim, uint32_t step, uint32_t mask,
                                         uint32_t skip) {
  uint32_t A1 = A + keep_lo(skip) * step, A2 = A + keep_hi(skip) * step;  // A1 < A2 < A1 + 3 step
  const uint32_t s3 = 3u * step;
  for (; A2 + s3 < alim; A1 += 2u * s3, A2 += 2u * s3) {
    red_or(A1, mask);
    red_or(A2, mask);
    red_or(A1 + s3, mask);
    red_or(A2 + s3, mask);
  }
  if (A1 < alim) {
    red_or(A1, mask);
    if (A2 < alim) {
      red_or(A2, mask);
      if (A1 + s3 < alim) red_or(A1 + s3, mask);
    }
  }
}

// Byte limit of the residue class mod 1024 through slot j (bank b = j & 31):
// its slots are j + 1024 p s at bytes 4 b + 128 (block), and slot < valid
// <=> block < VB + [(j & 1023) < (valid & 1023)], VB = valid >> 10.
__device__ __forceinline__ uint32_t class_limit(uint32_t j, uint32_t valid) {
  const uint32_t lim = (valid >> 10) + ((j & 1023u) < (valid & 1023u) ? 1u : 0u);
  return ((j & 31u) << 2) + (lim << 7);
}

// A4/A5: mark the odd multiples of every base prime in [R.start, R.end).
// Hit k of prime p in the segment is slot j0 + k p.  In the transposed
// layout the bank of slot j is j mod 32, so (p odd):
//  * 32 consecutive hits of p sit in 32 distinct banks;
//  * hits k and k + 1024 (one residue class mod 1024) share bank and bit
//    position and sit 32 p words apart: a lane walking a class keeps one mask
//    and adds 128 p bytes per atomic, and 32 consecutive classes are 32 banks.
// Regions by K = S/p (internal.h):
//  (A1) K >= kUnitHits: units (prime, group g of 32 classes) round robin over
//       the warps; lane l walks class 32 g + l.
//  (A2) kClassHits <= K < kUnitHits: one prime per warp; lane l walks the
//       classes l, l + 32, ..., l + 992 (moving from one class to the next is
//       a rotation of the mask and an add: slot + 32 p).
//  (B)  kWarpHits <= K < kClassHits: one prime per warp; lane l takes the
//       hits l + 32 s (row += p, mask rotated by p per hit).
//  (C)  K < kWarpHits: one prime per lane, unrolled by kLargeILP loads, in
//       up to three loops over index ranges: K >= kC15Hits [R.warp, R.few)
//       skips the multiples of 3 and 5 (8 kept hits per 15), then the
//       multiples of 3 only, and in the batch kernel K <= kPlainHits
//       [R.two, ...) plainly; the bucket primes (K < kBucketHits, see
//       bucket_drain) when the runtime enables buckets.
// Every atomic of (A1)-(B) is conflict-free; (C) has random banks.  Hits
// that are multiples of 3 (k = m0 mod 3, skip_residue) are skipped in every
// region: one atomic in three (the wheel marked them).  First hits come
// from a Barrett reduction, 32 primes per warp at a time, with shuffle
// broadcast; p^2 >= segment end stops a warp.  Work is dealt statically and
// evenly: (A2) in pieces round robin, (B) and (C) in boustrophedon order over
// the warps / threads.
template <int kPlainU>  // primes per thread and pass of the plain loop; 0 = no plain loop
__device__ __forceinline__ void mark_segment(uint32_t sb, const uint32_t *__restrict__ primes,
                                             const uint64_t *__restrict__ recips,
                                             const PrimeRegions R, uint32_t flags,
                                             uint64_t a, uint32_t valid, unsigned long long *prof,
                                             const uint32_t *k15, const uint2 *__restrict__ pk44 = nullptr) {
  constexpr bool kPlainTwo = kPlainU > 0;
  // diagnostics (sieve_debug_set_flags): drop whole regions (wrong results)
  const uint32_t a1_end = flags & kFlagSkipA ? R.start : R.unit;
  const uint32_t a2_end = flags & kFlagSkipA ? R.unit : R.cls;
  const uint32_t b_end = flags & kFlagSkipB ? R.cls : R.warp;
  const uint32_t c_end = flags & kFlagSkipC ? R.warp : R.big;
  const long long t0 = prof ? clock64() : 0;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint64_t seg_end = a + 2ull * valid;
  const bool whole = (valid & 1023u) == 0;  // every class has the same block limit
  const uint32_t a3 = (uint32_t)(a % 3u), a5 = (uint32_t)(a % 5u);

  // (A1) units (prime, class group), dealt round robin over the warps:
  // unit 32 i + g goes to warp (32 i + g) mod nw, rot = 32 i mod nw
  const uint32_t c32 = 32u % nw;
  uint32_t rot = (32u * R.start) % nw;
  for (uint32_t ib = R.start; ib < a1_end; ib += 32) {
    const uint32_t i = ib + lane;
    uint32_t pl = 0, jl = kNone;
    if (i < a1_end) {
      pl = __ldg(primes + i);
      jl = first_hit(a, seg_end, pl, __ldg(recips + i));
    }
    const uint32_t nb = min(32u, a1_end - ib);
    for (uint32_t k = 0; k < nb; ++k) {
      const uint32_t p = __shfl_sync(0xffffffffu, pl, k);
      const uint32_t j0 = __shfl_sync(0xffffffffu, jl, k);
      if (j0 == kNone) break;  // p^2 past the segment, and so for every later prime
      const uint32_t g0 = warp >= rot ? warp - rot : warp + nw - rot;
      rot += c32;
      if (rot >= nw) rot -= nw;
      const uint32_t r0 = skip_residue(a3, j0, p);
      for (uint32_t g = g0; g < 32u; g += nw) {
        const uint32_t c = 32u * g + lane;  // class c: hits k = c + 1024 t = c + t (mod 3)
        const uint32_t j = j0 + c * p;      // its first hit
        mark_run(sb + t_addr(j), sb + class_limit(j, valid), 128u * p, t_mask(j), (r0 + 1026u - c) % 3u);
      }
    }
  }
  const long long t1 = prof ? clock64() : 0;

  // (A2) lane l walks the classes l + 32 g of one prime; the 32 class
  // groups of a prime are cut into kA2Parts pieces dealt round robin over the
  // warps (few primes, each a lot of work: whole primes per warp would load
  // a dozen warps with most of the phase)
  {
    const uint32_t nitems = (a2_end - R.unit) * kA2Parts;
    for (uint32_t q = warp; q < nitems; q += nw) {
      const uint32_t i = R.unit + q / kA2Parts, h = q % kA2Parts;
      const uint32_t p = __ldg(primes + i);
      const uint32_t j0 = first_hit(a, seg_end, p, __ldg(recips + i));
      if (j0 == kNone) break;  // p^2 past the segment: so for every later item of this warp
      const uint32_t g0 = h * (32u / kA2Parts), g1 = g0 + 32u / kA2Parts;
      uint32_t j = j0 + (lane + 32u * g0) * p;  // first hit of class lane + 32 g0
      uint32_t mask = t_mask(j);
      const uint32_t step = 128u * p, dj = 32u * p;
      // class c = lane + 32 g skips t = r0 - c (mod 3); c + 32 steps it by +1
      uint32_t skip = (skip_residue(a3, j0, p) + 1026u - (lane + 32u * g0)) % 3u;
      if (whole) {
        const uint32_t alim = sb + ((j & 31u) << 2) + ((valid >> 10) << 7);
        for (uint32_t g = g0; g < g1; ++g, j += dj, mask = rotl(mask, p), skip = skip == 2u ? 0u : skip + 1u)
          mark_run(sb + t_addr(j), alim, step, mask, skip);
      } else {
        for (uint32_t g = g0; g < g1; ++g, j += dj, mask = rotl(mask, p), skip = skip == 2u ? 0u : skip + 1u)
          mark_run(sb + t_addr(j), sb + class_limit(j, valid), step, mask, skip);
      }
    }
  }
  const long long t2 = prof ? clock64() : 0;

  // (B) one prime per warp, lane l takes the hits l + 32 s: slot j advances
  // by 32 p, i.e. its row j >> 5 by p (bank fixed), so the byte offset is
  // (4 row) & ~127 | 4 bank and the mask rotates by p.
  const bool w32 = (valid & 31u) == 0;
  const uint32_t Qlim32 = sb + ((valid >> 5) << 2);
  // lane l skips s = 2 r0 + l (mod 3): for each r0, the lane's first kept
  // step o1 and the gap d to its second (2 bits per r0, indexed by 2 r0)
  uint32_t o1t = 0, dt = 0;
#pragma unroll
  for (uint32_t r = 0; r < 3u; ++r) {
    const uint32_t sig = (2u * r + lane) % 3u;
    o1t |= keep_lo(sig) << (2u * r);
    dt |= (keep_hi(sig) - keep_lo(sig)) << (2u * r);
  }
  // prime nw m + (m even ? w : nw - 1 - w) to warp w (boustrophedon: the
  // primes grow with the index, so a plain i mod nw loads the low warps)
  for (uint32_t ib = R.cls; ib < b_end; ib += 32u * nw) {
    const uint32_t i = ib + lane * nw + ((lane & 1u) ? nw - 1u - warp : warp);
    uint32_t pl = 0, jl = kNone;
    if (i < b_end) {
      pl = __ldg(primes + i);
      jl = first_hit(a, seg_end, pl, __ldg(recips + i));
      if (jl != kNone) jl |= skip_residue(a3, jl, pl) << 30;  // j0 < 2^22: r0 rides in bits 30-31
    }
    bool stop = false;
    for (uint32_t k = 0; k < 32u; ++k) {
      const uint32_t p = __shfl_sync(0xffffffffu, pl, k);
      const uint32_t jp = __shfl_sync(0xffffffffu, jl, k);
      if (jp == kNone) { stop = true; break; }  // and so for every later prime
      // lane l's hits k = l + 32 s: multiples of 3 at s = 2 r0 + l (mod 3);
      // two streams over the kept steps (o1, o1 + d) of each period of three
      const uint32_t r2 = (jp >> 29) & 6u;  // 2 r0
      const uint32_t o1 = (o1t >> r2) & 3u, d = (dt >> r2) & 3u;
      const uint32_t j = (jp & 0x3FFFFFFFu) + (lane + 32u * o1) * p;  // the lane's first kept hit
      const uint32_t row = j >> 5;
      const uint32_t b4 = (j << 2) & 124u;  // 4 bank
      // Q = shared byte address of the hit's block plus 4 (row & 31): the
      // 128-byte aligned base keeps (Q & ~127) | b4 the hit's word
      uint32_t Q1 = sb + 4u * row;
      uint32_t m1 = __funnelshift_l(0u, 1u, row);
      // slot < valid <=> row < ceil((valid - bank) / 32) (0 when bank >= valid);
      // valid a multiple of 32: row < valid / 32 for every bank
      const uint32_t Qlim = w32 ? Qlim32 : sb + (((valid + 31u - (j & 31u)) >> 5) << 2);
      const uint32_t s4 = 4u * p;
      uint32_t Q2 = Q1 + d * s4;
      uint32_t m2 = rotl(m1, d * p);
      const uint32_t s3 = 3u * s4, p3 = 3u * p;
#if SIEVE_B_PAIR
      // Paired blocks: hits 96 steps apart (96 = 0 mod 32 and mod 3) have the
      // same bit (row + 96 p = row mod 32) and the same skip residue, and their
      // byte offsets differ by D = 384 p, a multiple of 128: one mask rotation
      // and one LOP3 serve two atomics, the second address is one add.  Each
      // block marks steps [0, 96) and [96, 192) of the lane's walk in 16
      // iterations, then skips the 96 steps its second stream covered (the
      // masks rotate by 32 x 3p = 0 mod 32 per block: unchanged).  Only whole
      // blocks inside the segment; the loop below takes the rest.
      const uint32_t D = 32u * s3;
      for (; Q2 + 31u * s3 + D < Qlim; Q1 += D, Q2 += D) {
#pragma unroll 2
        for (int c = 0; c < 16; ++c, Q1 += 2u * s3, Q2 += 2u * s3) {
          const uint32_t a1 = (Q1 & ~127u) | b4, a2 = (Q2 & ~127u) | b4;
          red_or(a1, m1);
          red_or(a1 + D, m1);
          red_or(a2, m2);
          red_or(a2 + D, m2);
          m1 = rotl(m1, p3);
          m2 = rotl(m2, p3);
          const uint32_t a3 = ((Q1 + s3) & ~127u) | b4, a4 = ((Q2 + s3) & ~127u) | b4;
          red_or(a3, m1);
          red_or(a3 + D, m1);
          red_or(a4, m2);
          red_or(a4 + D, m2);
          m1 = rotl(m1, p3);
          m2 = rotl(m2, p3);
        }
      }
#endif
      for (; Q2 + s3 < Qlim; Q1 += 2u * s3, Q2 += 2u * s3) {
        red_or((Q1 & ~127u) | b4, m1);
        red_or((Q2 & ~127u) | b4, m2);
        m1 = rotl(m1, p3);
        m2 = rotl(m2, p3);
        red_or(((Q1 + s3) & ~127u) | b4, m1);
        red_or(((Q2 + s3) & ~127u) | b4, m2);
        m1 = rotl(m1, p3);
        m2 = rotl(m2, p3);
      }
      if (Q1 < Qlim) {  // the last < 4 kept hits, predicated (Q1 < Q2 < Q1 + s3)
        red_or((Q1 & ~127u) | b4, m1);
        if (Q2 < Qlim) {
          red_or((Q2 & ~127u) | b4, m2);
          if (Q1 + s3 < Qlim) red_or(((Q1 + s3) & ~127u) | b4, rotl(m1, p3));
        }
      }
    }
    if (stop) break;
  }
  const long long t3 = prof ? clock64() : 0;

  // (C) large primes: lane per prime (few hits each).  Thread t takes the
  // primes t + nt m, kLargeILP at a time, and issues all their loads and
  // Barrett reductions before marking, so the L2 latency of the prime list
  // overlaps.  The lane walks J = 4 j + 32 sb: the byte offset
  // of slot j is (J >> 5) & ~127 | J & 127 and its bit is (J >> 7) & 31 (the
  // base term is a multiple of 4096, invisible to both).
  const uint32_t Jlim = 4u * valid + 32u * sb;
  // round m of nt primes: thread t takes prime m nt + (m even ? t : nt - 1 - t).
  // Primes [R.warp, few) have >= kC15Hits hits per full segment and skip the
  // multiples of 5 as well (8 kept hits per period of 15); [few, c_end) skip
  // the multiples of 3 only.  Two loops: no per-lane branch on the walk kind.
  const uint32_t few = min(R.few, c_end);
  // the scale of first_hit_scaled: a < 2^(32+t); the walks use it when every
  // prime of the region exceeds 2^t (the region's first prime is its
  // smallest) and t <= 28 (p < 2^30).  Only in the kernels with the plain
  // pass (r > S / kPlainHits): there the (C) walks gain too (configs 4 and 5:
  // 1.7 % / 1.4 %), while in the others config 3 (+0.5 %) and config 2
  // (+1.5 %) lose (profiles/r02_negative_ab.txt item 12).
  uint32_t t = 0, a_sh = 0, na_lo = 0, sh = 32;
  bool scaled_c = false;
  if constexpr (kPlainTwo) {
    t = (a >> 32) ? 32u - __clz((uint32_t)(a >> 32)) : 0u;
    a_sh = (uint32_t)(a >> t);
    na_lo = 0u - (uint32_t)a;
    sh = 32u - t;
    scaled_c = SIEVE_C_SCALED && R.warp < c_end && t <= 28u && (1u << t) < __ldg(primes + R.warp);
  }
  auto c_loop = [&](uint32_t cb, uint32_t ce, auto by15) {
    for (uint32_t k0 = cb; k0 < ce; k0 += kLargeILP * blockDim.x) {
      uint32_t pk[kLargeILP], jk[kLargeILP];
      uint64_t rk[kLargeILP];
#pragma unroll
      for (int u = 0; u < kLargeILP; ++u) {
        const uint32_t ku = k0 + u * blockDim.x + ((u & 1) ? blockDim.x - 1u - threadIdx.x : threadIdx.x);
        const uint32_t k = min(ku, ce - 1u);
        pk[u] = __ldg(primes + k);
        rk[u] = __ldg(recips + k);
      }
      if (kPlainTwo && scaled_c && (uint64_t)pk[kLargeILP - 1] * pk[kLargeILP - 1] <= a) {  // the lane's largest
#pragma unroll
        for (int u = 0; u < kLargeILP; ++u) {
          const uint32_t ku = k0 + u * blockDim.x + ((u & 1) ? blockDim.x - 1u - threadIdx.x : threadIdx.x);
          const uint32_t j = first_hit_scaled(a_sh, na_lo, sh, pk[u], rk[u]);
          jk[u] = ku >= ce ? kNone : j;
        }
      } else {
#pragma unroll
        for (int u = 0; u < kLargeILP; ++u) {
          jk[u] = first_hit(a, seg_end, pk[u], rk[u]);
          const uint32_t ku = k0 + u * blockDim.x + ((u & 1) ? blockDim.x - 1u - threadIdx.x : threadIdx.x);
          if (ku >= ce) jk[u] = kNone;
        }
      }
      if (jk[0] == kNone) break;  // p^2 past the segment: so for every later prime
#pragma unroll
      for (int u = 0; u < kLargeILP; ++u) {
        if (jk[u] == kNone) break;
        const uint32_t P4 = 4u * pk[u], S3 = 3u * P4;
        const uint32_t r0 = skip_residue(a3, jk[u], pk[u]);  // hits k = r0 (mod 3): multiples of 3
        if constexpr (decltype(by15)::value) {
          const uint32_t nib = k15[5u * r0 + skip_residue5(a5, jk[u], pk[u])];
          uint32_t off[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) off[q] = ((nib >> (4 * q)) & 15u) * P4;
          uint32_t J = 4u * jk[u] + 32u * sb;
          for (; J + off[7] < Jlim; J += 5u * S3) {  // whole periods
#pragma unroll
            for (int q = 0; q < 8; ++q) red_or(j_addr(J + off[q]), j_mask(J + off[q]));
          }
#pragma unroll
          for (int q = 0; q < 7; ++q)  // the last partial period (offsets ascending)
            if (J + off[q] < Jlim) red_or(j_addr(J + off[q]), j_mask(J + off[q]));
        } else {
          uint32_t J1 = 4u * jk[u] + 32u * sb + keep_lo(r0) * P4;
          uint32_t J2 = J1 + (keep_hi(r0) - keep_lo(r0)) * P4;  // J1 < J2 < J1 + S3
          for (; J2 + S3 < Jlim; J1 += 2u * S3, J2 += 2u * S3) {
            red_or(j_addr(J1), j_mask(J1));
            red_or(j_addr(J2), j_mask(J2));
            red_or(j_addr(J1 + S3), j_mask(J1 + S3));
            red_or(j_addr(J2 + S3), j_mask(J2 + S3));
          }
          if (J1 < Jlim) {
            red_or(j_addr(J1), j_mask(J1));
            if (J2 < Jlim) {
              red_or(j_addr(J2), j_mask(J2));
              if (J1 + S3 < Jlim) red_or(j_addr(J1 + S3), j_mask(J1 + S3));
            }
          }
        }
      }
    }
  };
  c_loop(R.warp, few, std::true_type{});
  // batch kernel (kPlainTwo): p > S / kPlainHits has at most kPlainHits hits,
  // marked as they come (skipping a multiple of 3 would cost more than its
  // atomic); compiled
  // out of the other kernels, whose loops it would perturb (+0.7 % measured)
  const uint32_t two = kPlainTwo ? max(few, min(R.two, c_end)) : c_end;
  c_loop(few, two, std::false_type{});
  // The plain primes (batch kernel): kPlainILP per thread and pass.  While
  // the pass's largest prime has p^2 <= a (the item lies above p^2 -- almost
  // always in a batch far from 0), the first hit needs neither the p^2 clamp
  // nor the 64-bit compares of first_hit: with r = a mod p (Barrett), the
  // first odd multiple a + 2 j has j = (((r & 1) ? p : 2 p) - r) / 2 mod p.
  // (Config 5 spends most of its time here: one such reduction per (prime,
  // item) for ~1.1e9 pairs, most of them without a hit.)
  if constexpr (kPlainTwo) {
    constexpr int U = kPlainU > 0 ? kPlainU : 1;
    // a first hit of kFar puts the walk start past Jlim: no hit, no branch
    constexpr uint32_t kFar = 1u << 29;
    // first_hit_scaled when every plain prime > 2^t (the first is the smallest)
    const bool scaled = two < c_end && t <= 28u && (1u << t) < __ldg(primes + two);
    // one pass of U primes per thread; kFull: all of them below c_end (no
    // clamp, no compare).  Returns false when p^2 is past the segment.
    auto plain_pass = [&](uint32_t k0, auto full) -> bool {
      constexpr bool kFull = decltype(full)::value;
      uint32_t pk[U], jk[U], kk[U];
      uint64_t rk[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        kk[u] = k0 + u * blockDim.x + ((u & 1) ? blockDim.x - 1u - threadIdx.x : threadIdx.x);
        const uint32_t k = kFull ? kk[u] : min(kk[u], c_end - 1u);
        pk[u] = __ldg(primes + k);
        rk[u] = __ldg(recips + k);
      }
      if ((uint64_t)pk[U - 1] * pk[U - 1] <= a) {  // the largest of the pass: so for all
        if (scaled) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t j = first_hit_scaled(a_sh, na_lo, sh, pk[u], rk[u]);
            jk[u] = (kFull || kk[u] < c_end) ? j : kFar;
          }
        } else {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t j = first_hit_above(a, pk[u], rk[u]);
            jk[u] = (kFull || kk[u] < c_end) ? j : kFar;
          }
        }
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t j = first_hit(a, seg_end, pk[u], rk[u]);
          jk[u] = ((!kFull && kk[u] >= c_end) || j == kNone) ? kFar : j;
        }
        if (jk[0] == kFar) return false;  // p^2 past the segment: so for every later prime
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t P4 = 4u * pk[u];
        for (uint32_t J = 4u * jk[u] + 32u * sb; J < Jlim; J += P4) red_or(j_addr(J), j_mask(J));
      }
      return true;
    };
    // batch kernel (pk44 != nullptr): {p, floor(2^44 / p)} in one 8-byte load
    // per prime instead of 4 + 8 bytes in two loads, M = floor(2^44/p) >> (12 - t)
    // (floors nest; needs a < 2^44 and every plain prime > 2^12, so that the
    // quotient fits 32 bits)
    const bool packed = pk44 != nullptr && scaled && t <= 12u && 4096u < __ldg(primes + two);
    const uint32_t sh44 = 12u - t;
    auto plain_pass_packed = [&](uint32_t k0, auto full) -> bool {
      constexpr bool kFull = decltype(full)::value;
      uint32_t pk[U], jk[U], kk[U], mk[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        kk[u] = k0 + u * blockDim.x + ((u & 1) ? blockDim.x - 1u - threadIdx.x : threadIdx.x);
        const uint32_t k = kFull ? kk[u] : min(kk[u], c_end - 1u);
        const uint2 v = __ldg(pk44 + k);
        pk[u] = v.x;
        mk[u] = v.y >> sh44;
      }
      if ((uint64_t)pk[U - 1] * pk[U - 1] <= a) {  // the largest of the pass: so for all
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t j = first_hit_m(a_sh, na_lo, pk[u], mk[u]);
          jk[u] = (kFull || kk[u] < c_end) ? j : kFar;
        }
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t k = kFull ? kk[u] : min(kk[u], c_end - 1u);
          const uint32_t j = first_hit(a, seg_end, pk[u], __ldg(recips + k));
          jk[u] = ((!kFull && kk[u] >= c_end) || j == kNone) ? kFar : j;
        }
        if (jk[0] == kFar) return false;  // p^2 past the segment: so for every later prime
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t P4 = 4u * pk[u];
        for (uint32_t J = 4u * jk[u] + 32u * sb; J < Jlim; J += P4) red_or(j_addr(J), j_mask(J));
      }
      return true;
    };
    const uint32_t step = U * blockDim.x;
    uint32_t k0 = two;
    bool more = true;
    if (packed) {
      for (; more && c_end - k0 >= step && k0 < c_end; k0 += step) more = plain_pass_packed(k0, std::true_type{});
      if (more && k0 < c_end) plain_pass_packed(k0, std::false_type{});
    } else {
      for (; more && c_end - k0 >= step && k0 < c_end; k0 += step) more = plain_pass(k0, std::true_type{});
      if (more && k0 < c_end) plain_pass(k0, std::false_type{});
    }
  }
  if (prof) {  // per-warp busy cycles of the regions (diagnostics only)
    const long long t4 = clock64();
    if ((threadIdx.x & 31u) == 0) {
      atomicAdd(prof + 3, (unsigned long long)(t1 - t0));
      atomicAdd(prof + 4, (unsigned long long)(t2 - t1));
      atomicAdd(prof + 5, (unsigned long long)(t3 - t2));
      atomicAdd(prof + 7, (unsigned long long)(t4 - t3));
      const uint32_t w = (threadIdx.x >> 5) & 31u;  // per-warp region cycles (load balance)
      atomicAdd(prof + 8 + w, (unsigned long long)(t2 - t0));
      atomicAdd(prof + 40 + w, (unsigned long long)(t3 - t2));
      atomicAdd(prof + 72 + w, (unsigned long long)(t4 - t3));
    }
  }
}

// ---------------------------------------------------------------------------
// A5: per-segment buckets for the large primes (K < kBucketHits), so that a
// segment a prime does not hit costs it nothing.  A CTA sieves a contiguous
// run of segments [s0, s1); warp w owns the bucket primes R.big + w + nw m.
// An entry {p, o} in ring slot s mod R of warp w says: prime p next hits
// slot o of segment s (o >= S: only parked there, re-queued further).  Per
// segment the warp drains its slot: marks the hits o, o + p, ... < valid,
// then re-queues p in the slot of its next segment s + d, 1 <= d < R.  The
// fill counts of the warp's R slots live in registers (lane t: slot t); an
// append ranks the lanes with the same target slot by one ballot per slot,
// so there are no atomics on the bookkeeping and the entries are
// warp-private.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint2 *bucket_at(const SieveParams &P, uint32_t slot, uint32_t warp,
                                           uint32_t nw) {
  return P.buckets + ((size_t)(blockIdx.x * P.ring + slot) * nw + warp) * P.capw;
}

// append e to ring slot `slot` for every lane with `alive`; cnt: lane t holds
// the fill count of slot t
__device__ __forceinline__ void bucket_push(const SieveParams &P, uint32_t &cnt, bool alive,
                                            uint32_t slot, uint2 e, uint32_t warp, uint32_t nw) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t pos = 0;
  for (uint32_t t = 0; t < P.ring; ++t) {  // ring slots in turn: rank = lanes below with slot t
    const uint32_t m = __ballot_sync(0xffffffffu, alive && slot == t);
    const uint32_t base = __shfl_sync(0xffffffffu, cnt, t);
    if (slot == t) pos = base + __popc(m & ((1u << lane) - 1u));
    if (lane == t) cnt += __popc(m);
  }
  SV_CHECK(!alive || (pos < P.capw && slot < P.ring), kVioScratch);
  if (alive) bucket_at(P, slot, warp, nw)[pos] = e;
}

// o / S for o < 2^31 (S = seg_bits >= 2^13): multiply-high, then one correction
__device__ __forceinline__ uint32_t div_seg(const SieveParams &P, uint32_t o) {
  uint32_t d = __umulhi(o, P.inv_seg);
  if (d * P.seg_bits > o) --d;
  return d;
}

// fill the warp's buckets at the start of its run: first hit of every owned
// bucket prime at or after slot 0 of segment s0 (64-bit: the hit may lie far
// ahead when p^2 is beyond the run start)
__device__ __forceinline__ void bucket_fill(const SieveParams &P, const PrimeRegions &R,
                                            uint32_t &cnt, uint64_t s0, uint64_t s1) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint64_t a = P.o0 + 2ull * s0 * P.seg_bits;  // first odd integer of the run
  const uint64_t run = (s1 - s0) * (uint64_t)P.seg_bits;
  for (uint32_t ib = R.big + warp; ib < R.end; ib += 32u * nw) {
    const uint32_t i = ib + lane * nw;
    bool alive = i < R.end;
    uint32_t p = 0, slot = 0, o = 0;
    if (alive) {
      p = __ldg(P.primes + i);
      const uint64_t pp = (uint64_t)p * p;
      const uint64_t q = __umul64hi(a, __ldg(P.recips + i));
      uint32_t r = (uint32_t)(a - q * (uint64_t)p);
      r = min(r, r - p);
      uint64_t d = r ? p - r : 0u;
      d += (d & 1u) ? p : 0u;  // a odd: the next odd multiple is a + d, d even
      uint64_t j = d >> 1;
      if (a + 2ull * j < pp) j = (pp - a) >> 1;
      alive = j < run;
      if (alive) {
        const uint64_t dseg = j / P.seg_bits;
        const uint32_t dd = (uint32_t)min(dseg, (uint64_t)(P.ring - 1u));
        o = (uint32_t)(j - (uint64_t)dd * P.seg_bits);
        slot = (uint32_t)((s0 + dd) % P.ring);
      }
    }
    bucket_push(P, cnt, alive, slot, make_uint2(p, o), warp, nw);
  }
}

// drain the warp's ring slot of segment s: mark, then re-queue
__device__ __forceinline__ void bucket_drain(const SieveParams &P, uint32_t &cnt, uint32_t sb,
                                             uint32_t q, uint32_t left, uint32_t valid) {
  // q = s mod R, left = s1 - s: no 64-bit division here (a runtime 64-bit
  // modulo is a subroutine call, and ptxas then puts YIELDs in every loop of
  // the kernel: measured 1.5x slower marking)
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t n = __shfl_sync(0xffffffffu, cnt, q);
  const uint2 *src = bucket_at(P, q, warp, nw);
  for (uint32_t e0 = 0; e0 < n; e0 += 32u * kDrainILP) {
    uint2 v[kDrainILP];
#pragma unroll
    for (uint32_t u = 0; u < kDrainILP; ++u) {  // all loads first: their latency overlaps
      const uint32_t e = e0 + 32u * u + lane;
      v[u] = e < n ? __ldcg(src + e) : make_uint2(0u, 0u);
    }
#pragma unroll
    for (uint32_t u = 0; u < kDrainILP; ++u) {
      const uint32_t p = v[u].x;
      uint32_t o = v[u].y, slot = 0;
      bool alive = e0 + 32u * u + lane < n;
      if (alive) {
        // the hits of this segment: p > S / kBucketHits, so at most
        // kBucketHits of them (o >= S: an entry parked here, no hit)
#pragma unroll
        for (uint32_t h = 0; h < kBucketHits; ++h) {
          if (o < valid) {
            const uint32_t J = 4u * o + 32u * sb;
            red_or(j_addr(J), j_mask(J));
            o += p;
          }
        }
        const uint32_t d = min(div_seg(P, o), P.ring - 1u);
        o -= d * P.seg_bits;
        alive = d >= 1u && d < left;
        slot = q + d >= P.ring ? q + d - P.ring : q + d;
      }
      bucket_push(P, cnt, alive, slot, make_uint2(p, o), warp, nw);
    }
  }
  if (lane == q) cnt = 0;  // no push above targets slot q (d >= 1)
}

// In-place 32x32 bit transpose of every 1024-slot block of the segment
// (transposed layout -> natural layout: word w holds slots 32 w .. 32 w + 31,
// LSB first), one block per warp at a time.  Lane r holds row r; stage w
// swaps the off-diagonal w x w sub-blocks of every 2w x 2w block: the lane
// below (lane & w == 0) needs its partner's columns c - w, the lane above
// its partner's columns c + w, so each lane sends itself rotated right by w
// (upper partner) or 32 - w (lower partner) and merges with one bit-select:
// three instructions (SHF, SHFL, LOP3) per stage.
template <bool kInvert = false>
__device__ __forceinline__ void untranspose(uint32_t *seg, uint32_t valid) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t nblk = (valid + 1023u) >> 10;
  uint32_t amt[5], keep[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const uint32_t w = 16u >> k;
    const uint32_t m = k == 0 ? 0x0000FFFFu : k == 1 ? 0x00FF00FFu : k == 2 ? 0x0F0F0F0Fu
                     : k == 3 ? 0x33333333u : 0x55555555u;  // columns c with (c & w) == 0
    amt[k] = (lane & w) ? 32u - w : w;
    keep[k] = (lane & w) ? ~m : m;
  }
  // kUT independent blocks per warp and pass: the five shuffle stages of one
  // block are a dependent chain (~200 cycles), interleaving hides it
  constexpr int kUT = SIEVE_UNTRANSPOSE_ILP;
  for (uint32_t B = warp; B < nblk; B += kUT * nw) {
    uint32_t x[kUT];
#pragma unroll
    for (int u = 0; u < kUT; ++u) {
      const uint32_t Bu = B + u * nw;
      x[u] = Bu < nblk ? seg[32u * Bu + lane] : 0u;
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) {
#pragma unroll
      for (int u = 0; u < kUT; ++u) {
        const uint32_t y = __shfl_xor_sync(0xffffffffu, __funnelshift_r(x[u], x[u], amt[k]), 16u >> k);
        asm("lop3.b32 %0, %0, %1, %2, 0xE4;" : "+r"(x[u]) : "r"(y), "r"(keep[k]));  // (x & keep) | (y & ~keep)
      }
    }
#pragma unroll
    for (int u = 0; u < kUT; ++u) {
      const uint32_t Bu = B + u * nw;
      SV_CHECK(Bu >= nblk || 4u * (32u * Bu + lane) + (uint32_t)__cvta_generic_to_shared(seg) < s_chk_hi,
               kVioScratch);
      if (Bu < nblk) seg[32u * Bu + lane] = kInvert ? ~x[u] : x[u];
    }
  }
}

// A7 by TMA (bitmap mode): the segment's words go from shared memory to HBM
// as one bulk copy issued by one thread (cp.async.bulk, async proxy), so the
// stores cost no instructions of the other threads and drain while they count.
// The threads' generic-proxy writes are fenced to the async proxy before the
// block barrier that precedes the copy; the issuing thread waits for the
// copy's shared-memory reads before the buffer is reused.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_store(void *gdst, const void *ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
               "cp.async.bulk.commit_group;"
               ::"l"(gdst), "r"((uint32_t)__cvta_generic_to_shared(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// A6/A7: count, sum and (bitmap mode) write-back of one segment.
//
// Sum of the primes of the segment = C*a + 2*J, where a is the segment's
// first odd integer, C the number of set (prime) bits and J the sum of their
// slots j.  Per quad the thread needs the quad's popcount (for C and the
// quad's weight) and the word popcounts; the bit-position part sum_b b * n_b
// is accumulated without popcounts in carry-save bit planes (Harley-Seal
// adder tree: plane k holds bit k of the per-position count n_b), and read
// once per segment.
//  * natural layout (bitmap mode, after untranspose): word 4q + e, bit b is
//    slot 128 q + 32 e + b;
//  * transposed layout (count and batch modes): word 4q + e, bit i is slot
//    1024 (q >> 3) + 4 (q & 7) + e + 32 i = 128 q - 124 (q & 7) + e + 32 i,
//    and q & 7 = tid & 7 for every quad of a thread (nt is a multiple of 8).
__device__ __forceinline__ void csa(uint32_t &carry, uint32_t &sum, uint32_t a, uint32_t b,
                                    uint32_t c) {
  const uint32_t u = a ^ b;
  carry = (a & b) | (u & c);
  sum = u ^ c;
}

template <int MODE>
__device__ __forceinline__ void epilogue(const uint32_t *seg, uint64_t a, uint64_t bit0,
                                         uint32_t valid, uint32_t *out, uint64_t out_words,
                                         uint32_t vec4, unsigned long long &cnt,
                                         unsigned long long &sum) {
  constexpr bool kNatural = MODE == kBitmap;
  const uint32_t nq = kNatural ? (valid + 127u) >> 7 : ((valid + 1023u) >> 10) << 3;
  const uint4 *seg4 = reinterpret_cast<const uint4 *>(seg);
  const uint64_t w0 = bit0 >> 5;  // first word of the segment in the call's grid
  // planes of per-bit-position counts (counts < 512: <= 127 quads per thread)
  uint32_t ones = 0, twos = 0, fours = 0, p8 = 0, p16 = 0, p32 = 0, p64 = 0, p128 = 0;
  uint32_t C = 0, X = 0, Q = 0;  // count, sum of e c_e, sum of k c_k
  // bitmap mode: seg holds the prime words (untranspose<true>); with a
  // 16-byte aligned output the whole 16-byte prefix of the segment's words
  // goes by one bulk copy (the call's last segment may end in < 4 words,
  // stored below)
  uint32_t n16 = 0;
  if (MODE == kBitmap && SIEVE_TMA_STORE && vec4) {
    const uint64_t nw = out_words > w0 ? min((uint64_t)4u * nq, out_words - w0) : 0ull;
    n16 = (uint32_t)nw & ~3u;
#if SIEVE_WB_DIAG != 2
    SV_CHECK(threadIdx.x != 0 || n16 == 0 || w0 + n16 <= out_words, kVioBitmapStore);
    if (threadIdx.x == 0 && n16) bulk_store(out + w0, seg, 4u * n16);
#endif
  }
  uint32_t k = 0;
  uint32_t q = threadIdx.x;
  if (!kNatural && SIEVE_EPI_PAIRS) {
    // count/batch modes: two quads (8 words) per carry-save step, so the
    // half-adder chain above weight 8 runs once per 8 words instead of 4
    for (; q + blockDim.x < nq; q += 2u * blockDim.x, k += 2u) {
      const uint4 v = seg4[q], u = seg4[q + blockDim.x];
      const uint32_t c0 = __popc(v.x), c1 = __popc(v.y), c2 = __popc(v.z), c3 = __popc(v.w);
      const uint32_t d0 = __popc(u.x), d1 = __popc(u.y), d2 = __popc(u.z), d3 = __popc(u.w);
      const uint32_t cq = c0 + c1 + c2 + c3, dq = d0 + d1 + d2 + d3;
      C += cq + dq;
      Q += k * (cq + dq) + dq;  // quads k and k + 1
      X += (c1 + d1) + 2u * (c2 + d2) + 3u * (c3 + d3);
      uint32_t tA, tB, fA, tC, tD, fB, e;
      csa(tA, ones, ones, v.x, v.y);
      csa(tB, ones, ones, v.z, v.w);
      csa(fA, twos, twos, tA, tB);
      csa(tC, ones, ones, u.x, u.y);
      csa(tD, ones, ones, u.z, u.w);
      csa(fB, twos, twos, tC, tD);
      csa(e, fours, fours, fA, fB);
      uint32_t cz = p8 & e; p8 ^= e;
      uint32_t cy = p16 & cz; p16 ^= cz;
      cz = p32 & cy; p32 ^= cy;
      cy = p64 & cz; p64 ^= cz;
      p128 ^= cy;
    }
  }
  for (; q < nq; q += blockDim.x, ++k) {
    const uint4 v = seg4[q];
    // count mode counts the composite (set) bits and converts at the end
    // (every statistic below is linear in the per-position counts); bitmap
    // mode holds the prime words themselves
    const uint32_t x0 = v.x, x1 = v.y, x2 = v.z, x3 = v.w;
    const uint32_t c0 = __popc(x0), c1 = __popc(x1), c2 = __popc(x2), c3 = __popc(x3);
    const uint32_t cq = c0 + c1 + c2 + c3;
    C += cq;
    Q += k * cq;
    X += c1 + 2u * c2 + 3u * c3;
    uint32_t tA, tB, fA;
    csa(tA, ones, ones, x0, x1);
    csa(tB, ones, ones, x2, x3);
    csa(fA, twos, twos, tA, tB);
    uint32_t cy = fours & fA;  // half-adder chain for the weight-4 carries
    fours ^= fA;
    uint32_t cz = p8 & cy; p8 ^= cy;
    cy = p16 & cz; p16 ^= cz;
    cz = p32 & cy; p32 ^= cy;
    cy = p64 & cz; p64 ^= cz;
    p128 ^= cy;
    if (MODE == kBitmap) {
      const uint64_t gw = w0 + 4ull * q;
      if (SIEVE_TMA_STORE && vec4) {
        if (4u * q >= n16) {  // past the bulk copy
          if (gw < out_words) out[gw] = x0;
          if (gw + 1 < out_words) out[gw + 1] = x1;
          if (gw + 2 < out_words) out[gw + 2] = x2;
          if (gw + 3 < out_words) out[gw + 3] = x3;
        }
      } else if (vec4 && gw + 4 <= out_words) {
        SV_CHECK((gw & 3) == 0, kVioBitmapStore);
        reinterpret_cast<uint4 *>(out)[gw >> 2] = make_uint4(x0, x1, x2, x3);
      } else {
        if (gw < out_words) out[gw] = x0;
        if (gw + 1 < out_words) out[gw + 1] = x1;
        if (gw + 2 < out_words) out[gw + 2] = x2;
        if (gw + 3 < out_words) out[gw + 3] = x3;
      }
    }
  }
  // sum of bit positions over all set bits = sum_k 2^k bit_index_sum(plane_k)
  uint32_t Bs = bit_index_sum(ones) + 2u * bit_index_sum(twos) + 4u * bit_index_sum(fours) +
                8u * bit_index_sum(p8) + 16u * bit_index_sum(p16) + 32u * bit_index_sum(p32) +
                64u * bit_index_sum(p64) + 128u * bit_index_sum(p128);
  if (!kNatural) {  // composite -> prime over the thread's k quads (128 bits each)
    C = 128u * k - C;                  // set bits
    Q = 64u * k * (k - 1u) - Q;        // sum of (quad index) x (set bits), 128 sum_{i<k} i
    X = 192u * k - X;                  // sum of e c_e: 32 (1 + 2 + 3) per quad
    Bs = 4u * 496u * k - Bs;           // per bit position: 4 k bits, positions sum to 496
  }
  // sum of 128 q over set bits, q = tid + k nt
  const uint64_t Jq = 128ull * ((uint64_t)threadIdx.x * C + (uint64_t)blockDim.x * Q);
  const uint64_t J = kNatural ? Jq + 32ull * X + Bs
                              : Jq - 124ull * (threadIdx.x & 7u) * C + X + 32ull * Bs;
  cnt += C;
  sum += (unsigned long long)C * a + 2ull * J;
#if SIEVE_WB_DIAG == 0
  if (MODE == kBitmap && SIEVE_TMA_STORE && threadIdx.x == 0 && n16) bulk_wait_read();
#endif
}

// ---------------------------------------------------------------------------
// Partial-block 32x32 bit transpose in registers (round 2 of A7; replaces
// the shuffle transpose above in bitmap and list modes).  kWbLanes = L
// lanes (u = lane mod L) share a 1024-slot block B: lane u holds rows
// R u .. R u + R - 1 (R = 32 / L) of its 32 transposed words in R
// registers.  Stage j (16, 8, 4, 2, 1) swaps the off-diagonal j x j
// sub-blocks of every 2j x 2j block between the row pairs (r, r + j): the
// lower row keeps its columns c with (c & j) == 0 and takes its partner's
// low columns moved up by j, the upper row keeps its high columns and takes
// its partner's high columns moved down -- a shift and a bit-select LOP3 per
// row.  Stages j >= R pair two lanes (one SHFL per row: with L = 4, stages
// 16 and 8); the others pair registers of one lane.  The shuffle transpose
// does all five stages with a SHFL per row (tools/transpose_bench.cu).
// L = 4 (default) gives 4 x 1664 quarter blocks per 208 KiB segment, 6.5
// per thread of 1024 -- 7 rounds, where halves take 4 rounds for 3.25 (the
// slowest thread sets the phase; same-box A/B in DESIGN.md).
//
// Bank skew: a warp holds 32 / L consecutive blocks, 128 bytes apart, so
// quad q of every block sits in the same 4 banks.  Lane (B, u) with
// t = B mod (8 / L) therefore loads and stores quad (8 / L) u + (q ^ t) in
// its q-th access (8 distinct quads over the warp: conflict-free LDS.128 /
// STS.128).  Register i of the lane then holds row R u + (i ^ 4t), and
// natural word R u + c must end in register c ^ 4t; the transpose absorbs
// both XOR permutations (of the row and column index bits that 4t can set,
// all below R): in those in-register stages j where bit j of 4t is set, the
// pair's roles swap (the lower row keeps its high columns and takes the
// partner's shifted down, and vice versa) -- a lane-dependent rotation
// amount and mask, the same two instructions.
// ---------------------------------------------------------------------------
constexpr uint32_t kWbLanes = SIEVE_WB_LANES;
constexpr uint32_t kWbRows = 32u / kWbLanes;   // rows per lane
constexpr uint32_t kWbQuads = kWbRows / 4u;    // quads per lane
static_assert(kWbLanes == 2 || kWbLanes == 4, "SIEVE_WB_LANES is 2 or 4");

__device__ __forceinline__ uint32_t bitsel(uint32_t x, uint32_t y, uint32_t k) {  // (x & k) | (y & ~k)
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(r) : "r"(x), "r"(y), "r"(k));
  return r;
}
template <uint32_t J>
struct TMask {  // columns c with (c & J) == 0
  static constexpr uint32_t v =
      J == 16 ? 0x0000FFFFu : J == 8 ? 0x00FF00FFu : J == 4 ? 0x0F0F0F0Fu : J == 2 ? 0x33333333u : 0x55555555u;
};
// in-register stage, roles swapped where `flip`
template <uint32_t J>
__device__ __forceinline__ void tstage_reg(uint32_t (&A)[kWbRows], bool flip) {
  if constexpr (J < kWbRows) {
    constexpr uint32_t m = TMask<J>::v;
    if (J >= 4) {  // lane-dependent (the skew reaches index bits 2 .. log2(kWbQuads) + 1)
      const uint32_t keep = flip ? ~m : m, amt = flip ? 32u - J : J;
#pragma unroll
      for (int r = 0; r < (int)kWbRows; ++r) {
        if (r & J) continue;
        const uint32_t x = A[r], y = A[r + J];
        A[r] = bitsel(x, __funnelshift_l(y, y, amt), keep);
        A[r + J] = bitsel(__funnelshift_r(x, x, amt), y, keep);
      }
    } else {
#pragma unroll
      for (int r = 0; r < (int)kWbRows; ++r) {
        if (r & J) continue;
        const uint32_t x = A[r], y = A[r + J];
        A[r] = bitsel(x, y << J, m);
        A[r + J] = bitsel(x >> J, y, m);
      }
    }
  }
}
// cross-lane stage j >= kWbRows: the partner is lane ^ (j / kWbRows); the
// lower lane takes the partner's row rotated left by j, the upper lane the
// partner's rotated right by j, so each lane sends its own row rotated the
// way its partner needs
template <uint32_t J>
__device__ __forceinline__ void tstage_lane(uint32_t (&A)[kWbRows], uint32_t u) {
  if constexpr (J >= kWbRows) {
    constexpr uint32_t m = TMask<J>::v, x = J / kWbRows;
    const bool upper = u & x;
    const uint32_t keep = upper ? ~m : m, send = upper ? J : 32u - J;
#pragma unroll
    for (int r = 0; r < (int)kWbRows; ++r) {
      const uint32_t y = __shfl_xor_sync(0xffffffffu, __funnelshift_l(A[r], A[r], send), x);
      A[r] = bitsel(A[r], y, keep);
    }
  }
}
// byte address (shared window) of the lane's first quad: its q-th quad is
// qa ^ (16 q) (a block is 128-byte aligned, the lane's quads 16 kWbQuads)
__device__ __forceinline__ uint32_t part_block_addr(const uint32_t *seg, uint32_t B, uint32_t u) {
  return (uint32_t)__cvta_generic_to_shared(seg) + 128u * B + 16u * kWbQuads * u + 16u * (B & (kWbQuads - 1u));
}
__device__ __forceinline__ void load_part_block(uint32_t qa, uint32_t (&A)[kWbRows]) {
#pragma unroll
  for (int q = 0; q < (int)kWbQuads; ++q)
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(A[4 * q]), "=r"(A[4 * q + 1]), "=r"(A[4 * q + 2]), "=r"(A[4 * q + 3])
                 : "r"(qa ^ (16u * q)));
}
template <bool kInvert>
__device__ __forceinline__ void store_part_block(uint32_t qa, const uint32_t (&A)[kWbRows]) {
  SV_CHECK((qa | (16u * (kWbQuads - 1u))) + 16u <= s_chk_hi, kVioScratch);
#pragma unroll
  for (int q = 0; q < (int)kWbQuads; ++q) {
    if (kInvert)
      asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(qa ^ (16u * q)), "r"(~A[4 * q]),
                   "r"(~A[4 * q + 1]), "r"(~A[4 * q + 2]), "r"(~A[4 * q + 3]) : "memory");
    else
      asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(qa ^ (16u * q)), "r"(A[4 * q]),
                   "r"(A[4 * q + 1]), "r"(A[4 * q + 2]), "r"(A[4 * q + 3]) : "memory");
  }
}
// rows -> natural words of the lane's part (register c = natural word
// kWbRows u + (c ^ 4t)).  Every lane of the warp must call it (shuffles).
__device__ __forceinline__ void transpose_part_block(uint32_t B, uint32_t u, uint32_t (&A)[kWbRows]) {
  tstage_lane<16>(A, u);
  tstage_lane<8>(A, u);
  const uint32_t k = 4u * (B & (kWbQuads - 1u));
  tstage_reg<8>(A, k & 8u);
  tstage_reg<4>(A, k & 4u);
  tstage_reg<2>(A, false);
  tstage_reg<1>(A, false);
}

// list mode: the in-place transpose of every block (no inversion)
__device__ __forceinline__ void untranspose_reg(uint32_t *seg, uint32_t valid) {
  const uint32_t nblk = (valid + 1023u) >> 10, lane = threadIdx.x & 31u, u = lane & (kWbLanes - 1u);
  for (uint32_t P0 = threadIdx.x & ~31u; P0 < kWbLanes * nblk; P0 += blockDim.x) {
    const bool own = (P0 + lane) / kWbLanes < nblk;
    const uint32_t B = min((P0 + lane) / kWbLanes, nblk - 1u);  // tail lanes redo the last block
    const uint32_t qa = part_block_addr(seg, B, u);
    uint32_t A[kWbRows];
    load_part_block(qa, A);
    transpose_part_block(B, u, A);
    __syncwarp();  // every lane's loads before a duplicate of the last block is stored
    if (own) store_part_block<false>(qa, A);
  }
}

// Carry-save accumulation of a lane's kWbRows prime words into 8 bit-sliced
// planes (plane k = bit k of the per-bit-position count, counts < 256),
// depth first: one CSA (two LOP3) per word and a short ripple of the top
// carry -- the count for a few ALU instructions per word and no POPC (POPC
// issues at a quarter of the LOP3 rate, tools/pipe_bench.cu: 0.5 vs 2 warp
// instructions per clock and SM).
__device__ __forceinline__ void planes_add(uint32_t (&pl)[8], const uint32_t (&A)[kWbRows]) {
  uint32_t c8[kWbRows / 8];
#pragma unroll
  for (int g = 0; g < (int)kWbRows / 8; ++g) {
    const uint32_t *w = A + 8 * g;
    uint32_t a, b, fA, fB;
    csa(a, pl[0], pl[0], ~w[0], ~w[1]);
    csa(b, pl[0], pl[0], ~w[2], ~w[3]);
    csa(fA, pl[1], pl[1], a, b);
    csa(a, pl[0], pl[0], ~w[4], ~w[5]);
    csa(b, pl[0], pl[0], ~w[6], ~w[7]);
    csa(fB, pl[1], pl[1], a, b);
    csa(c8[g], pl[2], pl[2], fA, fB);
  }
  uint32_t cy;
  int k = 3;
  if constexpr (kWbRows == 16) {
    csa(cy, pl[3], pl[3], c8[0], c8[1]);
    k = 4;
  } else {
    cy = c8[0];
  }
#pragma unroll
  for (; k < 8; ++k) {
    const uint32_t t = pl[k] & cy;
    pl[k] ^= cy;
    cy = t;
  }
}

// A6/A7 fused (bitmap mode): per part block, count and sum from the
// transposed rows as loaded, then transpose in registers, invert to prime
// words and store them back (natural layout) -- no second pass over the
// segment.  Input row b (bit n) of block B is natural word n (bit b), slot
// 1024 B + 32 n + b, so over the prime bits
//   sum of slots = 1024 sum_B B C_B + 32 sum_n n c_n + sum_b b r_b
// with r_b = 32 - popc(row b) (a POPC per row, also giving C_B) and c_n =
// 32 - popc(natural word n) (a POPC per transposed word), each lane adding
// its part.  The words go to HBM by TMA bulk copies (cp.async.bulk): with
// SIEVE_WB_WARP_COPY each warp sends its 32 / L consecutive blocks as soon
// as its lanes have stored them, so the copies drain while the other warps
// transpose; otherwise one copy per segment after a block barrier.  Words
// past the 16-byte bulk prefix (and every word of an output that is not
// 16-byte aligned) are stored from shared memory after a barrier.
// kSum = false (kFlagNoSum: sieve_bitmap, option bitmap_count_only): the
// count alone, from carry-save planes of the prime words (no POPC per word).
template <bool kSum>
__device__ __forceinline__ void writeback_fused(uint32_t *seg, uint64_t a, uint64_t bit0, uint32_t valid,
                                                uint32_t *out, uint64_t out_words, uint32_t vec4,
                                                unsigned long long &cnt, unsigned long long &sum) {
  const uint32_t nblk = (valid + 1023u) >> 10;
  const uint32_t lane = threadIdx.x & 31u, u = lane & (kWbLanes - 1u);
  const uint64_t w0 = bit0 >> 5;
  const uint32_t nq = (valid + 127u) >> 7;
  const uint32_t nw = out_words > w0 ? (uint32_t)min((uint64_t)4u * nq, out_words - w0) : 0u;
  const uint32_t n16 = (SIEVE_TMA_STORE && vec4) ? (nw & ~3u) : 0u;
  // composite bits, sum of (row) x popc(row), sum of (word) x popc(word), sum of B x (prime bits)
  uint32_t comp = 0, wrow = 0, wnat = 0, bc = 0, np = 0;
  uint32_t pl[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // kSum = false: planes of the prime words
  for (uint32_t P0 = threadIdx.x & ~31u; P0 < kWbLanes * nblk; P0 += blockDim.x) {
    const bool own = (P0 + lane) / kWbLanes < nblk;
    const uint32_t B = min((P0 + lane) / kWbLanes, nblk - 1u);  // tail lanes redo the last block, uncounted
    const uint32_t qa = part_block_addr(seg, B, u);
    const uint32_t t4 = 4u * (B & (kWbQuads - 1u)) + kWbRows * u;  // index of register 4q + e: (t4 ^ 4q) + e
    uint32_t A[kWbRows];
    load_part_block(qa, A);
    uint32_t cb = 0, wr = 0;
#pragma unroll
    for (int q = 0; q < (int)kWbQuads && kSum; ++q) {  // register 4q + e = row (t4 ^ 4q) + e
      const uint32_t c0 = __popc(A[4 * q]), c1 = __popc(A[4 * q + 1]), c2 = __popc(A[4 * q + 2]),
                     c3 = __popc(A[4 * q + 3]);
      const uint32_t cq = c0 + c1 + c2 + c3;
      cb += cq;
      wr += (t4 ^ (4u * q)) * cq + c1 + 2u * c2 + 3u * c3;
    }
    if (SIEVE_WB_DIAG != 3) transpose_part_block(B, u, A);
    uint32_t wn = 0;
#pragma unroll
    for (int q = 0; q < (int)kWbQuads && kSum; ++q) {  // register 4q + e = natural word (t4 ^ 4q) + e
      const uint32_t c1 = __popc(A[4 * q + 1]), c2 = __popc(A[4 * q + 2]), c3 = __popc(A[4 * q + 3]);
      wn += (t4 ^ (4u * q)) * (__popc(A[4 * q]) + c1 + c2 + c3) + c1 + 2u * c2 + 3u * c3;
    }
    if (!kSum && own) planes_add(pl, A);
    if (kSum && own) {
      comp += cb;
      wrow += wr;
      wnat += wn;
      bc += B * (32u * kWbRows - cb);
      ++np;
    }
    __syncwarp();  // every lane's loads before a duplicate of the last block is stored
    if (own) store_part_block<true>(qa, A);
#if SIEVE_WB_WARP_COPY
    const uint32_t wa = 32u * (P0 / kWbLanes);  // first word of the warp's blocks
    if (n16 > wa) {
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0 && SIEVE_WB_DIAG != 2)
        bulk_store(out + w0 + wa, seg + wa, 4u * min(32u * 32u / kWbLanes, n16 - wa));
    }
#endif
  }
#if !SIEVE_WB_WARP_COPY
  if (n16) fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0 && n16 && SIEVE_WB_DIAG != 2) bulk_store(out + w0, seg, 4u * n16);
#else
  if (n16 < nw) __syncthreads();
#endif
  for (uint32_t w = n16 + threadIdx.x; w < nw; w += blockDim.x) {
    SV_CHECK(w0 + w < out_words, kVioBitmapStore);
    out[w0 + w] = seg[w];
  }
  if (kSum) {
    // per part: kWbRows rows / words of 32 bits with indices R u .. R u + R - 1
    const uint32_t C = 32u * kWbRows * np - comp;
    const uint64_t full = 32ull * (kWbRows * kWbRows * u + kWbRows * (kWbRows - 1u) / 2u) * np;
    const uint64_t J = 1024ull * bc + 32ull * (full - wnat) + (full - wrow);
    cnt += C;
    sum += (unsigned long long)C * a + 2ull * J;
  } else {
    uint32_t C = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) C += (uint32_t)__popc(pl[k]) << k;
    cnt += C;
  }
#if SIEVE_WB_DIAG == 0
  if (SIEVE_WB_WARP_COPY ? lane == 0 : threadIdx.x == 0) bulk_wait_read();
#endif
}

constexpr uint64_t kFlagAgg = 1, kFlagIncl = 2;  // look-back flag states (A2 K1, A8 list)

// A8 (list mode): the primes of one segment (natural layout, after
// untranspose) written to the list in order.  Warp w owns a contiguous range
// of the segment's words; pass 1 counts its primes; thread 0 publishes the
// segment's count, finds the segment's place in the list by a decoupled
// look-back over the earlier segments, and publishes its inclusive prefix;
// pass 2 has the lanes of a warp take 32 x SIEVE_LIST_WORDS consecutive words at a time, place
// them by a warp scan of their popcounts, and write their primes.  Returns
// the segment's count in thread 0 (0 elsewhere).
__device__ __forceinline__ uint64_t list_emit(const uint32_t *seg, uint64_t s, uint64_t a,
                                              uint32_t valid, const SieveParams &P, uint32_t *s_wc,
                                              unsigned long long *s_off) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t nwords = (valid + 31u) >> 5;
  const uint32_t wb = warp * nwords / nw, we = (warp + 1u) * nwords / nw;
  uint32_t c = 0;
  for (uint32_t w = wb + lane; w < we; w += 32u) c += __popc(~seg[w]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) s_wc[warp] = c;
  __syncthreads();
  if (warp == 0) {
    // segment total and exclusive warp offsets (lane 0), then the decoupled
    // look-back by the whole warp: 32 predecessor flags per step, the
    // nearest inclusive one found by a ballot, the aggregates before it
    // summed by a warp reduction (a one-thread walk would read up to a wave
    // of flags one L2 round trip at a time)
    volatile unsigned long long *fl = P.lflags;
    const unsigned long long tag = (unsigned long long)P.lepoch << 48;
    uint32_t t = 0;
    if (lane == 0) {
      for (uint32_t k = 0; k < nw; ++k) {
        const uint32_t x = s_wc[k];
        s_wc[k] = t;  // exclusive warp offsets
        t += x;
      }
      s_wc[32] = t;
      if (s == 0) {
        const unsigned long long pre0 = P.add_two ? 1ull : 0ull;  // list[0] = 2
        fl[0] = tag | ((pre0 + t) << 2) | kFlagIncl;
        *s_off = pre0;
        if (P.add_two && P.list_cap > 0) P.list[0] = 2;
      } else {
        fl[s] = tag | ((unsigned long long)t << 2) | kFlagAgg;
      }
    }
    if (s > 0) {
      unsigned long long pre = 0;
      for (int64_t j = (int64_t)s - 1;; j -= 32) {
        const int64_t idx = j - (int64_t)lane;  // lane 0 the nearest
        unsigned long long f = 0;
        if (idx >= 0) {
          do { f = fl[idx]; } while ((f >> 48) != P.lepoch);  // not yet published in this launch
        }
        const unsigned incl = __ballot_sync(0xffffffffu, idx >= 0 && (f & 3u) == kFlagIncl);
        const uint32_t stop = incl ? (uint32_t)(__ffs(incl) - 1) : 31u;
        unsigned long long v = (idx >= 0 && lane <= stop) ? ((f >> 2) & ((1ull << 46) - 1)) : 0ull;
        pre += warp_sum_u64(v);
        if (incl) break;  // segment 0 is always inclusive: the walk ends
      }
      if (lane == 0) {
        __threadfence();
        fl[s] = tag | ((pre + s_wc[32]) << 2) | kFlagIncl;
        *s_off = pre;
      }
    }
  }
  __syncthreads();
  unsigned long long base = *s_off + s_wc[warp];
  // lane l takes kLW consecutive words per pass (one scan and one set of
  // 64-bit offsets per kLW words); their primes go out word by word
  constexpr uint32_t kLW = SIEVE_LIST_WORDS;
  static_assert(kLW >= 1 && kLW <= 4, "SIEVE_LIST_WORDS: 1 to 4");
  auto emit_direct = [&](const uint32_t w0) {
    const uint32_t w = w0 + kLW * lane;
    uint32_t xs[kLW];
    uint32_t cx = 0;
#pragma unroll
    for (uint32_t e = 0; e < kLW; ++e) {
      xs[e] = w + e < we ? ~seg[w + e] : 0u;
      cx += __popc(xs[e]);
    }
    uint32_t incl = cx;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (uint32_t)o) incl += y;
    }
    unsigned long long k = base + incl - cx;
    const uint64_t v0 = a + 64ull * w;
    if (k + cx <= P.list_cap) {  // the lane's words fit: no per-prime check
      // two primes per 16-byte store once the address is 16-byte aligned:
      // the emission is bound by the number of store instructions
      uint64_t *dst = P.list + k;
      SV_CHECK(k + cx <= P.list_cap, kVioListStore);
#pragma unroll
      for (uint32_t e = 0; e < kLW; ++e) {
        uint32_t x = xs[e];
        const uint64_t ve = v0 + 64ull * e;
        if ((reinterpret_cast<uintptr_t>(dst) & 8u) && x) {
          *dst++ = ve + 2ull * (uint32_t)(__ffs(x) - 1);
          x &= x - 1;
        }
        while (x) {
          const uint32_t b1 = __ffs(x) - 1;
          x &= x - 1;
          if (x) {
            const uint32_t b2 = __ffs(x) - 1;
            x &= x - 1;
            SV_CHECK(dst + 2 <= P.list + P.list_cap && ((uintptr_t)dst & 15u) == 0, kVioListStore);
            *reinterpret_cast<ulonglong2 *>(dst) = make_ulonglong2(ve + 2ull * b1, ve + 2ull * b2);
            dst += 2;
          } else {
            *dst++ = ve + 2ull * b1;
          }
        }
      }
    } else {
#pragma unroll
      for (uint32_t e = 0; e < kLW; ++e) {
        uint32_t x = xs[e];
        while (x) {
          const uint32_t b = __ffs(x) - 1;
          x &= x - 1;
          if (k < P.list_cap) P.list[k] = v0 + 64ull * e + 2ull * b;
          ++k;
        }
      }
    }
    base += __shfl_sync(0xffffffffu, incl, 31);
  };
#if SIEVE_LIST_DIAG == 1
  // diagnostics build: no pass 2 (wrong list) -- what the untranspose, the
  // count pass and the look-back cost without the emission
#elif SIEVE_LIST_STAGE
  // Staged passes (internal.h SIEVE_LIST_STAGE): lane l takes kSW consecutive
  // words of a pass of 32 kSW; one warp scan per pass; the lanes drop the
  // 16-bit slot numbers of their primes (slot within the pass) in list order
  // into the bytes of the warp's words already consumed -- up to a pass
  // before this one and, once every lane holds its words in registers, this
  // pass's own: 4 bytes per word, room for two primes per word -- and the warp
  // then writes the pass's primes in order, two per lane and 16-byte store.
  // The warp's first pass, a pass too dense for that room and a list that
  // would overflow take the direct path.
  static_assert(kLW == 1, "SIEVE_LIST_STAGE needs SIEVE_LIST_WORDS = 1");
  constexpr uint32_t kSW = SIEVE_LIST_STAGE, kPW = 32u * kSW;
  static_assert(kSW >= 2 && kSW <= 8, "SIEVE_LIST_STAGE: 2 to 8 words per lane");
  uint32_t w0 = wb;
  // direct until half a pass of the warp's words is consumed: with the
  // pass's own words that is room for 3 primes per 2 words of the pass
  for (; w0 < we && w0 < wb + kPW / 2u; w0 += 32u) emit_direct(w0);
  for (; w0 < we; w0 += kPW) {
    const uint32_t wl = w0 + kSW * lane;
    uint32_t xs[kSW];
    uint32_t cx = 0;
#pragma unroll
    for (uint32_t e = 0; e < kSW; ++e) {
      xs[e] = wl + e < we ? ~seg[wl + e] : 0u;
      cx += __popc(xs[e]);
    }
    uint32_t incl = cx;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (uint32_t)o) incl += y;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    __syncwarp();  // every lane holds its words: the pass's bytes are free
    uint32_t st0 = w0 - wb >= kPW ? w0 - kPW : wb;             // first word of the staging area
#if SIEVE_LIST_QUAD
    st0 += st0 & 1u;  // 8-byte aligned (the segment is 128-byte aligned)
#endif
    const uint32_t room = 2u * (min(w0 + kPW, we) - st0);      // 16-bit entries
    const uint32_t head = (uint32_t)(reinterpret_cast<uintptr_t>(P.list + base) >> 3) & 1u;
#if SIEVE_LIST_QUAD
    // four entries per lane and step of the ordered write (one 8-byte load,
    // two 16-byte stores): the odd first prime sits at entry 3, so that the
    // aligned part starts at entry 4 (8-byte aligned in the staging area)
    const uint32_t off = 3u * head;
#else
    const uint32_t off = head;
#endif
    if (off + tot <= room && base + tot <= P.list_cap) {
      // the staging area is shared memory reinterpreted as 16-bit entries
      unsigned short *st = reinterpret_cast<unsigned short *>(const_cast<uint32_t *>(seg) + st0);
      unsigned short *q = st + off + (incl - cx);
#pragma unroll
      for (uint32_t e = 0; e < kSW; ++e) {
        const uint32_t s16 = 32u * (kSW * lane + e);
#if SIEVE_LIST_BFIND
        // one BREV per word, then one FLO (bfind) per prime: the lowest set
        // bit of x is the highest of y, at position 31 - b (BREV and FLO
        // share the quarter-rate pipe, the loop's bound)
        uint32_t y = __brev(xs[e]);
        while (y) {
          uint32_t f;
          asm("bfind.u32 %0, %1;" : "=r"(f) : "r"(y));
          *q++ = (unsigned short)(s16 + 31u - f);
          y ^= 1u << f;
        }
#else
        uint32_t x = xs[e];
        while (x) {
          *q++ = (unsigned short)(s16 + (uint32_t)(__ffs(x) - 1));
          x &= x - 1;
        }
#endif
      }
      __syncwarp();
      const uint64_t v0 = a + 64ull * w0;  // slot 0 of the pass
      uint64_t *dst = P.list + base;       // staged entry t goes to dst[t - off]
      const uint32_t T = off + tot, t0 = off + head;  // the aligned part: entries [t0, T)
      SV_CHECK(base + tot <= P.list_cap, kVioListStore);
#if SIEVE_LIST_QUAD
      constexpr uint32_t kQ = 4;
      for (uint32_t t = t0 + kQ * lane; t + (kQ - 1u) < T; t += 32u * kQ) {
        const uint2 pr = *reinterpret_cast<const uint2 *>(st + t);
        SV_CHECK((reinterpret_cast<uintptr_t>(dst + (t - off)) & 15u) == 0, kVioListStore);
        ulonglong2 *d2 = reinterpret_cast<ulonglong2 *>(dst + (t - off));
        d2[0] = make_ulonglong2(v0 + 2ull * (pr.x & 0xFFFFu), v0 + 2ull * (pr.x >> 16));
        d2[1] = make_ulonglong2(v0 + 2ull * (pr.y & 0xFFFFu), v0 + 2ull * (pr.y >> 16));
      }
#else
      constexpr uint32_t kQ = 2;
      for (uint32_t t = t0 + kQ * lane; t + (kQ - 1u) < T; t += 32u * kQ) {
        const uint32_t pr = *reinterpret_cast<const uint32_t *>(st + t);
        SV_CHECK((reinterpret_cast<uintptr_t>(dst + (t - off)) & 15u) == 0, kVioListStore);
        *reinterpret_cast<ulonglong2 *>(dst + (t - off)) =
            make_ulonglong2(v0 + 2ull * (pr & 0xFFFFu), v0 + 2ull * (pr >> 16));
      }
#endif
      // the odd first prime and the last (T - t0) mod kQ, one lane each
      if (lane == 31u && head && tot) dst[0] = v0 + 2ull * st[off];
      if (T > t0) {
        const uint32_t rem = (T - t0) % kQ, tt = T - rem;
        if (lane < rem) dst[tt + lane - off] = v0 + 2ull * st[tt + lane];
      }
      base += tot;
    } else {
      for (uint32_t u = w0; u < we && u < w0 + kPW; u += 32u) emit_direct(u);
    }
  }
#else
  for (uint32_t w0 = wb; w0 < we; w0 += 32u * kLW) emit_direct(w0);
#endif
  const uint64_t tot = s_wc[32];
  __syncthreads();  // s_wc is reused by the next segment
  return threadIdx.x == 0 ? tot : 0ull;  // counted once per CTA
}

// block-wide sum of two u64 values; result valid in thread 0
__device__ __forceinline__ void block_sum2(unsigned long long &x, unsigned long long &y,
                                           unsigned long long *red) {
  x = warp_sum_u64(x);
  y = warp_sum_u64(y);
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) { red[warp] = x; red[32 + warp] = y; }
  __syncthreads();
  if (warp == 0) {
    x = lane < nw ? red[lane] : 0ull;
    y = lane < nw ? red[32 + lane] : 0ull;
    x = warp_sum_u64(x);
    y = warp_sum_u64(y);
  }
}

// ---------------------------------------------------------------------------
// A2 building blocks shared by the base-prime kernel K1 and its fused form
// in the sieve kernel (base_phase): odd n = 2i + 1, bit b of a word <-> i = I + b.
// ---------------------------------------------------------------------------
constexpr int kNumPat = 10;  // pattern primes 3..31
constexpr uint32_t kMaxSmall = 1024;  // odd primes <= 4096 number 563
// bits (q - 3) / 2 of the odd numbers from 3 (i = 1 at bit 0): the pattern
// primes themselves, and (kSelfMini) also the mini-sieve primes 37..61
constexpr uint32_t kSelfPat = (1u << 0) | (1u << 1) | (1u << 2) | (1u << 4) | (1u << 5) |
                              (1u << 7) | (1u << 8) | (1u << 10) | (1u << 13) | (1u << 14);
constexpr uint32_t kSelfMini = kSelfPat | (1u << 17) | (1u << 19) | (1u << 20) | (1u << 22) |
                               (1u << 25) | (1u << 28) | (1u << 29);

// bit b of the result is set iff 2(I + b) + 1 is an odd multiple of a pattern
// prime 3..31: for q, the bits b = ((q-1)/2 - I) mod q + k q
__device__ __forceinline__ uint32_t pattern_word(uint32_t I) {
  constexpr uint32_t kQ[kNumPat] = {3, 5, 7, 11, 13, 17, 19, 23, 29, 31};
  uint32_t v = 0;
#pragma unroll
  for (int k = 0; k < kNumPat; ++k) {
    const uint32_t q = kQ[k], h = (q - 1u) / 2u;
    uint32_t pat = 0;  // bits 0, q, 2q, ... < 32 (constant-folded)
    for (uint32_t b = 0; b < 32u; b += q) pat |= 1u << b;
    const uint32_t t = I % q;
    const uint32_t f = h >= t ? h - t : h + q - t;
    v |= pat << f;
  }
  return v;
}

// The odd primes 3 <= q <= rs (rs <= 4096), ascending, into sp[]: a
// mini-sieve of i = 1..2047 by the primes <= 61 (warps 0 and 1, one word per
// thread) and an ordered compaction.  Called by the whole CTA (>= 64
// threads); stage needs 128 words; returns the count (all threads).
__device__ __forceinline__ uint32_t small_primes(uint32_t rs, uint32_t *sp, uint32_t *stage,
                                                 uint32_t *s_w2) {
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  if (warp < 2u) {
    const uint32_t I = 1u + 32u * tid;  // first i of word tid
    uint32_t v = pattern_word(I);
    constexpr uint32_t big[7] = {37, 41, 43, 47, 53, 59, 61};  // at most one multiple per word
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      const uint32_t q = big[k], h = (q - 1u) / 2u, t = I % q;
      const uint32_t f = h >= t ? h - t : h + q - t;
      if (f < 32u) v |= 1u << f;
    }
    if (tid == 0) v &= ~kSelfMini;
    uint32_t x = ~v;
    const uint32_t imax_s = rs >= 3u ? (rs - 1u) / 2u : 0u;  // keep n = 2i + 1 <= rs
    if (I > imax_s) x = 0;
    else if (imax_s - I < 31u) x &= (2u << (imax_s - I)) - 1u;
    const uint32_t c = __popc(x);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (uint32_t)o) incl += y;
    }
    if (lane == 31u) s_w2[warp] = incl;
    stage[tid] = x;
    stage[64u + tid] = incl - c;
  }
  __syncthreads();
  if (warp < 2u) {
    uint32_t x = stage[tid], o = stage[64u + tid] + (warp ? s_w2[0] : 0u);
    while (x) {
      const uint32_t b = __ffs(x) - 1u;
      x &= x - 1u;
      if (o < kMaxSmall) sp[o] = 2u * (1u + 32u * tid + b) + 1u;
      ++o;
    }
  }
  __syncthreads();
  return min(s_w2[0] + s_w2[1], kMaxSmall);
}

// Mark the odd multiples >= q^2 of the small primes q = sp[m31..nsp) > 31 in
// the slice bitmap bm (bit j <-> odd a + 2j, nbits bits): one warp per prime,
// lanes on consecutive hits.  sp ascending: per warp, q^2 >= e ends the loop.
__device__ __forceinline__ void mark_slice(uint32_t *bm, const uint32_t *sp, uint32_t m31,
                                           uint32_t nsp, uint32_t a, uint32_t nbits) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t e = a + 2u * nbits;
  for (uint32_t m = m31 + warp; m < nsp; m += nw) {
    const uint32_t q = sp[m];
    uint32_t f = q * q;
    if (f >= e) break;
    if (f < a) {
      f = ((a + q - 1u) / q) * q;
      if (!(f & 1u)) f += q;
    }
    for (uint32_t j = (f - a) / 2u + lane * q; j < nbits; j += 32u * q)
      atomicOr(&bm[j >> 5], 1u << (j & 31));
  }
}

// First index with v[idx] > x, by one warp: 32-ary search (each round the
// 32 lanes sample 32 evenly spaced entries; a ballot of "<= x" narrows the
// interval 32-fold), so a search over 2^18 primes costs ~4 dependent loads.
__device__ __forceinline__ uint32_t warp_upper_bound(const uint32_t *v, uint32_t n, uint64_t x) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t lo = 0, hi = n;  // answer in [lo, hi]
  while (hi - lo > 32u) {
    const uint32_t step = (hi - lo + 31u) / 32u;
    const uint32_t idx = lo + lane * step;
    const bool le = idx < hi && (uint64_t)__ldg(v + idx) <= x;
    const uint32_t c = __popc(__ballot_sync(0xffffffffu, le));  // sampled prefix <= x
    if (c == 0) return lo;
    const uint32_t nlo = lo + (c - 1u) * step + 1u;
    hi = min(hi, lo + c * step);
    lo = nlo;
  }
  const uint32_t idx = lo + lane;
  const bool le = idx < hi && (uint64_t)__ldg(v + idx) <= x;
  return lo + __popc(__ballot_sync(0xffffffffu, le));
}

// Region boundaries (indices into primes[]): warps 0..3 search in parallel,
// then thread 0 clamps.  Must be called by the whole CTA (contains a barrier
// before the clamp; the caller syncs after).
__device__ __forceinline__ void compute_regions(const SieveParams &P, uint32_t r, PrimeRegions &R,
                                                uint32_t *scratch, uint32_t ng_start,
                                                bool only_end) {
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t nb = *P.nbase;
  if (warp < (only_end ? 1u : 7u)) {
    const uint64_t x = warp == 0 ? (uint64_t)r
                     : warp == 1 ? P.seg_bits / kUnitHits
                     : warp == 2 ? P.seg_bits / kClassHits
                     : warp == 3 ? P.seg_bits / kWarpHits
                     : warp == 4 ? (P.buckets ? P.seg_bits / kBucketHits : ~0ull)
                     : warp == 5 ? P.seg_bits / kC15Hits
                     : P.seg_bits / kPlainHits;
    const uint32_t u = warp_upper_bound(P.primes, nb, x);
    if ((threadIdx.x & 31u) == 0) scratch[warp] = u;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    R.end = scratch[0];
    R.start = min(ng_start, R.end);
    R.unit = max(R.start, min(R.end, scratch[1]));
    R.cls = max(R.unit, min(R.end, scratch[2]));
    R.warp = max(R.cls, min(R.end, scratch[3]));
    R.big = max(R.warp, min(R.end, scratch[4]));
    R.few = max(R.warp, min(R.big, scratch[5]));
    R.two = max(R.few, min(R.big, scratch[6]));
  }
}

// Grid-wide barrier of a cooperative launch: thread 0 of each CTA arrives
// on *bar and waits for `target` arrivals (the counter only grows within a
// launch: the n-th barrier waits for n * gridDim.x).
// Split-phase grid barrier of a cooperative launch: arrive (thread 0 of
// each CTA counts in on *bar after the CTA's writes), do independent work,
// then wait for `target` arrivals (the counter only grows within a launch:
// the n-th barrier waits for n * gridDim.x).
__device__ __forceinline__ void grid_arrive(unsigned int *bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
  }
}
__device__ __forceinline__ void grid_wait(unsigned int *bar, unsigned int target) {
  if (threadIdx.x == 0) {
    unsigned int v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if (v >= target) break;
      __nanosleep(32);
    }
  }
  __syncthreads();
}

// Fused A2 (the base-prime kernel's work inside the sieve kernel, before the
// first segment): CTA c sieves slice c of the odd numbers 3..r (L bits,
// L = ceil(imax / G) rounded up to 32; the host checks that the small
// primes, the slice bitmap and its staged primes fit in the segment buffer
// below the wheel tables, used here as scratch), counts its
// primes and publishes the count; after a grid barrier it places them by the
// counts of the slices before it and writes primes and reciprocals; a second
// grid barrier makes the whole list visible before any CTA reads it.  Both
// barriers are split (arrive ... wait): the staging and reciprocals run
// while the other CTAs arrive at the first, and the caller initialises its
// first segment (wheel) between arrive and wait of the second.
__device__ __forceinline__ void base_phase(const SieveParams &P, uint32_t *seg) {
  __shared__ uint32_t s_w[32];
  __shared__ unsigned long long s_base;  // this slice's first list index
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5, nw = blockDim.x >> 5;
  const uint32_t G = gridDim.x;
  uint32_t *sp = seg;                   // [kMaxSmall]
  uint32_t *bm = seg + kMaxSmall + 128u;  // slice bitmap
  const uint32_t nsp = small_primes(P.rs, sp, seg + kMaxSmall, s_w);
  const uint32_t m31 = min(nsp, (uint32_t)kNumPat);
  const uint32_t imax = P.r >= 3u ? (P.r - 1u) / 2u : 0u;
  const uint32_t L = ((imax + G - 1u) / G + 31u) & ~31u;
  const uint32_t i0 = 1u + blockIdx.x * L;
  const uint32_t nbits = i0 <= imax ? min(L, imax - i0 + 1u) : 0u;
  const uint32_t nwd = (nbits + 31u) >> 5;
  const uint32_t a = 2u * i0 + 1u;
  SV_CHECK(4u * nwd + (uint32_t)__cvta_generic_to_shared(bm) <= s_chk_hi, kVioScratch);  // fused_fits
  for (uint32_t w = tid; w < nwd; w += blockDim.x) {
    uint32_t v = pattern_word(i0 + 32u * w);
    if (blockIdx.x == 0 && w == 0) v &= ~kSelfPat;  // 3..31 are prime
    bm[w] = v;
  }
  __syncthreads();
  mark_slice(bm, sp, m31, nsp, a, nbits);
  __syncthreads();
  // survivors of word w (primes = clear bits below nbits)
  auto word = [&](uint32_t w) {
    uint32_t x = ~bm[w];
    const uint32_t vb = nbits - 32u * w;
    if (vb < 32u) x &= (1u << vb) - 1u;
    return x;
  };
  uint32_t c = 0;
  for (uint32_t w = tid; w < nwd; w += blockDim.x) c += __popc(word(w));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) s_w[warp] = c;
  __syncthreads();
  if (tid == 0) {
    uint32_t t = 0;
    for (uint32_t k = 0; k < nw; ++k) t += s_w[k];
    P.bcounts[blockIdx.x] = t;
    if (P.prof) atomicMax(P.prof + 110, global_ns());
  }
  grid_arrive(P.gbar);
  // while the other CTAs arrive: the slice's primes staged in order (a block
  // scan per row of blockDim.x words) and the first two per thread with
  // their reciprocals in registers
  uint32_t *stage = bm + nwd;  // <= nbits / 3 + 2 entries (host-checked space)
  uint32_t o = 0;
  for (uint32_t w0 = 0; w0 < nwd; w0 += blockDim.x) {
    const uint32_t w = w0 + tid;
    uint32_t x = w < nwd ? word(w) : 0u;
    const uint32_t cw = __popc(x);
    uint32_t incl = cw;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= (uint32_t)d) incl += y;
    }
    __syncthreads();  // s_w reuse
    if (lane == 31u) s_w[warp] = incl;
    __syncthreads();
    uint32_t excl = incl - cw, row = 0;
    for (uint32_t k = 0; k < nw; ++k) {
      if (k < warp) excl += s_w[k];
      row += s_w[k];
    }
    uint32_t q = o + excl;
    while (x) {
      const uint32_t b = __ffs(x) - 1u;
      x &= x - 1u;
      SV_CHECK(4u * q + (uint32_t)__cvta_generic_to_shared(stage) < s_chk_hi, kVioScratch);
      stage[q++] = a + 2u * (32u * w + b);
    }
    o += row;
  }
  __syncthreads();
  const uint32_t t1 = tid + blockDim.x;
  const uint32_t p0 = tid < o ? stage[tid] : 3u, p1 = t1 < o ? stage[t1] : 3u;
  const uint64_t q0 = recip_of(p0), q1 = recip_of(p1);
  grid_wait(P.gbar, G);
  if (P.prof && tid == 0) atomicMax(P.prof + 111, global_ns());
  if (warp == 0) {  // this slice's offset and the total
    unsigned long long before = 0, all = 0;
    for (uint32_t k = lane; k < G; k += 32u) {
      const unsigned long long v = __ldcg(P.bcounts + k);
      all += v;
      if (k < blockIdx.x) before += v;
    }
    before = warp_sum_u64(before);
    all = warp_sum_u64(all);
    if (lane == 0) {
      s_base = before;
      if (blockIdx.x == 0) *P.bnbase = (uint32_t)min(all, (unsigned long long)P.bcap);
    }
    // the region boundaries of compute_regions (first index with a prime
    // > x = number of odd primes <= x), published by the slice holding x;
    // P.bcounts[G + k], k = 1 unit, 2 class, 3 warp, 4 bucket, 5 few, 6 two
    unsigned int *reg = P.bcounts + G;
#pragma unroll
    for (uint32_t k = 1; k < 7u; ++k) {
      const uint64_t x = k == 1u ? P.seg_bits / kUnitHits
                       : k == 2u ? P.seg_bits / kClassHits
                       : k == 3u ? P.seg_bits / kWarpHits
                       : k == 4u ? (P.buckets ? P.seg_bits / kBucketHits : ~0ull)
                       : k == 5u ? P.seg_bits / kC15Hits
                       : P.seg_bits / kPlainHits;
      const uint64_t ix = x >= 3u ? (x - 1u) / 2u : 0u;  // largest i with 2i + 1 <= x
      if (ix == 0 || ix > imax) {  // below 3, or past r: 0 or every prime
        if (blockIdx.x == 0 && lane == 0) reg[k] = ix == 0 ? 0u : (uint32_t)all;
        continue;
      }
      if (ix < i0 || ix >= (uint64_t)i0 + nbits) continue;  // another slice's
      const uint32_t last = (uint32_t)(ix - i0);               // bits 0 .. last count
      uint32_t cnt = 0;
      for (uint32_t w = lane; w <= last / 32u; w += 32u) {
        uint32_t xw = word(w);
        if (w == last / 32u && (last & 31u) != 31u) xw &= (2u << (last & 31u)) - 1u;
        cnt += __popc(xw);
      }
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o2);
      if (lane == 0) reg[k] = (uint32_t)before + cnt;
    }
  }
  __syncthreads();
  const unsigned long long base = s_base;
  // the plain pass's packed table (kPlain kernels): {p, floor(2^44 / p)}, k_pack44's rule
  auto pack44 = [](uint32_t p, uint64_t q) { return make_uint2(p, p > 4096u ? (uint32_t)(q >> 20) : 0u); };
  if (tid < o && base + tid < P.bcap) {
    P.bprimes[base + tid] = p0;
    P.brecips[base + tid] = q0;
    if (P.pk44) P.pk44[base + tid] = pack44(p0, q0);
  }
  if (t1 < o && base + t1 < P.bcap) {
    P.bprimes[base + t1] = p1;
    P.brecips[base + t1] = q1;
    if (P.pk44) P.pk44[base + t1] = pack44(p1, q1);
  }
  for (uint32_t t = t1 + blockDim.x; t < o; t += blockDim.x) {  // large r only
    if (base + t < P.bcap) {
      const uint32_t p = stage[t];
      const uint64_t q = recip_of(p);
      P.bprimes[base + t] = p;
      P.brecips[base + t] = q;
      if (P.pk44) P.pk44[base + t] = pack44(p, q);
    }
  }
  if (P.prof && tid == 0) atomicMax(P.prof + 117, global_ns());
  grid_arrive(P.gbar);  // the caller does independent work, then grid_wait(2 G)
}

// ---------------------------------------------------------------------------
// The segmented sieve kernel.  Persistent CTAs walk the segments round robin;
// each segment lives in shared memory for its whole life (init -> mark ->
// count/write-back), so nothing but the bitmap (bitmap mode) and 16 bytes per
// CTA ever reach HBM.
// ---------------------------------------------------------------------------
// kPlain: the plain-prime pass of the batch kernel (primes with at most
// kPlainHits hits per segment: clamp-free first hits, several per thread and
// pass) compiled into the count, bitmap and list kernels too, chosen at
// launch when such primes exist (r > S / kPlainHits: config 4) -- a separate
// instantiation, so that the kernels of small r (config 3) keep their code
// generation.  Config 4: 1.931 -> 1.751 ms (same-box A/B).
template <int NG, int MODE, bool kPlain = false>
__global__ void __launch_bounds__(SIEVE_MAX_THREADS, 1) k_sieve(const SieveParams P) {
  extern __shared__ __align__(16) uint32_t smem[];
  constexpr int kWheelUnrollOf = MODE == kCount ? kWheelUnroll : 1;
  // segment at the first 128-byte boundary of the dynamic shared memory (the
  // runtime allocates kSmemAlign spare bytes), wheel tables after it
  const uint32_t sraw = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t sb = (sraw + (kSmemAlign - 1u)) & ~(kSmemAlign - 1u);
  uint32_t *seg = smem + (sb - sraw) / 4u;
  uint32_t *tab = seg + P.seg_bits / 32;
#if SIEVE_CHECK_BOUNDS
  if (threadIdx.x == 0) {
    s_chk_lo = sb;
    s_chk_hi = sb + P.seg_bits / 8u;  // S odd slots = S / 32 words
  }
  __syncthreads();
#endif
  __shared__ unsigned long long red[64];
  __shared__ PrimeRegions sR;
  __shared__ uint32_t s_last;
  __shared__ uint32_t s_ub[7];
  __shared__ uint32_t s_wc[33];            // list mode: warp counts / offsets, segment total
  __shared__ unsigned long long s_off;     // list mode: the segment's place in the list

  // diagnostics timeline (P.prof[104..109], globaltimer ns; min as max of ~t)
  if (P.prof && threadIdx.x == 0) {
    const unsigned long long t = global_ns();
    atomicMax(P.prof + 104, ~t);
    atomicMax(P.prof + 105, t);
  }
  __shared__ uint32_t s_k15[15];  // kept15(r3, r5) at 5 r3 + r5
  if (threadIdx.x < 15u) s_k15[threadIdx.x] = kept15(threadIdx.x / 5u, threadIdx.x % 5u);
  // wheel tables to shared memory; with the fused A2, warps >= 2 copy them
  // while warps 0-1 run its mini-sieve of the small primes (small_primes
  // syncs the block before anything reads them)
  if (MODE != kBatch && P.bprimes) {
    if (threadIdx.x >= 64u)
      for (uint32_t i = threadIdx.x - 64u; i < tables_words(NG); i += blockDim.x - 64u) tab[i] = P.tables[i];
  } else {
    for (uint32_t i = threadIdx.x; i < tables_words(NG); i += blockDim.x) tab[i] = P.tables[i];
  }
  // segments round robin; with the buckets of step A5 a range is sieved in
  // contiguous runs (the buckets carry each large prime from one segment of
  // the run to the next)
  const bool buckets = MODE != kBatch && P.buckets != nullptr && !(P.flags & kFlagSkipMarking);
  const uint64_t nseg = (MODE == kBatch && P.nitems) ? (uint64_t)__ldg(P.nitems) : P.nseg;
  const uint64_t s_begin = buckets ? blockIdx.x * nseg / gridDim.x : blockIdx.x;
  const uint64_t s_end = buckets ? (blockIdx.x + 1ull) * nseg / gridDim.x : nseg;
  const uint64_t s_step = buckets ? 1u : gridDim.x;
  // fused A2: the base primes, then the first segment's wheel pattern while
  // the other CTAs finish theirs (between arrive and wait of the last barrier)
  const bool pre_init = MODE != kBatch && P.bprimes && s_begin < s_end;
  // diagnostics (kFlagReverse, bitmap mode without buckets): the CTA's
  // segments in the reverse order -- schedule invariance.  Compiled into the
  // bitmap kernel only: the count kernel's code generation is sensitive to
  // its segment loop (a same-box A/B measured +2 % with it there)
  const bool reverse = MODE == kBitmap && !buckets && (P.flags & kFlagReverse);
  if (MODE != kBatch && P.bprimes) {
    base_phase(P, seg);
    if (pre_init) {
      const uint64_t s0 = reverse ? P.nseg - 1u - s_begin : s_begin;
      const uint64_t bit0 = s0 * (uint64_t)P.seg_bits, left = P.nbits - bit0;
      wheel_init<NG, kWheelUnrollOf>(seg, tab, P.o0, bit0, left < P.seg_bits ? (uint32_t)left : P.seg_bits,
                                     P.o0 + 2ull * bit0);
    }
    grid_wait(P.gbar, 2u * gridDim.x);
    if (P.prof && threadIdx.x == 0) atomicMax(P.prof + 118, global_ns());
  }
  if (MODE != kBatch && P.bprimes) {  // fused A2 published the boundaries
    if (threadIdx.x == 0) {
      const unsigned int *reg = P.bcounts + gridDim.x;
      sR.end = __ldcg(P.bnbase);
      sR.start = min(wheel_nprimes(NG), sR.end);
      sR.unit = max(sR.start, min(sR.end, __ldcg(reg + 1)));
      sR.cls = max(sR.unit, min(sR.end, __ldcg(reg + 2)));
      sR.warp = max(sR.cls, min(sR.end, __ldcg(reg + 3)));
      sR.big = max(sR.warp, min(sR.end, __ldcg(reg + 4)));
      sR.few = max(sR.warp, min(sR.big, __ldcg(reg + 5)));
      sR.two = max(sR.few, min(sR.big, __ldcg(reg + 6)));
    }
  } else {
    compute_regions(P, P.r, sR, s_ub, wheel_nprimes(NG), false);
  }
  __syncthreads();
  if (P.prof && threadIdx.x == 0) atomicMax(P.prof + 106, global_ns());

  unsigned long long cnt = 0, sum = 0;
  uint32_t bcnt = 0;  // lane t: fill count of the warp's bucket slot t
  uint32_t bq = 0;    // ring slot of the current segment
  if (buckets && s_begin < s_end) {
    bucket_fill(P, sR, bcnt, s_begin, s_end);
    bq = (uint32_t)(s_begin % P.ring);
  }
  for (uint64_t s_it = s_begin; s_it < s_end; s_it += s_step) {
    const uint64_t s = reverse ? P.nseg - 1u - s_it : s_it;
    uint64_t a, bit0, o0;
    uint32_t valid;
    PrimeRegions Ri = sR;
    if (MODE == kBatch) {
      const BatchItem it = P.items[s];
      a = it.a; valid = it.valid; o0 = it.a; bit0 = 0;
      // the item's primes are the prefix < it.nend (k_plan_emit): clamp the
      // regions, no search and no barrier per item
      Ri.end = min(Ri.end, it.nend);
      Ri.start = min(Ri.start, Ri.end);
      Ri.unit = min(Ri.unit, Ri.end);
      Ri.cls = min(Ri.cls, Ri.end);
      Ri.warp = min(Ri.warp, Ri.end);
      Ri.few = min(Ri.few, Ri.end);
      Ri.two = min(Ri.two, Ri.end);
      Ri.big = min(Ri.big, Ri.end);
    } else {
      o0 = P.o0;
      bit0 = s * (uint64_t)P.seg_bits;
      const uint64_t left = P.nbits - bit0;
      valid = left < P.seg_bits ? (uint32_t)left : P.seg_bits;
      a = o0 + 2ull * bit0;
    }
    const long long c0 = P.prof ? clock64() : 0;
    if (!(pre_init && s_it == s_begin) && !(MODE == kBitmap && (P.flags & kFlagSkipWheel)))
      wheel_init<NG, kWheelUnrollOf>(seg, tab, o0, bit0, valid, a);
    __syncthreads();
    const long long c1 = P.prof ? clock64() : 0;
    if (!(P.flags & kFlagSkipMarking)) mark_segment<MODE == kBatch ? kPlainILP : kPlain ? kPlainILPCount : 0>(sb, P.primes, P.recips, Ri, P.flags, a, valid, P.prof, s_k15, (MODE == kBatch || kPlain) ? P.pk44 : nullptr);
    if (buckets) {
      bucket_drain(P, bcnt, sb, bq, (uint32_t)(s_end - s_it), valid);
      bq = bq + 1u == P.ring ? 0u : bq + 1u;
    }
    __syncthreads();
    const long long c2 = P.prof ? clock64() : 0;
    if (MODE == kBatch) {
      unsigned long long c = 0, sm = 0;
      epilogue<kCount>(seg, a, bit0, valid, nullptr, 0, 0, c, sm);
      block_sum2(c, sm, red);
      if (threadIdx.x == 0) {
        const uint32_t iv = P.items[s].interval;
        atomicAdd(reinterpret_cast<unsigned long long *>(P.result) + 2 * iv, c);
        atomicAdd(reinterpret_cast<unsigned long long *>(P.result) + 2 * iv + 1, sm);
      }
      __syncthreads();
    } else if (MODE == kList) {
      if (SIEVE_REG_TRANSPOSE) untranspose_reg(seg, valid);
      else untranspose(seg, valid);
      __syncthreads();
      cnt += list_emit(seg, s, a, valid, P, s_wc, &s_off);
    } else {
      if (MODE == kBitmap && SIEVE_WB_FUSED) {
        if (P.flags & kFlagNoSum) writeback_fused<false>(seg, a, bit0, valid, P.out, P.out_words, P.out_vec4, cnt, sum);
        else writeback_fused<true>(seg, a, bit0, valid, P.out, P.out_words, P.out_vec4, cnt, sum);
      } else {
        if (MODE == kBitmap) {
          if (SIEVE_WB_DIAG != 3) untranspose<true>(seg, valid);
          if (SIEVE_TMA_STORE) fence_proxy_async_smem();
          __syncthreads();
        }
        epilogue<MODE>(seg, a, bit0, valid, P.out, P.out_words, P.out_vec4, cnt, sum);
      }
      __syncthreads();
    }
    if (P.prof && threadIdx.x == 0) {  // CTA-level phase cycles (diagnostics only)
      const long long c3 = clock64();
      atomicAdd(P.prof + 0, (unsigned long long)(c1 - c0));
      atomicAdd(P.prof + 1, (unsigned long long)(c2 - c1));
      atomicAdd(P.prof + 2, (unsigned long long)(c3 - c2));
      atomicAdd(P.prof + 6, 1ull);
    }
  }
  if (MODE == kBatch) return;
  if (MODE == kBitmap && SIEVE_TMA_STORE &&
      ((SIEVE_WB_FUSED && SIEVE_WB_WARP_COPY) ? (threadIdx.x & 31u) == 0 : threadIdx.x == 0))
    bulk_wait_all();

  // per-CTA partial added into the launch's accumulator (u64 atomics: exact
  // mod 2^64, so the order does not matter); the last CTA to finish takes
  // the total and resets the accumulator for the next launch.
  if (P.prof && threadIdx.x == 0) {
    const unsigned long long t = global_ns();
    atomicMax(P.prof + 107, t);
    atomicMax(P.prof + 109, ~t);
  }
  block_sum2(cnt, sum, red);
  if (threadIdx.x == 0) {
    unsigned long long *acc = reinterpret_cast<unsigned long long *>(P.partials);
    atomicAdd(acc, cnt);
    atomicAdd(acc + 1, sum);
    __threadfence();
    const unsigned int t = atomicAdd(P.done, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last) {
    unsigned long long c = 0, sm = 0;
    if (threadIdx.x == 0) {
      __threadfence();
      unsigned long long *acc = reinterpret_cast<unsigned long long *>(P.partials);
      c = atomicExch(acc, 0ull);
      sm = atomicExch(acc + 1, 0ull);
    }
    if (threadIdx.x == 0) {
      if (P.add_two) { c += 1; sm += 2; }
      // F4: the cross-GPU all-reduce, fused (peer.cuh); sentinel on timeout
      if (MODE == kCount && P.peers) {
        const ulonglong2 t = peer_allreduce(P.peers, P.world, P.rank, P.pepoch, P.timeout_ns, c, sm);
        c = t.x;
        sm = t.y;
      }
      P.result[0] = c;
      P.result[1] = (MODE == kBitmap && (P.flags & kFlagNoSum)) ? 0ull : sm;
      *P.done = 0u;  // ready for the next launch
      if (P.gbar) *P.gbar = 0u;  // every CTA is past both grid barriers
      if (P.prof) atomicMax(P.prof + 108, global_ns());
    }
  }
}

// ---------------------------------------------------------------------------
// F3: the paper's "bidirectional" sieve of one deque by two
// workers (Alg. 1) re-expressed as a thread-block CLUSTER
// of two CTAs (two SMs) sieving one super-segment of 2 S slots: CTA rank r
// holds half r (its own shared-memory segment, as in k_sieve).  Small and
// medium primes (regions A, B) are marked by each CTA in its own half.  The
// large primes (region C, lane per prime) are split between the two CTAs and
// each is walked ONCE over the whole super-segment: one first-hit reduction
// per prime and super-segment instead of per segment, and walks twice as
// long; a hit in the partner's half is a distributed-shared-memory atomic
// (mapa + red.shared::cluster).  Two cluster barriers per super-segment: both
// halves initialised before any mark, every mark (local and remote) done
// before either epilogue.  Count mode only, base primes from K1; a
// diagnostics variant for the A/B of DESIGN.md (kFlagCluster), not the
// product path: DSMEM atomics run at a fraction of local ones
// (profiles/r01_micro_pipes.json), which this kernel measures in context.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// OR into the partner CTA's segment at the same shared-window offset
__device__ __forceinline__ void red_or_remote(uint32_t saddr, uint32_t rank, uint32_t mask) {
#if SIEVE_CHECK_BOUNDS
  SV_CHECK(saddr >= s_chk_lo && saddr < s_chk_hi && __popc(mask) == 1, kVioSmemMark);
#endif
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(saddr), "r"(rank));
  asm volatile("red.shared::cluster.or.b32 [%0], %1;" ::"r"(ra), "r"(mask) : "memory");
}

template <int NG>
__global__ void __launch_bounds__(SIEVE_MAX_THREADS, 1) k_sieve_cluster(const SieveParams P) {
  extern __shared__ __align__(16) uint32_t smem[];
  const uint32_t sraw = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t sb = (sraw + (kSmemAlign - 1u)) & ~(kSmemAlign - 1u);
  uint32_t *seg = smem + (sb - sraw) / 4u;
  uint32_t *tab = seg + P.seg_bits / 32;
  __shared__ unsigned long long red[64];
  __shared__ PrimeRegions sR;
  __shared__ uint32_t s_last;
  __shared__ uint32_t s_ub[7];
  __shared__ uint32_t s_k15[15];
#if SIEVE_CHECK_BOUNDS
  if (threadIdx.x == 0) {
    s_chk_lo = sb;
    s_chk_hi = sb + P.seg_bits / 8u;
  }
#endif
  if (threadIdx.x < 15u) s_k15[threadIdx.x] = kept15(threadIdx.x / 5u, threadIdx.x % 5u);
  for (uint32_t i = threadIdx.x; i < tables_words(NG); i += blockDim.x) tab[i] = P.tables[i];
  compute_regions(P, P.r, sR, s_ub, wheel_nprimes(NG), false);
  __syncthreads();
  const uint32_t rank = cluster_ctarank();
  const uint32_t ncl = gridDim.x >> 1, cid = blockIdx.x >> 1;
  const uint32_t S = P.seg_bits;
  const PrimeRegions R = sR;
  unsigned long long cnt = 0, sum = 0;
  for (uint64_t u = cid; 2u * u < P.nseg; u += ncl) {
    const uint64_t s = 2u * u + rank;
    auto valid_of = [&](uint64_t x) -> uint32_t {
      if (x >= P.nseg) return 0u;
      const uint64_t left = P.nbits - x * S;
      return left < S ? (uint32_t)left : S;
    };
    const uint32_t valid = valid_of(s), V = valid_of(2u * u) + valid_of(2u * u + 1u);
    const uint64_t a = P.o0 + 2ull * s * S;          // this half's first odd integer
    const uint64_t a0 = P.o0 + 4ull * u * S;         // the super-segment's
    if (valid) wheel_init<NG, 1>(seg, tab, P.o0, s * (uint64_t)S, valid, a);
    cluster_sync_all();  // both halves initialised before any mark
    if (valid) mark_segment<0>(sb, P.primes, P.recips, R, P.flags | kFlagSkipC, a, valid, nullptr, s_k15);
    // region C over the super-segment, primes split between the two CTAs:
    // cluster thread T = rank nt + t takes primes R.warp + T + 2 nt m
    {
      const uint64_t send = a0 + 2ull * V;
      const uint32_t a3 = (uint32_t)(a0 % 3u);
      const uint32_t nt = blockDim.x, T = rank * nt + threadIdx.x;
      for (uint32_t k = R.warp + T; k < R.end; k += 2u * nt) {
        const uint32_t p = __ldg(P.primes + k);
        const uint32_t j0 = first_hit(a0, send, p, __ldg(P.recips + k));
        if (j0 == kNone) break;  // p^2 past the super-segment: so for every later prime
        const uint32_t r0 = skip_residue(a3, j0, p);  // hits k = r0 (mod 3): multiples of 3
        uint32_t j1 = j0 + keep_lo(r0) * p, j2 = j0 + keep_hi(r0) * p;
        const uint32_t p3 = 3u * p;
        for (; j1 < V; j1 += p3, j2 += p3) {
          const uint32_t o1 = j1 >= S ? 1u : 0u, l1 = j1 - o1 * S;
          if (o1 == rank) red_or(sb + t_addr(l1), t_mask(l1)); else red_or_remote(sb + t_addr(l1), o1, t_mask(l1));
          if (j2 < V) {
            const uint32_t o2 = j2 >= S ? 1u : 0u, l2 = j2 - o2 * S;
            if (o2 == rank) red_or(sb + t_addr(l2), t_mask(l2)); else red_or_remote(sb + t_addr(l2), o2, t_mask(l2));
          }
        }
      }
    }
    cluster_sync_all();  // every mark of both halves done
    if (valid) epilogue<kCount>(seg, a, s * (uint64_t)S, valid, nullptr, 0, 0, cnt, sum);
    __syncthreads();
  }
  block_sum2(cnt, sum, red);
  if (threadIdx.x == 0) {
    unsigned long long *acc = reinterpret_cast<unsigned long long *>(P.partials);
    atomicAdd(acc, cnt);
    atomicAdd(acc + 1, sum);
    __threadfence();
    const unsigned int t = atomicAdd(P.done, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    unsigned long long *acc = reinterpret_cast<unsigned long long *>(P.partials);
    unsigned long long c = atomicExch(acc, 0ull), sm = atomicExch(acc + 1, 0ull);
    if (P.add_two) { c += 1; sm += 2; }
    P.result[0] = c;
    P.result[1] = sm;
    *P.done = 0u;
  }
  cluster_sync_all();  // no CTA leaves while its partner may still address its shared memory
}

// ---------------------------------------------------------------------------
// A2: base primes, the odd primes <= r (r <= 2^24), ascending, with their
// Barrett reciprocals.  The odd numbers n = 2i + 1 <= r (i >= 1) are cut into
// slices of kSliceBits; a CTA of kBaseThreads threads takes slices b, b + G,
// ... (all CTAs resident).  Latency-shaped (the kernel runs before the sieve
// on a handful of SMs, so its critical path is the step's):
//  * the odd primes q <= sqrt(r) (<= 4096) come from a 2048-bit mini-sieve by
//    the primes <= 61 (one word per thread of the first two warps), kept in
//    shared memory;
//  * per slice, thread t builds word t from the periodic patterns of the
//    primes 3..31 (a shifted constant per prime: no atomics), then one warp
//    per remaining prime q > 31 marks its odd multiples >= q^2 (lanes on
//    consecutive hits);
//  * the block counts the survivors, publishes the slice's count and finds
//    the slice's place in the list by a decoupled look-back over the earlier
//    slices (flags tagged with the launch's epoch: no reset between launches);
//  * the slice's primes are staged in shared memory in order, then written
//    with their reciprocals by all threads (coalesced, independent).
// A pattern prime q itself (bit (q - 3) / 2 of slice 0) is cleared again: the
// patterns mark every odd multiple of q, which is composite except q.
// ---------------------------------------------------------------------------
constexpr uint32_t kBaseThreads = 256;
constexpr uint32_t kSliceBits = 32u * kBaseThreads;  // one word per thread
__device__ __forceinline__ uint64_t make_flag(uint32_t epoch, uint64_t v, uint64_t st) {
  return ((uint64_t)epoch << 48) | (v << 2) | st;
}

constexpr uint32_t kMaxSlicePrimes = 2048;           // primes among 8192 odd n: <= 1899 (slice 0)
__global__ void __launch_bounds__(kBaseThreads) k_base_primes(uint32_t r, uint32_t rs, uint32_t *primes,
                                                              uint64_t *recips, uint32_t cap,
                                                              uint32_t *nbase, uint64_t *flags,
                                                              uint32_t epoch, unsigned long long *prof) {
  __shared__ uint32_t bm[kSliceBits / 32];
  __shared__ uint32_t sp[kMaxSmall];
  __shared__ uint32_t s_list[kMaxSlicePrimes];
  __shared__ uint32_t s_w[kBaseThreads / 32];
  __shared__ unsigned long long s_off;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5, nw = blockDim.x >> 5;
  // diagnostics timeline (prof[112..116], globaltimer ns; min as max of ~t)
  auto stamp = [&](int k) {
    if (prof && tid == 0) atomicMax(prof + k, k == 112 ? ~global_ns() : global_ns());
  };
  stamp(112);

  // odd primes 3 <= q <= rs (rs <= 4096), ascending
  const uint32_t nsp = small_primes(rs, sp, bm, s_w);
  // first index with sp > 31 (sp holds 3, 5, ..., 31 first when rs >= 31)
  const uint32_t m31 = min(nsp, (uint32_t)kNumPat);
  stamp(113);

  const uint32_t imax = r >= 3 ? (r - 1) / 2 : 0;
  const uint32_t nslice = (imax + kSliceBits - 1) / kSliceBits;
  for (uint32_t k = blockIdx.x; k < nslice; k += gridDim.x) {
    const uint32_t i0 = 1 + k * kSliceBits;
    const uint32_t nbits = min(kSliceBits, imax - i0 + 1);
    const uint32_t a = 2u * i0 + 1u;  // odd integers [a, a + 2 nbits)
    uint32_t v = pattern_word(i0 + 32u * tid);
    if (k == 0 && tid == 0) v &= ~kSelfPat;  // 3..31 are prime
    bm[tid] = v;
    __syncthreads();
    mark_slice(bm, sp, m31, nsp, a, nbits);
    __syncthreads();
    stamp(114);
    uint32_t x = ~bm[tid];
    const uint32_t vb = nbits > 32u * tid ? nbits - 32u * tid : 0u;  // valid bits of word tid
    if (vb < 32u) x &= (1u << vb) - 1u;
    const uint32_t c = __popc(x);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (uint32_t)o) incl += y;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    uint32_t excl = incl - c, tot = 0;
    for (uint32_t w = 0; w < nw; ++w) {
      if (w < warp) excl += s_w[w];
      tot += s_w[w];
    }
    if (tid == 0) {  // publish, then look back for the slice's offset
      volatile unsigned long long *fl = reinterpret_cast<volatile unsigned long long *>(flags);
      if (k == 0) {
        fl[0] = make_flag(epoch, tot, kFlagIncl);
        s_off = 0;
      } else {
        fl[k] = make_flag(epoch, tot, kFlagAgg);
        uint64_t pre = 0;
        for (uint32_t j = k; j-- > 0;) {
          uint64_t f;
          do { f = fl[j]; } while ((f >> 48) != epoch);  // not yet published in this launch
          pre += (f >> 2) & ((1ull << 46) - 1);
          if ((f & 3u) == kFlagIncl) break;
        }
        __threadfence();
        fl[k] = make_flag(epoch, pre + tot, kFlagIncl);
        s_off = pre;
      }
      if (k == nslice - 1) *nbase = (uint32_t)min((uint64_t)cap, (uint64_t)(s_off + tot));
    }
    // stage the slice's primes in order (tot <= kMaxSlicePrimes: see above)
    uint32_t o = excl;
    while (x) {
      const uint32_t b = __ffs(x) - 1;
      x &= x - 1;
      if (o < kMaxSlicePrimes) s_list[o] = a + 2u * (32u * tid + b);
      ++o;
    }
    __syncthreads();
    stamp(115);
    const uint64_t off = s_off;
    for (uint32_t t = tid; t < min(tot, kMaxSlicePrimes); t += blockDim.x) {
      const uint32_t p = s_list[t];
      if (off + t < cap) {
        primes[off + t] = p;
        recips[off + t] = recip_of(p);
      }
    }
    __syncthreads();  // bm, s_w and s_list are reused by the next slice
  }
  stamp(116);
  if (nslice == 0 && blockIdx.x == 0 && tid == 0) *nbase = 0;
}

__global__ void k_prepare(const uint32_t *primes, const uint32_t *nbase, uint64_t *recips,
                          uint32_t cap) {
  const uint32_t n = min(*nbase, cap);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    recips[i] = recip_of(primes[i]);
}

// ---------------------------------------------------------------------------
// A10 planning on the device (internal.h launch_batch_plan).  Three small
// kernels, no host round trip: per-interval item counts and cost classes
// (with the histogram of items per class), one CTA scanning the classes
// largest first, per-interval emission of its items at its class cursor.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t isqrt_dev(uint64_t x) {  // x < 2^53
  uint64_t r = (uint64_t)sqrt((double)x);
  while (r * r > x) --r;
  while ((r + 1) * (r + 1) <= x) ++r;
  return r;
}

struct PlanIv {  // one interval's plan
  uint64_t B;     // odd slots
  uint32_t k;     // items (0: empty or over kcap)
  uint32_t cls;   // cost class (larger = costlier)
  uint32_t r;     // isqrt(hi - 1)
  bool two, over;
};

__device__ __forceinline__ PlanIv plan_interval(uint64_t lo, uint64_t hi, uint32_t S,
                                                uint64_t width_max) {
  PlanIv v;
  v.B = hi > lo ? hi / 2 - lo / 2 : 0;
  const uint64_t k = (v.B + S - 1) / S;  // <= the runtime's kcap when hi - lo <= width_max
  v.over = hi - lo > width_max;
  v.k = v.over ? 0u : (uint32_t)k;
  v.r = hi >= 2 ? (uint32_t)isqrt_dev(hi - 1) : 0u;
  v.two = lo <= 2 && 2 < hi;
  // cost of one item: its slots plus one first-hit reduction per base prime
  const float np = v.r > 2 ? (float)v.r / __logf((float)v.r) : 1.0f;
  const float cost = 0.6f * (float)(v.k ? v.B / v.k : 0) + 20.0f * np;
  v.cls = (uint32_t)min(kPlanBuckets - 1.0f, fmaxf(0.0f, 8.0f * __log2f(fmaxf(cost, 1.0f))));
  return v;
}

__global__ void k_plan_count(const uint64_t *lo, const uint64_t *hi, uint64_t n, uint32_t S,
                             uint64_t width_max, uint32_t *hist, uint64_t *result) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const PlanIv v = plan_interval(lo[i], hi[i], S, width_max);
    if (v.k) atomicAdd(hist + v.cls, v.k);
    result[2 * i] = v.over ? ~0ull : (v.two ? 1ull : 0ull);
    result[2 * i + 1] = v.over ? ~0ull : (v.two ? 2ull : 0ull);
  }
}

// one CTA of kPlanBuckets threads: cursor[c] = items of the classes above c
__global__ void k_plan_scan(uint32_t *hist, uint32_t *cursor, uint32_t *nitems) {
  __shared__ uint32_t sh[kPlanBuckets];
  const uint32_t t = threadIdx.x;
  const uint32_t c = kPlanBuckets - 1u - t;  // descending cost
  sh[t] = hist[c];
  __syncthreads();
  for (uint32_t d = 1; d < kPlanBuckets; d <<= 1) {  // inclusive Hillis-Steele scan
    const uint32_t y = t >= d ? sh[t - d] : 0u;
    __syncthreads();
    sh[t] += y;
    __syncthreads();
  }
  cursor[c] = sh[t] - hist[c];
  if (t == kPlanBuckets - 1u) *nitems = sh[t];
  __syncthreads();
  hist[c] = 0u;  // ready for the next plan
}

__global__ void k_plan_emit(const uint64_t *lo, const uint64_t *hi, uint64_t n, uint32_t S,
                            uint64_t width_max, uint32_t *cursor, const uint32_t *__restrict__ primes,
                            const uint32_t *__restrict__ nbase, BatchItem *items) {
  const uint32_t nb = *nbase;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t l = lo[i];
    const PlanIv v = plan_interval(l, hi[i], S, width_max);
    if (!v.k) continue;
    const uint32_t pos = atomicAdd(cursor + v.cls, v.k);
    const uint32_t nend = upper_bound_u32(primes, nb, v.r);
    const uint64_t q = v.B / v.k, rem = v.B % v.k;
    uint64_t b = 0;
    for (uint32_t t = 0; t < v.k; ++t) {
      BatchItem it;
      it.a = (l | 1u) + 2 * b;
      it.valid = (uint32_t)(q + (t < rem ? 1 : 0));
      it.interval = (uint32_t)i;
      it.r = v.r;
      it.nend = nend;
      b += it.valid;
      items[pos + t] = it;
    }
  }
}

cudaError_t launch_batch_plan(const uint64_t *lo, const uint64_t *hi, uint64_t n, uint32_t S,
                              uint64_t width_max, const uint32_t *primes, const uint32_t *nbase,
                              uint32_t *scratch, BatchItem *items, uint32_t *nitems,
                              uint64_t *result, cudaStream_t s) {
  uint32_t *hist = scratch, *cursor = scratch + kPlanBuckets;
  const uint64_t blocks = (n + 255) / 256;
  const int g = (int)(blocks < 1184 ? (blocks ? blocks : 1) : 1184);
  k_plan_count<<<g, 256, 0, s>>>(lo, hi, n, S, width_max, hist, result);
  k_plan_scan<<<1, kPlanBuckets, 0, s>>>(hist, cursor, nitems);
  k_plan_emit<<<g, 256, 0, s>>>(lo, hi, n, S, width_max, cursor, primes, nbase, items);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
template <int NG, int MODE, bool kPlain = false>
static cudaError_t launch_tp(const SieveParams &p, int grid, int threads, size_t smem, cudaStream_t s) {
  if (p.bprimes) {  // fused A2: grid barriers need every CTA resident
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_sieve<NG, MODE, kPlain>, p);
  }
  k_sieve<NG, MODE, kPlain><<<grid, threads, smem, s>>>(p);
  return cudaGetLastError();
}

template <int NG, int MODE>
static cudaError_t launch_t(const SieveParams &p, int grid, int threads, size_t smem, cudaStream_t s) {
  // primes with <= kPlainHits hits per segment exist: the plain-prime pass
  // (instantiated for the default wheel only; other wheels keep the (C) loops)
  if constexpr (NG == SIEVE_PLAIN_NG && MODE != kBatch && SIEVE_COUNT_PLAIN) {
    if ((uint64_t)p.r > p.seg_bits / kPlainHits) return launch_tp<NG, MODE, true>(p, grid, threads, smem, s);
  }
  return launch_tp<NG, MODE, false>(p, grid, threads, smem, s);
}

template <int MODE>
static cudaError_t launch_m(int ng, const SieveParams &p, int grid, int threads, size_t smem,
                            cudaStream_t s) {
  switch (ng) {
    case 1: return launch_t<1, MODE>(p, grid, threads, smem, s);
    case 2: return launch_t<2, MODE>(p, grid, threads, smem, s);
    case 3: return launch_t<3, MODE>(p, grid, threads, smem, s);
    case 4: return launch_t<4, MODE>(p, grid, threads, smem, s);
    case 5: return launch_t<5, MODE>(p, grid, threads, smem, s);
    case 6: return launch_t<6, MODE>(p, grid, threads, smem, s);
    default: return cudaErrorInvalidValue;
  }
}

template <int NG>
static cudaError_t launch_cluster_t(const SieveParams &p, int grid, int threads, size_t smem, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(k_sieve_cluster<NG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(grid & ~1));
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_sieve_cluster<NG>, p);
}

cudaError_t launch_sieve_cluster(int ng, const SieveParams &p, int grid, int threads, size_t smem,
                                 cudaStream_t s) {
  switch (ng) {
    case 1: return launch_cluster_t<1>(p, grid, threads, smem, s);
    case 2: return launch_cluster_t<2>(p, grid, threads, smem, s);
    case 3: return launch_cluster_t<3>(p, grid, threads, smem, s);
    case 4: return launch_cluster_t<4>(p, grid, threads, smem, s);
    case 5: return launch_cluster_t<5>(p, grid, threads, smem, s);
    case 6: return launch_cluster_t<6>(p, grid, threads, smem, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_sieve(int ng, int mode, const SieveParams &p, int grid, int threads, size_t smem,
                         cudaStream_t s) {
  switch (mode) {
    case kCount: return launch_m<kCount>(ng, p, grid, threads, smem, s);
    case kBitmap: return launch_m<kBitmap>(ng, p, grid, threads, smem, s);
    case kBatch: return launch_m<kBatch>(ng, p, grid, threads, smem, s);
    case kList: return launch_m<kList>(ng, p, grid, threads, smem, s);
    default: return cudaErrorInvalidValue;
  }
}

template <int NG>
static cudaError_t set_attr_ng(size_t smem) {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k_sieve<NG, kCount>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
  if constexpr (NG == SIEVE_PLAIN_NG) {
    if ((e = cudaFuncSetAttribute(k_sieve<NG, kCount, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
    if ((e = cudaFuncSetAttribute(k_sieve<NG, kBitmap, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
    if ((e = cudaFuncSetAttribute(k_sieve<NG, kList, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
  }
  if ((e = cudaFuncSetAttribute(k_sieve<NG, kBitmap>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
  if ((e = cudaFuncSetAttribute(k_sieve<NG, kBatch>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
  return cudaFuncSetAttribute(k_sieve<NG, kList>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t set_sieve_smem_limits(size_t smem) {
  cudaError_t e;
  if ((e = set_attr_ng<1>(smem))) return e;
  if ((e = set_attr_ng<2>(smem))) return e;
  if ((e = set_attr_ng<3>(smem))) return e;
  if ((e = set_attr_ng<4>(smem))) return e;
  if ((e = set_attr_ng<5>(smem))) return e;
  if ((e = set_attr_ng<6>(smem))) return e;
  return cudaSuccess;
}

template <int NG, int MODE>
static int occ_t(int threads, size_t smem) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_sieve<NG, MODE>, threads, smem) != cudaSuccess)
    return 0;
  return n;
}

int sieve_max_ctas_per_sm(int ng, int mode, int threads, size_t smem) {
  (void)ng; (void)mode;
  return occ_t<4, kCount>(threads, smem);
}

cudaError_t read_violations(unsigned long long *out, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_violations, sizeof(unsigned long long) * kVioClasses);
  if (e == cudaSuccess && reset) {
    static const unsigned long long zero[kVioClasses] = {};
    e = cudaMemcpyToSymbol(g_violations, zero, sizeof zero);
  }
  return e;
}

uint32_t base_slices(uint32_t r) {
  const uint32_t imax = r >= 3 ? (r - 1) / 2 : 0;
  return (imax + kSliceBits - 1) / kSliceBits;
}

cudaError_t launch_base_primes(uint32_t r, uint32_t rs, uint32_t *primes, uint64_t *recips,
                               uint32_t cap, uint32_t *nbase, uint64_t *flags, uint32_t epoch,
                               int nsm, unsigned long long *prof, cudaStream_t s) {
  const uint32_t ns = base_slices(r);
  // all CTAs resident (the look-back waits on earlier slices): <= 4 per SM
  const uint32_t grid = ns < 4u * (uint32_t)nsm ? (ns ? ns : 1u) : 4u * (uint32_t)nsm;
  k_base_primes<<<grid, kBaseThreads, 0, s>>>(r, rs, primes, recips, cap, nbase, flags, epoch, prof);
  return cudaGetLastError();
}

// batch plain pass: pk44[i] = {p_i, floor(2^44 / p_i)} (0 for p_i < 2^12,
// where the quotient does not fit 32 bits and the packed pass is not used):
// recip = floor((2^64 - 1) / p) = floor(2^64 / p) for odd p, and floors nest
__global__ void k_pack44(const uint32_t *primes, const uint64_t *recips, const uint32_t *nbase, uint2 *pk44,
                         uint32_t cap) {
  const uint32_t n = min(*nbase, cap);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t p = primes[i];
    pk44[i] = make_uint2(p, p > 4096u ? (uint32_t)(recips[i] >> 20) : 0u);
  }
}

cudaError_t launch_pack44(const uint32_t *primes, const uint64_t *recips, const uint32_t *nbase, uint2 *pk44,
                          uint32_t cap, cudaStream_t s) {
  const int grid = (int)((cap + 255) / 256 < 1184 ? (cap + 255) / 256 : 1184);
  k_pack44<<<grid > 0 ? grid : 1, 256, 0, s>>>(primes, recips, nbase, pk44, cap);
  return cudaGetLastError();
}

cudaError_t launch_prepare(const uint32_t *primes, const uint32_t *nbase, uint64_t *recips,
                           uint32_t cap, cudaStream_t s) {
  const int grid = (int)((cap + 255) / 256 < 1184 ? (cap + 255) / 256 : 1184);
  k_prepare<<<grid > 0 ? grid : 1, 256, 0, s>>>(primes, nbase, recips, cap);
  return cudaGetLastError();
}


}  // namespace sv
