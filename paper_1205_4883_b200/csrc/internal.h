// internal.h -- shared between the kernels (kernels.cu) and the host runtime
// (runtime.cu) of libsieve.so.  Nothing here is visible through the C ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sv {

// ---------------------------------------------------------------------------
// Segment layout in shared memory: BANK-TRANSPOSED.  Bit j of a segment
// (odd slot j, integer a + 2j) lives in word T(j) = 32 (j >> 10) + (j & 31),
// at bit position (j >> 5) & 31: every 1024-slot block is a 32x32 bit matrix
// stored transposed, so the shared-memory bank of slot j is j mod 32.  For an
// odd prime p, any 32 consecutive hits j0 + k p (or 32 consecutive residue
// classes k mod 1024) then fall into 32 distinct banks: the marking atomics of
// a warp that works on one prime never conflict.
//
// Wheel pre-sieve groups (step A3).  Group g is a set of small odd primes
// whose product P_g is the period of their composite pattern on the odd-only
// grid (global odd index x <-> odd integer 2x+1).  Word table g holds, for
// y in [0, P_g), TT_g[y] bit i = pattern_g[(y + 32 i) mod P_g]: the transposed
// word of bank b in block B of a segment starting at global index X0 is
// TT_g[(X0 + 1024 B + b) mod P_g] -- ONE table load per word, whose index
// advances by a constant (mod P_g) from one word of a thread to the next.
// ---------------------------------------------------------------------------
constexpr int kMaxGroups = 6;
__host__ __device__ constexpr uint32_t group_period(int g) {
  return g == 0 ? 1155u    // 3*5*7*11
       : g == 1 ? 221u     // 13*17
       : g == 2 ? 437u     // 19*23
       : g == 3 ? 899u     // 29*31
       : g == 4 ? 1517u    // 37*41
                : 2021u;   // 43*47
}
__host__ __device__ constexpr uint32_t group_words(int g) { return group_period(g); }
__host__ __device__ constexpr uint32_t group_offset(int g) {
  return g == 0 ? 0u : group_offset(g - 1) + group_words(g - 1);
}
__host__ __device__ constexpr uint32_t tables_words(int ng) { return group_offset(ng); }
// largest prime covered by the first ng groups (the wheel bound w)
__host__ __device__ constexpr uint32_t wheel_bound(int ng) {
  return ng == 1 ? 11u : ng == 2 ? 17u : ng == 3 ? 23u : ng == 4 ? 31u : ng == 5 ? 41u : 47u;
}
// number of odd primes <= wheel_bound(ng): index of the first marking prime
__host__ __device__ constexpr uint32_t wheel_nprimes(int ng) {
  return ng == 1 ? 4u : ng == 2 ? 6u : ng == 3 ? 8u : ng == 4 ? 10u : ng == 5 ? 12u : 14u;
}
// bit n set iff n is an odd prime <= 61
constexpr uint64_t kOddPrimesBelow64 =
    (1ull << 3) | (1ull << 5) | (1ull << 7) | (1ull << 11) | (1ull << 13) | (1ull << 17) |
    (1ull << 19) | (1ull << 23) | (1ull << 29) | (1ull << 31) | (1ull << 37) | (1ull << 41) |
    (1ull << 43) | (1ull << 47) | (1ull << 53) | (1ull << 59) | (1ull << 61);

// Marking-work partition (steps A4/A5) by K = S / p, the hits of prime p in a
// full segment of S slots:
//   K >= kUnitHits            : (prime, class group) units over all warps
//   kClassHits <= K < kUnitHits: warp per prime, lanes walk residue classes
//                                mod 1024 (constant mask and stride)
//   kWarpHits <= K < kClassHits: warp per prime, lanes on consecutive hits
//   K < kWarpHits             : lane per prime
#ifndef SIEVE_UNIT_HITS
#define SIEVE_UNIT_HITS 49152  // A/B-tuned with the 3-skip (32768 -> 49152)
#endif
constexpr uint32_t kUnitHits = SIEVE_UNIT_HITS;
#ifndef SIEVE_CLASS_HITS
#define SIEVE_CLASS_HITS 28672  // A/B-tuned: 16384 -> 24576 with the 3-skip, -> 28672 with the paired (B) blocks
#endif
constexpr uint32_t kClassHits = SIEVE_CLASS_HITS;
#ifndef SIEVE_A2_PARTS
#define SIEVE_A2_PARTS 4  // A/B after the skips and w = 31: 1, 2, 4, 8, 16 -> 4 (config 3 -1.8 %)
#endif
constexpr uint32_t kA2Parts = SIEVE_A2_PARTS;  // pieces per (A2) prime (divides 32)
#ifndef SIEVE_WARP_HITS
#define SIEVE_WARP_HITS 384  // A/B-tuned: 128 -> 256 with the 3-skip (-5 %), -> 384 with w = 31 and 4 (A2) pieces (-1.3 %)
#endif
constexpr uint32_t kWarpHits = SIEVE_WARP_HITS;
// step A5: primes with fewer than kBucketHits hits per full segment (p > S /
// kBucketHits) go through per-segment buckets when enabled (option buckets)
// (C) primes with >= kC15Hits hits left in the segment also skip the
// multiples of 5 (8 kept hits per 15); fewer hits: only the multiples of 3
#ifndef SIEVE_C15_HITS
#define SIEVE_C15_HITS 32  // A/B: 16, 32, 48 -> 32
#endif
constexpr uint32_t kC15Hits = SIEVE_C15_HITS;
// (C) first hits by first_hit_scaled where the lane's largest prime has
// p^2 <= a (else first_hit with the p^2 clamp)
#ifndef SIEVE_C_SCALED
#define SIEVE_C_SCALED 1
#endif
// batch kernel: (C) primes with at most kPlainHits hits per segment are
// marked without the multiple-of-3 skip
#ifndef SIEVE_PLAIN_HITS
#define SIEVE_PLAIN_HITS 8  // A/B on config 5: 2 -> 6.49, 4 -> 6.40, 8 -> 6.34, 16 -> 6.37, 32 -> 6.40 ms
#endif
constexpr uint32_t kPlainHits = SIEVE_PLAIN_HITS;
#ifndef SIEVE_PLAIN_ILP  // batch kernel: plain primes per thread and pass
#define SIEVE_PLAIN_ILP 8  // config 5: 2 -> 5.39, 4 -> 5.13, 8 -> 5.07 ms
#endif
constexpr int kPlainILP = SIEVE_PLAIN_ILP;
#ifndef SIEVE_PLAIN_ILP_COUNT  // the same pass in the count/bitmap/list kernels of large r
#define SIEVE_PLAIN_ILP_COUNT 4  // config 4: 2 -> 1.782, 4 -> 1.761, 8 -> 1.751 ms; with the packed table 2 / 4 / 6 / 8 -> 1.666 / 1.625 / 1.635 / 1.644 ms
#endif
#ifndef SIEVE_PLAIN_NG  // the wheel (groups) for which the plain-pass kernels are instantiated
#define SIEVE_PLAIN_NG 4
#endif
constexpr int kPlainILPCount = SIEVE_PLAIN_ILP_COUNT;
#ifndef SIEVE_COUNT_PLAIN  // count mode with r > S / kPlainHits: the plain-prime pass (k_sieve<.., kCount, true>)
#define SIEVE_COUNT_PLAIN 1
#endif
#ifndef SIEVE_BUCKET_HITS
#define SIEVE_BUCKET_HITS 1
#endif
constexpr uint32_t kBucketHits = SIEVE_BUCKET_HITS;
// ring of at most kMaxRing buckets per warp (a later hit is parked in the
// last bucket and re-queued from there)
constexpr uint32_t kMaxRing = 32;
// bucket entries a lane loads at once when draining
#ifndef SIEVE_DRAIN_ILP
#define SIEVE_DRAIN_ILP 4
#endif
constexpr uint32_t kDrainILP = SIEVE_DRAIN_ILP;
// primes a thread handles at once in the lane-per-prime region (load ILP)
#ifndef SIEVE_LARGE_ILP
#define SIEVE_LARGE_ILP 2
#endif
constexpr int kLargeILP = SIEVE_LARGE_ILP;

// alignment of the segment in shared memory (the runtime adds this many spare
// bytes to the dynamic shared-memory size)
constexpr uint32_t kSmemAlign = 128;

// launch bound of the sieve kernel (threads per CTA); the runtime never
// launches more (sieve_options.threads is clamped to it)
// default options (build-time overridable for same-box A/B variants)
#ifndef SIEVE_DEFAULT_SEGMENT_KB
#define SIEVE_DEFAULT_SEGMENT_KB 208
#endif
#ifndef SIEVE_DEFAULT_WHEEL
#define SIEVE_DEFAULT_WHEEL 31
#endif
#ifndef SIEVE_TMA_STORE  // A7 bitmap write-back by cp.async.bulk (0: 128-bit st.global)
#define SIEVE_TMA_STORE 1
#endif
#ifndef SIEVE_WHEEL_DIAG  // diagnostics builds only: 1 = wheel init without table-index updates (wrong results)
#define SIEVE_WHEEL_DIAG 0
#endif
#ifndef SIEVE_WB_DIAG  // diagnostics builds only: 1 = no wait for the bulk copy's reads, 2 = no bulk copy, 3 = no transpose
#define SIEVE_WB_DIAG 0
#endif
#ifndef SIEVE_LIST_STAGE  // A8 list emission staged in the consumed words of the segment: words per lane and pass (0 = direct)
#define SIEVE_LIST_STAGE 4  // config 4 list, same box: 0 / 3 / 4 / 5 / 6 / 8 -> 2.834 / 2.542 / 2.512 / 2.525 / 2.528 / 2.614 ms
#endif
#ifndef SIEVE_LIST_QUAD  // staged emission: four entries per lane and step of the ordered write (else two)
#define SIEVE_LIST_QUAD 0
#endif
#ifndef SIEVE_LIST_DIAG  // 1: list mode without pass 2 (diagnostics build, wrong list)
#define SIEVE_LIST_DIAG 0
#endif
#ifndef SIEVE_LIST_BFIND  // staged emission: bit positions by one BREV per word + one FLO per prime
#define SIEVE_LIST_BFIND 1  // config 4 list, same box, 3 rounds: 2.515-2.519 -> 2.479-2.493 ms
#endif
#ifndef SIEVE_LIST_WORDS  // A8 list emission: consecutive words per lane and warp pass (1 to 4)
#define SIEVE_LIST_WORDS 1  // A/B on config 4 list: 1 / 2 / 3 / 4 -> 2.83 / 3.02 / 3.28 / 3.6 ms
#endif
#ifndef SIEVE_UNTRANSPOSE_ILP  // blocks per warp and pass of the bit transpose
#define SIEVE_UNTRANSPOSE_ILP 2
#endif
#ifndef SIEVE_WB_FUSED  // bitmap mode: fused in-register transpose + count (writeback_fused)
#define SIEVE_WB_FUSED 1
#endif
#ifndef SIEVE_WB_WARP_COPY  // fused write-back: one bulk copy per warp run (1) or per segment (0)
#define SIEVE_WB_WARP_COPY 1
#endif
#ifndef SIEVE_B_PAIR  // region (B): pair hits 96 steps apart (one mask and one LOP3 per two atomics)
#define SIEVE_B_PAIR 1
#endif
#ifndef SIEVE_PACK44  // batch plain pass: {p, floor(2^44/p)} in one load (1) or p + recip (0)
#define SIEVE_PACK44 1
#endif
#ifndef SIEVE_WB_LANES  // lanes per 1024-slot block in the in-register transpose (2 or 4)
#define SIEVE_WB_LANES 2
#endif
#ifndef SIEVE_REG_TRANSPOSE  // list mode: in-register transpose (1) or the shuffle transpose (0)
#define SIEVE_REG_TRANSPOSE 1
#endif
#ifndef SIEVE_WHEEL_UNROLL  // unroll of the wheel-init word loop (count mode)
#define SIEVE_WHEEL_UNROLL 4
#endif
#ifndef SIEVE_EPI_PAIRS  // count/batch epilogue: two quads per carry-save step
#define SIEVE_EPI_PAIRS 1
#endif
#ifndef SIEVE_MAX_THREADS
#define SIEVE_MAX_THREADS 1024
#endif
// Bounds-check build (make check -> libsieve_check.so; "no worker
// writes outside its segment's bitmap ... ownership checks in debug builds"):
// every shared-memory mark outside the CTA's segment words, every global
// store outside its output array and every scratch write outside its
// capacity is counted (never trapped) in a device counter per class, read by
// sieve_debug_violations().  0 on the product build: the checks compile out.
#ifndef SIEVE_CHECK_BOUNDS
#define SIEVE_CHECK_BOUNDS 0
#endif
enum ViolationClass { kVioSmemMark = 0, kVioBitmapStore = 1, kVioListStore = 2, kVioScratch = 3,
                      kVioClasses = 4 };

// One work item of the batch kernel (step A10): one segment of one interval.
struct BatchItem {
  uint64_t a;         // first odd integer of the segment
  uint32_t valid;     // odd slots in the segment (<= segment bits)
  uint32_t interval;  // index of the interval (result slot)
  uint32_t r;         // isqrt(hi_interval - 1): marking primes p <= r
  uint32_t nend;      // index of the first base prime > r (k_plan_emit)
};

struct SieveParams {
  uint64_t o0;        // lo | 1 : the odd integer of bit 0
  uint64_t nbits;     // B = hi/2 - lo/2 odd slots
  uint64_t nseg;      // segments (or batch items)
  uint32_t seg_bits;  // S, a multiple of 1024
  uint32_t r;         // marking primes p <= r
  const uint32_t *primes;  // odd primes ascending (3, 5, 7, ...)
  const uint64_t *recips;  // floor((2^64-1)/p)
  const uint32_t *nbase;   // device count of primes[]
  const uint32_t *tables;  // wheel tables, packed per group_offset()
  uint32_t *out;           // bitmap mode: output words (bit 0 = word 0 bit 0)
  uint64_t out_words;      // words of out
  uint32_t out_vec4;       // out is 16-byte aligned
  uint32_t add_two;        // 2 in [lo, hi): add (1, 2) to the result
  uint64_t *partials;      // [2] accumulator of (count, sum): 0 at launch, reset by the last CTA
  unsigned int *done;      // last-block-done ticket (self-resetting)
  uint64_t *result;        // [2] count, sum mod 2^64 (batch: [2 * nintervals])
  const BatchItem *items;  // batch mode
  unsigned long long *prof;  // optional phase-cycle counters + timelines (diagnostics), [120]
  uint32_t flags;            // diagnostics: kFlagSkipMarking
  // step A5 buckets (nullptr: off).  CTA c sieves the contiguous segments
  // [c nseg / grid, (c+1) nseg / grid); bucket (c, slot, warp) holds capw
  // entries {p, slot offset relative to its segment} at
  // buckets + ((c * ring + slot) * nwarps + warp) * capw.
  uint2 *buckets;
  uint32_t ring;     // ring size R (<= kMaxRing): a hit lands at most R-1 segments ahead
  uint32_t capw;     // capacity of one bucket (>= bucket primes / warps, rounded up)
  uint32_t inv_seg;  // ceil(2^32 / seg_bits): o / S by a multiply-high and one correction
  // list mode (step A8): the primes go straight from the segment to the list;
  // a segment's place comes from a decoupled look-back over the segments
  // before it (per-segment flags, tagged with the launch's epoch)
  uint64_t *list;       // ascending u64 primes, list[0] = 2 when 2 is in range
  uint64_t list_cap;    // entries list may hold (later primes are counted, not written)
  unsigned long long *lflags;  // [nseg]
  uint32_t lepoch;
  // F4 (count mode; peers == nullptr: off): the all-reduce of (count, sum)
  // over `world` GPUs fused into the last CTA (peer.cuh).  peers[q] is rank
  // q's slab, P2P-mapped into this process; pepoch numbers the fused launch.
  unsigned long long *const *peers;
  uint64_t pepoch;
  uint64_t timeout_ns;
  uint32_t world, rank;
  // fused A2 (count/bitmap/list; bprimes == nullptr: off): before sieving,
  // CTA c computes the odd primes of slice c of the odd numbers <= r into
  // bprimes/brecips (the buffers primes/recips point to) and *bnbase, with
  // two grid barriers (cooperative launch: all CTAs resident).
  uint32_t *bprimes;
  uint64_t *brecips;
  uint32_t *bnbase;
  uint32_t bcap;        // capacity of bprimes/brecips
  uint32_t rs;          // isqrt(r)
  uint32_t *bcounts;    // [gridDim.x] per-CTA prime counts, then [7] region boundaries
  unsigned int *gbar;   // grid barrier counter: 0 at launch, reset by the last CTA
  const uint32_t *nitems;  // batch mode, device-planned: the item count (overrides nseg)
  uint2 *pk44;             // plain pass (batch and kPlain kernels): {p, floor(2^44/p)} per base
                           // prime, or nullptr; written by the fused A2 when bprimes is set
};

// Diagnostic flag: skip step A4/A5 (wheel init + count/write-back only), to
// measure the bitmap write-back stage in isolation.  Results are then wrong
// by design; never set on the product path.
constexpr uint32_t kFlagSkipMarking = 1u;
// Diagnostic flags: skip marking regions (A1+A2), (B), (C) -- marginal cost
// of each region in context.  Wrong results by design.
constexpr uint32_t kFlagSkipA = 2u, kFlagSkipB = 4u, kFlagSkipC = 8u;
// Diagnostic flag (bitmap mode): every CTA walks its segments in the reverse
// order (segment nseg-1-s instead of s) -- the schedule invariance of
// SPEC.md:152-154; bitmap, count and sum must be identical.
constexpr uint32_t kFlagReverse = 16u;
// Diagnostic flag: never take the cooperative (fused A2) launch -- the path
// the runtime falls back to when a cooperative launch is refused.
constexpr uint32_t kFlagNoCoop = 32u;
// Diagnostic flag (count mode, F3): the cluster-pair kernel k_sieve_cluster
// (two CTAs per super-segment, region C over distributed shared memory), base
// primes by K1.  An A/B variant, not the product path.
constexpr uint32_t kFlagCluster = 64u;
// Bitmap mode without the prime sum (sieve_bitmap, option bitmap_count_only):
// the write-back counts from carry-save planes only; result[1] = 0.  A
// product flag, set by the runtime -- not a diagnostic.
constexpr uint32_t kFlagNoSum = 128u;
// Diagnostic flag: skip the wheel init too (with kFlagSkipMarking: the
// bitmap write-back -- transpose, count, copy -- alone).  Results are wrong.
constexpr uint32_t kFlagSkipWheel = 256u;

enum Mode { kCount = 0, kBitmap = 1, kBatch = 2, kList = 3 };

// fused A2 scratch in the segment buffer: small primes (words) + staging
constexpr uint64_t kMaxSmallWords = 1024;

// launchers (kernels.cu)
cudaError_t launch_sieve(int ng, int mode, const SieveParams &p, int grid, int threads,
                         size_t smem, cudaStream_t s);
cudaError_t set_sieve_smem_limits(size_t smem);
cudaError_t launch_sieve_cluster(int ng, const SieveParams &p, int grid, int threads, size_t smem,
                                 cudaStream_t s);
cudaError_t launch_base_primes(uint32_t r, uint32_t rs, uint32_t *primes, uint64_t *recips,
                               uint32_t cap, uint32_t *nbase, uint64_t *flags, uint32_t epoch,
                               int nsm, unsigned long long *prof, cudaStream_t s);
uint32_t base_slices(uint32_t r);  // look-back flags the base-prime kernel needs
cudaError_t launch_pack44(const uint32_t *primes, const uint64_t *recips, const uint32_t *nbase, uint2 *pk44,
                          uint32_t cap, cudaStream_t s);
cudaError_t launch_prepare(const uint32_t *primes, const uint32_t *nbase, uint64_t *recips,
                           uint32_t cap, cudaStream_t s);
// A10 planning on the device (no host pass over the intervals): interval i
// of B_i odd slots becomes k_i = ceil(B_i / S) equal items (an interval with
// hi - lo > width_max gets the sentinel result 2^64-1 instead), items ordered by a
// counting sort on a log2 cost class, largest first (cost = the slots plus
// one first-hit reduction per base prime <= r_i, as the host planner had);
// result[2i..2i+1] initialised with (1, 2) when 2 is in the interval, else 0.
// scratch: hist/cursor [2 x kPlanBuckets] u32, per-interval [2 x n] u32,
// *nitems.  The base primes <= isqrt(hi_max - 1) must be in primes/nbase.
constexpr uint32_t kPlanBuckets = 256;
cudaError_t launch_batch_plan(const uint64_t *lo, const uint64_t *hi, uint64_t n, uint32_t S,
                              uint64_t width_max, const uint32_t *primes, const uint32_t *nbase,
                              uint32_t *scratch, BatchItem *items, uint32_t *nitems,
                              uint64_t *result, cudaStream_t s);
// peer.cu: the fused all-reduce alone, for a rank whose
// block holds no odd slot (it still publishes, the peers wait for it)
cudaError_t launch_peer_only(unsigned long long *const *peers, uint32_t world, uint32_t rank,
                             uint64_t epoch, uint64_t timeout_ns, uint64_t count, uint64_t sum,
                             uint64_t *result, cudaStream_t s, bool wait = true);
// primality.cu (Alg. 2, Alg. 3, deterministic Miller-Rabin)
cudaError_t launch_modpow(const uint64_t *a, const uint64_t *b, const uint64_t *c, uint64_t n,
                          uint64_t *out, cudaStream_t s);
cudaError_t launch_fermat(const uint64_t *p, uint64_t n, const uint64_t *draws, uint32_t iters,
                          uint8_t *out, cudaStream_t s);
cudaError_t launch_is_prime(const uint64_t *nums, uint64_t n, uint8_t *out, cudaStream_t s);
int sieve_max_ctas_per_sm(int ng, int mode, int threads, size_t smem);
// bounds-check build: violations per ViolationClass since the last reset
// (all zero, and reset a no-op, in the product build)
cudaError_t read_violations(unsigned long long *out, bool reset);
// K0 (diagnostics): conflict-free shared-memory atomicOr
// lanes per SM-clock per SM, measured on the device the library runs on
cudaError_t k0_smem_atomic_rate(int nsm, double *lanes_per_clk_per_sm, double *sm_ghz);

}  // namespace sv
