/*
 * sieve.h -- C ABI of libsieve.so, the B200 (sm_100a) segmented sieve of
 * Eratosthenes.
 *
 * The operation (Sec. 3.1 "Algorithm Design"): "iteratively
 * marking as composite the multiples of each prime, starting with the
 * multiples of 2", applied to a contiguous range of integers that is split
 * into blocks ("average divide data into nodes"; Eq. 3,
 * PAPER.md:133-135).  The survivors are the primes, i.e. the integers n >= 2
 * with no divisor d in [2, sqrt(n)].  pi(x), the count of
 * primes, is the paper's PAPER.md:36 quantity.
 *
 * Conventions:
 *   R1  every range is HALF-OPEN [lo, hi); lo == hi is empty (not an error).
 *       Valid: lo <= hi <= SIEVE_MAX_HI (2^48).
 *   R2  0 and 1 are not prime; 2 is prime and is counted/summed/listed, but
 *       it is not in the odd-only bitmap.
 *   R5  bitmap: bit j (0 <= j < B, B = hi/2 - lo/2) of uint32 word j>>5,
 *       LSB first, is 1 iff the odd integer (lo|1) + 2j is prime.  Padding
 *       bits of the last word are 0.  Length sieve_bitmap_words(lo, hi).
 *   R7  sum = (sum of all primes in [lo, hi)) mod 2^64 (wrapping).
 *   R8  list = the primes in [lo, hi) ascending as uint64.
 *
 * Ownership and memory: output pointers are owned by the caller and may be
 * HOST or DEVICE memory (detected with cudaPointerGetAttributes).  Device
 * outputs are written in place on the library stream; host outputs receive a
 * device->host copy.  The library owns device scratch (base primes, partials,
 * list staging) and keeps it until sieve_shutdown().
 *
 * Threading: the synchronous calls return only after the GPU work finished.
 * All entry points are serialized by one internal mutex.  No C++ exception
 * ever crosses the ABI; failures return a negative SIEVE_E* code and set a
 * thread-local message readable with sieve_last_error().
 *
 * There is NO CPU fallback: without a usable CUDA device every compute call
 * returns SIEVE_ENODEV.
 */
#ifndef PAPER_1205_4883_B200_SIEVE_H
#define PAPER_1205_4883_B200_SIEVE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SIEVE_MAX_HI ((uint64_t)1 << 48)

/* error codes (all negative) */
#define SIEVE_OK 0
#define SIEVE_EINVAL -1 /* lo > hi, NULL output with non-zero size, bad option */
#define SIEVE_ERANGE -2 /* hi > SIEVE_MAX_HI */
#define SIEVE_ENOMEM -3 /* device or host allocation failed */
#define SIEVE_ECUDA -4  /* a CUDA runtime call or kernel launch failed */
#define SIEVE_ENODEV -5 /* no CUDA device / driver available */

/* Tuning options (sieve_set_options).  Zero fields mean "default". */
typedef struct sieve_options {
    uint32_t segment_kb;  /* maximum shared-memory segment size in KiB, in [4, 224] (default 208);
                             a call cuts [lo, hi) into equal segments of at most this size, a whole
                             number of waves of the persistent grid (at least 8 KiB) */
    uint32_t wheel;       /* wheel bound w (pre-sieved primes 3..w): 11, 17, 23, 31, 41 or 47 (default 31);
                             segment + wheel tables must fit 226 KiB of shared memory */
    uint32_t ctas_per_sm; /* resident CTAs per SM for the sieve kernel (default: occupancy maximum) */
    uint32_t threads;     /* threads per CTA: a multiple of 64 in [256, 1024] (default 1024) */
    uint32_t buckets;     /* step A5, primes p > S (at most one hit per segment of S odd slots):
                             0 = one Barrett first-hit reduction per prime and segment (default:
                             measured faster on B200 for every config);
                             1 = per-segment buckets (a skipped segment costs the prime nothing;
                             not used by sieve_batch, nor for ranges of more than 2^31 odd slots
                             per CTA, where the Barrett path runs) */
    uint32_t bitmap_count_only; /* 1: sieve_bitmap_async / sieve_bitmap_base_async compute the count
                             only and write result[1] = 0 (the write-back then needs no per-word
                             POPC); 0 (default): result[1] = the prime sum.  sieve_bitmap, which
                             returns the count alone, never computes the sum */
    uint32_t reserved[2]; /* must be zero */
} sieve_options;

/* ---------------------------------------------------------------------- */
/* The three calls named by north_star (BASELINE.json:5).                 */
/* ---------------------------------------------------------------------- */

/* pi(hi-1) - pi(lo-1): the number of primes in [lo, hi).  >= 0, or < 0 error. */
int64_t sieve_count(uint64_t lo, uint64_t hi);

/* Writes the odd-only prime bitmap of [lo, hi) (reading R5) into `out`
 * (sieve_bitmap_words(lo, hi) uint32 words, host or device).  Returns the
 * prime count (2 included when in range), or < 0 on error.  `out` may be
 * NULL only when the range holds no odd integer. */
int64_t sieve_bitmap(uint64_t lo, uint64_t hi, uint32_t *out);

/* Writes the min(count, cap) smallest primes of [lo, hi), ascending, into
 * `out` (uint64, host or device).  Returns the TOTAL count (> cap means the
 * list was truncated), or < 0 on error.  out may be NULL iff cap == 0, which
 * is a size query. */
int64_t sieve_primes(uint64_t lo, uint64_t hi, uint64_t *out, uint64_t cap);

/* ---------------------------------------------------------------------- */
/* Extensions the configs need.                        */
/* ---------------------------------------------------------------------- */

/* ceil((hi/2 - lo/2) / 32); 0 for an empty or odd-free range. */
uint64_t sieve_bitmap_words(uint64_t lo, uint64_t hi);

/* count and (sum of primes) mod 2^64 of [lo, hi) into host pointers. */
int sieve_stats(uint64_t lo, uint64_t hi, uint64_t *count, uint64_t *sum_mod_2_64);

/* n independent intervals [lo[i], hi[i]) (host arrays); per-interval count
 * and sum mod 2^64 written to host arrays in input order (config 5). */
int sieve_batch(const uint64_t *lo, const uint64_t *hi, uint64_t n, uint64_t *count,
                uint64_t *sum_mod_2_64);

/* ---------------------------------------------------------------------- */
/* Device-resident, stream-ordered API (multi-GPU orchestration, bench).   */
/* All pointers below are DEVICE pointers; calls enqueue work on the        */
/* library stream and return without synchronizing.                        */
/* ---------------------------------------------------------------------- */

/* Batch mode on device-resident intervals (config 5; what sieve_batch runs
 * after copying its host arrays): lo[i], hi[i] for i < n (device uint64),
 * result[2i] = count and result[2i+1] = sum mod 2^64 of [lo[i], hi[i])
 * (device, 2n uint64, overwritten).  hi_max >= every hi[i] (bounds the base
 * primes, <= 2^48) and width_max >= every hi[i] - lo[i] (bounds the items
 * per interval) are promises of the caller: an interval longer than
 * width_max gets the sentinel (2^64-1, 2^64-1); hi[i] > hi_max gives wrong
 * results.  lo[i] <= hi[i] is required.  The plan (items of at most one
 * segment, costliest first) is made on the device: no host pass. */
int sieve_batch_async(const uint64_t *lo, const uint64_t *hi, uint64_t n, uint64_t hi_max,
                      uint64_t width_max, uint64_t *result);

/* Upper bound on the number of odd primes <= r (sizes base-prime buffers). */
uint64_t sieve_base_capacity(uint64_t r);

/* Base primes (step A2): the odd primes p <= r ascending into primes[],
 * their Barrett reciprocals floor((2^64-1)/p) into recips[] and the count
 * into *nbase.  cap must be >= sieve_base_capacity(r).  r <= 2^24. */
int sieve_base_primes_async(uint64_t r, uint32_t *primes, uint64_t *recips, uint64_t cap,
                            uint32_t *nbase);

/* Recomputes recips[] for primes[] received from elsewhere (e.g. an NCCL
 * broadcast of primes[] and *nbase). */
int sieve_prepare_base_async(const uint32_t *primes, const uint32_t *nbase, uint64_t *recips,
                             uint64_t cap);

/* Count mode on [lo, hi) with the given base primes (all odd primes up to
 * at least isqrt(hi-1) must be present; larger ones are ignored).  Writes
 * result[0] = count, result[1] = sum mod 2^64 (overwrites). */
int sieve_stats_async(uint64_t lo, uint64_t hi, const uint32_t *primes, const uint64_t *recips,
                      const uint32_t *nbase, uint64_t *result);

/* Steps A2 + A3..A7 in ONE launch: the base primes <= isqrt(hi-1) are
 * computed into primes/recips/nbase (as sieve_base_primes_async would; cap
 * >= sieve_base_capacity(isqrt(hi-1))) by the sieve kernel itself -- every
 * CTA sieves a slice of the odd numbers <= r, two grid barriers of a
 * cooperative launch order them -- and then result[0..1] = (count, sum mod
 * 2^64) of [lo, hi).  allreduce != 0: the result is summed over the attached
 * peers as in sieve_stats_allreduce_async.  When a CTA's slice would not fit
 * its shared-memory segment (huge r, tiny range) the library runs the
 * base-prime kernel first instead; the results are the same. */
int sieve_stats_base_async(uint64_t lo, uint64_t hi, uint32_t *primes, uint64_t *recips,
                           uint32_t *nbase, uint64_t cap, int allreduce, uint64_t *result);

/* Bitmap mode: writes sieve_bitmap_words(lo,hi) words into out (device,
 * 16-byte aligned for vector stores; any alignment accepted) and
 * result[0..1] as above. */
int sieve_bitmap_async(uint64_t lo, uint64_t hi, const uint32_t *primes, const uint64_t *recips,
                       const uint32_t *nbase, uint32_t *out, uint64_t *result);

/* Bitmap mode with the base primes computed in the same launch (fused A2,
 * as sieve_stats_base_async; cap >= sieve_base_capacity(isqrt(hi-1))):
 * writes sieve_bitmap_words(lo,hi) words into out (device, any 4-byte
 * alignment) and result[0..1] = (count, sum mod 2^64) -- what sieve_bitmap
 * does, without the host round trip. */
int sieve_bitmap_base_async(uint64_t lo, uint64_t hi, uint32_t *primes, uint64_t *recips,
                            uint32_t *nbase, uint64_t cap, uint32_t *out, uint64_t *result);

/* ---------------------------------------------------------------------- */
/* SURVEY.md 8(f) F4 (overlap: the collective fused into the kernel,      */
/* PAPER.md:105-111) applied to the one exchange of the multi-GPU count    */
/* path, the all-reduce of A9 that ends the paper's flow (PAPER.md:163-169 */
/* "gather"): the sieve kernel's last CTA writes this                      */
/* rank's (count, sum) into every peer's slab over NVLink (P2P stores of   */
/* CUDA-IPC-mapped memory) and sums the slots the peers wrote into its own  */
/* -- no separate collective launch.  One process per GPU; the calls below */
/* are collective in the SPMD sense: every rank makes the same sequence of */
/* sieve_stats_allreduce_async calls.                                       */
/* ---------------------------------------------------------------------- */
#define SIEVE_IPC_HANDLE_BYTES 64
#define SIEVE_MAX_PEERS 64

/* Allocates (once) this process's slab on its device, zeroed, and writes
 * its cudaIpcMemHandle (SIEVE_IPC_HANDLE_BYTES bytes) into handle_out, to
 * be exchanged with the other ranks (e.g. an all_gather over the host). */
int sieve_peer_slab_handle(void *handle_out);

/* handles: world x SIEVE_IPC_HANDLE_BYTES, rank order (this rank's own
 * entry is ignored).  Opens every peer's slab (peer access enabled lazily),
 * zeroes this rank's slab and resets the launch epoch.  Every rank must
 * have attached (e.g. a barrier after this call) before the first fused
 * launch.  timeout_ms bounds each fused launch's wait for its peers (0 =
 * 10 s): a wait that expires yields result = {2^64-1, 2^64-1} instead of a
 * hung GPU.  1 <= world <= SIEVE_MAX_PEERS, 0 <= rank < world. */
int sieve_peer_attach(const void *handles, int world, int rank, uint32_t timeout_ms);

/* As sieve_peer_attach with the slabs given as device pointers valid in
 * this process (world entries, rank order; caller-owned, each >= 4 KiB;
 * slabs[rank] zeroed by the caller before the first fused launch). */
int sieve_peer_attach_ptrs(void *const *slabs, int world, int rank, uint32_t timeout_ms);

/* Closes the opened peer slabs; fused launches fail until the next attach. */
int sieve_peer_detach(void);

/* Number of fused launches since the last attach (launch e uses slab
 * parity e & 1; slot layout in csrc/peer.cuh). */
uint64_t sieve_peer_epoch(void);

/* Publishes this rank's (count, sum) for the NEXT fused epoch into every
 * attached slab and returns without waiting for the peers (the epoch
 * advances as for a fused launch).  Lets a test run the ranks' kernels one
 * after another on a single GPU -- rank 1 publishes, then rank 0's fused
 * launch finds rank 1's share already there -- so that no two kernels ever
 * wait on each other (B200_PROFILING.md: such kernels on one GPU are not
 * guaranteed to run concurrently).  SIEVE_EINVAL when nothing is attached. */
int sieve_peer_publish_async(uint64_t count, uint64_t sum);

/* As sieve_stats_async on this rank's [lo, hi), then result[0..1] = the
 * sums over all attached ranks of their (count, sum mod 2^64).  A rank
 * whose range holds no odd slot still takes part (a one-thread kernel).
 * SIEVE_EINVAL when no peers are attached. */
int sieve_stats_allreduce_async(uint64_t lo, uint64_t hi, const uint32_t *primes,
                                const uint64_t *recips, const uint32_t *nbase, uint64_t *result);

/* ---------------------------------------------------------------------- */
/* Configuration and diagnostics.                                          */
/* ---------------------------------------------------------------------- */
int sieve_set_device(int ordinal);
int sieve_set_stream(void *cuda_stream); /* NULL: the library's own stream */
void *sieve_get_stream(void);
int sieve_set_options(const sieve_options *o); /* NULL resets defaults */
int sieve_get_options(sieve_options *o);
const char *sieve_last_error(void);
void sieve_shutdown(void);

/* Number of kernels this library launched since load (evidence counter). */
uint64_t sieve_kernel_launches(void);

/* Diagnostics: when dev_counters (device, 120 x uint64, zeroed by the caller)
 * is non-NULL, later sieve launches add SM-clock cycles per phase:
 * [0] wheel init, [1] marking, [2] count/write-back (CTA level, summed over
 * segments), [3] small-, [4] medium-, [5] large-prime marking (per warp,
 * summed over warps), [6] segments, [8..103] per-warp region cycles, and a
 * globaltimer timeline of the count/bitmap kernel (ns): [104] ~min CTA
 * entry, [105] max entry, [106] max end of prologue, [107] max end of
 * sieving, [108] result written, [109] ~min end of sieving; of the base-
 * prime kernel: [112] ~min entry, [113] small primes, [114] slice marked,
 * [115] list offset known, [116] end (max over CTAs); of the fused A2 phase:
 * [110] slice counted, [111] barrier 1 passed, [117] primes written, [118]
 * barrier 2 passed.  The buffer must hold
 * 120 entries.  NULL disables (the default). */
int sieve_debug_set_profile(uint64_t *dev_counters);

/* Diagnostics: flags for later launches.  1 = skip the marking step (A4/A5):
 * wheel init + count/write-back only, to time the bitmap write-back stage in
 * isolation; 2 / 4 / 8 = skip the marking regions (A1+A2) /
 * (B) / (C) (marginal cost of a region).  Results are WRONG while any of
 * these is set.  16 = every CTA walks its segments in reverse order (bitmap
 * mode; schedule invariance: results must not change); 32 = never use the cooperative fused-A2 launch (the K1 + ordinary
 * launch path the library falls back to when a cooperative launch is
 * refused; results must not change); 64 = count mode through the F3
 * cluster-pair kernel (two CTAs per super-segment, the large primes over
 * distributed shared memory; an A/B variant, results must not change);
 * 256 = skip the wheel init as well (with 1: the bitmap transpose, count and
 * copy alone; results WRONG).
 * 0 restores. */
int sieve_debug_set_flags(uint32_t flags);

/* Diagnostics (bounds-check build, `make check` -> libsieve_check.so,
 * compiled with -DSIEVE_CHECK_BOUNDS=1): out[0..3] = counts of
 * shared-memory marks outside the CTA's segment words, bitmap stores outside
 * out[0, words), list stores outside list[0, cap), and scratch writes
 * (segment init/transpose, bucket rings, fused-A2 staging) outside their
 * capacity, since load or the last reset (reset != 0 zeroes them after
 * reading).  Synchronizes the library stream.  Returns 1 in the
 * bounds-check build, 0 in the product build (where nothing is checked and
 * the counts stay 0), < 0 on error. */
int sieve_debug_violations(uint64_t *out, int reset);

/* Diagnostics (K0): the conflict-free shared-memory
 * atomicOr rate of this GPU, in lanes per SM-clock per SM (~32 on B200),
 * and the SM clock the measurement ran at (GHz).  Runs a microbenchmark of
 * three launches on the current device; synchronous. */
int sieve_debug_k0(double *lanes_per_clk_per_sm, double *sm_ghz);

/* Diagnostics: cooperative (fused-A2) launches that were refused and re-run
 * as K1 + an ordinary launch, since load. */
uint64_t sieve_debug_coop_fallbacks(void);

/* ---------------------------------------------------------------------- */
/* the paper's second algorithm pair, batched on the    */
/* GPU (one candidate per thread).  Every pointer of a call is either a    */
/* device pointer (used in place, on the library stream) or a host pointer */
/* (staged through library-owned device scratch); mixing returns           */
/* SIEVE_EINVAL.  Calls are synchronous on return.                         */
/* ---------------------------------------------------------------------- */

/* Alg. 2 "modulo(a,b,c): exponentiating by squaring to (a^b) mod c"
 * (SPEC.md mod_pow): out[i] = a[i]^b[i] mod c[i] for
 * i < n, with the paper's loop (x = 1, y = a; while b > 0: if b & 1:
 * x = x y mod c; y = y y mod c; b >>= 1) on exact 128-bit products.
 * c[i] = 0 (a domain error) yields out[i] = UINT64_MAX; c[i] = 1 yields 0
 * (SPEC.md: "result mod c").  Returns 0 or an error code. */
int sieve_modpow(const uint64_t *a, const uint64_t *b, const uint64_t *c, uint64_t n, uint64_t *out);

/* Alg. 3 "Fermat(p, iterations)" (SPEC.md fermat_test):
 * out[i] = 1 iff p[i] passes `iterations` rounds, round t using the base
 * a = draws[i*iterations + t] mod (p[i]-1) + 1 -- the caller supplies the
 * random draws (Alg. 3's rand()), so verdicts are reproducible; draws holds
 * n*iterations values.  p = 1 yields 0 (Alg. 3's guard), p = 0 (a domain
 * error) yields 0.  iterations must be >= 1 (SIEVE_EINVAL otherwise). */
int sieve_fermat(const uint64_t *p, uint64_t n, const uint64_t *draws, uint32_t iterations, uint8_t *out);

/* Deterministic Miller-Rabin (bases 2, 3, 5, ..., 37: exact for every
 * 64-bit n), the "improved primality test" of PAPER.md:235-237, used as an
 * on-GPU verifier of sieve outputs: out[i] = 1 iff nums[i] is prime. */
int sieve_is_prime(const uint64_t *nums, uint64_t n, uint8_t *out);

#ifdef __cplusplus
}
#endif
#endif
