/*
 * oracle.c -- plain, slow, obviously-correct CPU sieve of Eratosthenes.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1205_4883_b200/) never links, imports or executes
 * anything under oracle/, and shares no code, header, table or constant
 * generator with it.
 *
 * What it computes:
 *   P(lo,hi) = { n in [lo,hi) : n >= 2 and no d in [2, sqrt(n)] divides n }
 *     -- the trial-division definition of a prime, PAPER.md:29 (Sec. 1,
 *        "integer n is prime if and only if it is not divisible by any prime
 *        not exceeding sqrt(n)").
 *   It is computed the way the paper states the method
 *   (Sec. 3.1 "Algorithm Design"): "iteratively marking as composite the
 *   multiples of each prime, starting with the multiples of 2".
 *
 * Deliberately a different layout from the GPU path: ONE BYTE PER INTEGER,
 * evens included, no wheel, no bit packing, no odd-only grid.  The range is
 * cut into chunks of CHUNK integers only so that memory stays bounded; the
 * chunk split is the paper's own "average divide data into nodes"
 * (Sec. 3.1 Eq. 3) with every chunk sieved independently by the
 * full base-prime set (SPEC.md:158 start rule max(p^2, ceil(a/p)*p)).
 *
 * Outputs, all exact:
 *   count            = |P|
 *   sum              = (sum of P) mod 2^64           (reading R7)
 *   list             = P ascending as uint64          (reading R8)
 *   bitmap           = bit j (word j>>5, bit j&31, LSB first) set iff
 *                      (lo|1) + 2j is in P, for 0 <= j < B,
 *                      B = floor(hi/2) - floor(lo/2); padding bits 0
 *                      (reading R5)
 *   fnv1a64(bytes)   = FNV-1a 64 over a byte string (reading R6)
 *
 * Threads: chunks are distributed over T pthreads (interleaved), partial
 * results are merged in chunk order, so results never depend on T.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define CHUNK ((uint64_t)1 << 24) /* integers per chunk; a multiple of 64 */
#define ORACLE_MAX_HI ((uint64_t)1 << 48)

/* ---------------------------------------------------------------------- */
/* isqrt: largest r with r*r <= x, integer Newton iteration plus a final   */
/* +-1 fix-up (no floating point anywhere).                                */
/* ---------------------------------------------------------------------- */
uint64_t oracle_isqrt(uint64_t x) {
    if (x < 2) return x;
    uint64_t r = x, y = (r + 1) / 2;
    while (y < r) {          /* classic decreasing Newton sequence */
        r = y;
        y = (r + x / r) / 2;
    }
    while (r * r > x) r--;   /* defensive fix-ups (never taken for x < 2^64 */
    while ((r + 1) * (r + 1) <= x) r++; /*  when r+1 < 2^32)              */
    return r;
}

/* ---------------------------------------------------------------------- */
/* Base primes: the textbook byte sieve on [0, r].          */
/* Returns a malloc'ed ascending array of all primes <= r (2 included).   */
/* ---------------------------------------------------------------------- */
static uint32_t *base_primes_upto(uint64_t r, uint64_t *n_out) {
    *n_out = 0;
    if (r < 2) return NULL;
    unsigned char *is = (unsigned char *)malloc(r + 1);
    if (!is) return NULL;
    memset(is, 1, r + 1);
    is[0] = 0;
    is[1] = 0;
    for (uint64_t p = 2; p * p <= r; p++)
        if (is[p])
            for (uint64_t m = p * p; m <= r; m += p) is[m] = 0;
    uint64_t n = 0;
    for (uint64_t i = 2; i <= r; i++) n += is[i];
    uint32_t *pr = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
    if (!pr) { free(is); return NULL; }
    n = 0;
    for (uint64_t i = 2; i <= r; i++)
        if (is[i]) pr[n++] = (uint32_t)i;
    free(is);
    *n_out = n;
    return pr;
}

/* exported for tests: writes min(n, cap) primes <= r, returns n */
int64_t oracle_base_primes(uint64_t r, uint32_t *out, uint64_t cap) {
    uint64_t n = 0;
    uint32_t *pr = base_primes_upto(r, &n);
    if (r >= 2 && !pr) return -3;
    for (uint64_t i = 0; i < n && i < cap; i++) out[i] = pr[i];
    free(pr);
    return (int64_t)n;
}

/* ---------------------------------------------------------------------- */
/* One chunk [a, b): flags[n - a] = 1 iff n is prime.                      */
/* ---------------------------------------------------------------------- */
static void sieve_chunk(uint64_t a, uint64_t b, const uint32_t *pr, uint64_t np,
                        unsigned char *flags) {
    uint64_t len = b - a;
    for (uint64_t i = 0; i < len; i++) flags[i] = (a + i >= 2) ? 1 : 0;
    for (uint64_t k = 0; k < np; k++) {
        uint64_t p = pr[k];
        if (p * p >= b) break;             /* p*p > b-1: p marks nothing here */
        uint64_t m = ((a + p - 1) / p) * p; /* ceil(a/p)*p                     */
        if (m < p * p) m = p * p;           /* never mark p itself */
        for (; m < b; m += p) flags[m - a] = 0;
    }
}

typedef struct {
    uint64_t lo, hi, o0, nchunks;
    const uint32_t *pr;
    uint64_t np;
    int tid, nthreads;
    int pass;                 /* 0: count/sum/bitmap, 1: fill list */
    uint64_t *chunk_count;    /* [nchunks] */
    uint64_t *chunk_sum;      /* [nchunks] */
    uint64_t *chunk_off;      /* [nchunks] (pass 1) */
    uint32_t *bitmap;         /* may be NULL */
    uint64_t *list;           /* may be NULL */
    uint64_t cap;
    int err;
} job_t;

static void *worker(void *arg) {
    job_t *J = (job_t *)arg;
    unsigned char *flags = (unsigned char *)malloc(CHUNK);
    if (!flags) { J->err = -3; return NULL; }
    for (uint64_t c = (uint64_t)J->tid; c < J->nchunks; c += (uint64_t)J->nthreads) {
        uint64_t a = J->lo + c * CHUNK;
        uint64_t b = (J->hi - a > CHUNK) ? a + CHUNK : J->hi;
        sieve_chunk(a, b, J->pr, J->np, flags);
        if (J->pass == 0) {
            uint64_t cnt = 0, sum = 0;
            for (uint64_t n = a; n < b; n++) {
                if (!flags[n - a]) continue;
                cnt += 1;
                sum += n;                   /* wraps mod 2^64 (reading R7) */
                if (J->bitmap && (n & 1)) { /* odd member: bit (n - o0)/2  */
                    uint64_t j = (n - J->o0) / 2;
                    J->bitmap[j >> 5] |= (uint32_t)1 << (j & 31);
                }
            }
            J->chunk_count[c] = cnt;
            J->chunk_sum[c] = sum;
        } else {
            uint64_t idx = J->chunk_off[c];
            for (uint64_t n = a; n < b; n++) {
                if (!flags[n - a]) continue;
                if (idx < J->cap) J->list[idx] = n;
                idx++;
            }
        }
    }
    free(flags);
    return NULL;
}

static int run_pass(job_t *tmpl, int nthreads) {
    pthread_t th[256];
    job_t jobs[256];
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    for (int t = 0; t < nthreads; t++) {
        jobs[t] = *tmpl;
        jobs[t].tid = t;
        jobs[t].nthreads = nthreads;
        jobs[t].err = 0;
    }
    if (nthreads == 1) {
        worker(&jobs[0]);
    } else {
        for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, worker, &jobs[t]);
        for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    }
    for (int t = 0; t < nthreads; t++)
        if (jobs[t].err) return jobs[t].err;
    return 0;
}

/* number of uint32 words of the odd-only bitmap of [lo, hi) */
uint64_t oracle_bitmap_words(uint64_t lo, uint64_t hi) {
    if (hi <= lo) return 0;
    uint64_t B = hi / 2 - lo / 2;
    return (B + 31) / 32;
}

/*
 * The oracle entry point.  [lo, hi) half-open (reading R1).
 *   count, sum          : required outputs
 *   bitmap (nullable)   : oracle_bitmap_words(lo,hi) uint32 words, zeroed here
 *   list (nullable)     : the min(count, cap) smallest primes ascending
 * Returns 0, or -1 (lo > hi), -2 (hi > 2^48), -3 (out of memory).
 */
int oracle_sieve(uint64_t lo, uint64_t hi, int nthreads, uint64_t *count, uint64_t *sum,
                 uint32_t *bitmap, uint64_t *list, uint64_t cap) {
    if (lo > hi) return -1;
    if (hi > ORACLE_MAX_HI) return -2;
    *count = 0;
    *sum = 0;
    if (bitmap) memset(bitmap, 0, oracle_bitmap_words(lo, hi) * sizeof(uint32_t));
    if (hi <= lo) return 0;

    uint64_t r = (hi >= 2) ? oracle_isqrt(hi - 1) : 0;
    uint64_t np = 0;
    uint32_t *pr = base_primes_upto(r, &np);
    if (r >= 2 && !pr) return -3;

    uint64_t nchunks = (hi - lo + CHUNK - 1) / CHUNK;
    uint64_t *cc = (uint64_t *)calloc(nchunks, sizeof(uint64_t));
    uint64_t *cs = (uint64_t *)calloc(nchunks, sizeof(uint64_t));
    uint64_t *co = (uint64_t *)calloc(nchunks, sizeof(uint64_t));
    if (!cc || !cs || !co) { free(pr); free(cc); free(cs); free(co); return -3; }

    job_t J;
    memset(&J, 0, sizeof J);
    J.lo = lo; J.hi = hi; J.o0 = lo | 1; J.nchunks = nchunks;
    J.pr = pr; J.np = np;
    J.chunk_count = cc; J.chunk_sum = cs; J.chunk_off = co;
    J.bitmap = bitmap; J.list = list; J.cap = cap;
    J.pass = 0;
    int rc = run_pass(&J, nthreads);
    if (rc == 0) {
        uint64_t c = 0, s = 0;
        for (uint64_t k = 0; k < nchunks; k++) { /* merge in chunk order */
            co[k] = c;
            c += cc[k];
            s += cs[k];
        }
        *count = c;
        *sum = s;
        if (list && cap) {
            J.pass = 1;
            rc = run_pass(&J, nthreads);
        }
    }
    free(pr); free(cc); free(cs); free(co);
    return rc;
}

/* FNV-1a 64 over n bytes (reading R6): h = 0xcbf29ce484222325;
 * for each byte b: h = (h ^ b) * 0x100000001b3 mod 2^64. */
uint64_t oracle_fnv1a64(const unsigned char *bytes, uint64_t n) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (uint64_t i = 0; i < n; i++) {
        h ^= bytes[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

/* Batch of independent intervals (config 5): results in input order.
 * Intervals are distributed over threads; each interval runs the
 * single-threaded oracle above. */
typedef struct {
    const uint64_t *lo, *hi;
    uint64_t n;
    uint64_t *count, *sum;
    int tid, nthreads, err;
} bjob_t;

static void *bworker(void *arg) {
    bjob_t *J = (bjob_t *)arg;
    for (uint64_t i = (uint64_t)J->tid; i < J->n; i += (uint64_t)J->nthreads) {
        int rc = oracle_sieve(J->lo[i], J->hi[i], 1, &J->count[i], &J->sum[i], NULL, NULL, 0);
        if (rc) { J->err = rc; return NULL; }
    }
    return NULL;
}

int oracle_batch(const uint64_t *lo, const uint64_t *hi, uint64_t n, int nthreads,
                 uint64_t *count, uint64_t *sum) {
    pthread_t th[256];
    bjob_t jobs[256];
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    for (int t = 0; t < nthreads; t++) {
        jobs[t].lo = lo; jobs[t].hi = hi; jobs[t].n = n;
        jobs[t].count = count; jobs[t].sum = sum;
        jobs[t].tid = t; jobs[t].nthreads = nthreads; jobs[t].err = 0;
    }
    if (nthreads == 1) {
        bworker(&jobs[0]);
    } else {
        for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, bworker, &jobs[t]);
        for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    }
    for (int t = 0; t < nthreads; t++)
        if (jobs[t].err) return jobs[t].err;
    return 0;
}
