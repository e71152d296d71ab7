/*
 * primality.c -- plain CPU oracle for SURVEY.md 8(f) F2: the paper's Alg. 2
 * and Alg. 3, written out step by step in the paper's order and notation.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.c's header): only tests/,
 * __graft_entry__.smoke() and bench.py's reference legs may load it; it
 * shares nothing with paper_1205_4883_b200/.
 *
 * Exact arithmetic: every product x*y of two values < 2^64 is formed in a
 * 128-bit integer and reduced with the C remainder operator -- no Montgomery
 * form, no tricks -- so a reader can check each line against PAPER.md.
 */
#include <stdint.h>

typedef unsigned __int128 u128;

/* Alg. 2 "modulo(a,b,c): Exponentiating by squaring to (a^b) mod c"
 * (PAPER.md:189-205):
 *   REQUIRE x = 1, y = a
 *   WHILE b > 0: IF b & 1: x = (x*y) mod c;  y = (y*y) mod c;  b >>= 1
 *   RETURN x mod c
 * c = 0 is a domain error (SPEC.md mod_pow): UINT64_MAX is returned. */
uint64_t oracle_modpow(uint64_t a, uint64_t b, uint64_t c) {
    if (c == 0) return UINT64_MAX;
    u128 x = 1, y = a;
    while (b > 0) {
        if (b & 1) x = (x * y) % c;
        y = (y * y) % c;
        b >>= 1;
    }
    return (uint64_t)(x % c);
}

/* Alg. 3 "Fermat(p, iterations)":
 *   IF p = 1 RETURN false
 *   FOR i := 1 TO iterations:
 *     a = rand() mod (p-1) + 1
 *     IF modulo(a, p-1, p) != 1 RETURN false
 *   RETURN true
 * rand() is the caller's stream: the i-th draw is draws[i-1] (DESIGN.md
 * reading: random numbers the method draws are inputs).  p = 0 is a domain
 * error, reported as false. */
int oracle_fermat(uint64_t p, uint32_t iterations, const uint64_t *draws) {
    if (p == 1 || p == 0) return 0;
    for (uint32_t i = 1; i <= iterations; ++i) {
        const uint64_t a = draws[i - 1] % (p - 1) + 1;
        if (oracle_modpow(a, p - 1, p) != 1) return 0;
    }
    return 1;
}

/* batch forms (argument marshalling only) */
void oracle_modpow_batch(const uint64_t *a, const uint64_t *b, const uint64_t *c, uint64_t n,
                         uint64_t *out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = oracle_modpow(a[i], b[i], c[i]);
}

void oracle_fermat_batch(const uint64_t *p, uint64_t n, const uint64_t *draws, uint32_t iterations,
                         uint8_t *out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = (uint8_t)oracle_fermat(p[i], iterations, draws + i * iterations);
}
