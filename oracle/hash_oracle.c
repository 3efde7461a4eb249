/*
 * oracle/hash_oracle.c -- TEST INFRASTRUCTURE ONLY (CPU checker, never shipped).
 *
 * Plain-C restatement of the CountSketch hash draw of the reference,
 * /root/reference/pkg/src/idsketch/sketch.py:77-84 (CountSketchOp.__init__):
 *
 *     rng = np.random.default_rng(seed)
 *     if surjective:
 *         tail = rng.integers(0, out_dim, size=in_dim - out_dim)     # phase A
 *         slots = np.concatenate([np.arange(out_dim), tail])
 *         bucket = rng.permutation(slots)                            # phase B
 *     else:
 *         bucket = rng.integers(0, out_dim, size=in_dim)             # phase A'
 *     sign = rng.integers(0, 2, size=in_dim) * 2.0 - 1.0             # signs
 *
 * The arithmetic lives in a third-party dependency that is not under
 * /root/reference: numpy (pinned here at 2.3.5; the reference's
 * pyproject.toml:10-14 only asks numpy>=1.24).  What is restated is numpy's
 * published algorithm for that call sequence:
 *   - PCG64: 128-bit LCG s <- s*M + inc, output XSL-RR of the NEW state;
 *   - 32-bit draws share one pending-half buffer: a 32-bit request returns
 *     the stored high half if any, else draws 64 bits, returns the low half
 *     and stores the high half;
 *   - integers(0, L) for L-1 <= 0xFFFFFFFF is 32-bit Lemire with rejection
 *     (accept iff (x*L mod 2^32) >= (2^32 - L) mod L); L == 1 draws nothing;
 *   - permutation() of a 1-D array is Fisher-Yates for i = n-1 .. 1 with
 *     j = masked rejection draw in [0, i] (mask = smallest 2^b-1 >= i).
 * The host passes the initial (state, inc) that numpy's SeedSequence
 * produced, so SeedSequence itself is not restated.
 *
 * Pinned against golden vectors produced by the real reference
 * (tests/golden/make_golden.py) and against numpy's Generator directly.
 */
#include <stdint.h>
#include <string.h>

typedef unsigned __int128 u128;

typedef struct {
    u128 state, inc;
    int has_half;
    uint32_t half;
    uint64_t n64; /* number of 64-bit outputs drawn so far */
} pcg64_t;

static const u128 PCG_MULT =
    (((u128)0x2360ED051FC65DA4ULL) << 64) | (u128)0x4385DF649FCCF645ULL;

static inline uint64_t pcg64_next64(pcg64_t *g) {
    g->state = g->state * PCG_MULT + g->inc;
    uint64_t hi = (uint64_t)(g->state >> 64), lo = (uint64_t)g->state;
    uint64_t x = hi ^ lo;
    unsigned rot = (unsigned)(hi >> 58);
    g->n64++;
    return (x >> rot) | (x << ((64 - rot) & 63));
}

static inline uint32_t pcg64_next32(pcg64_t *g) {
    if (g->has_half) {
        g->has_half = 0;
        return g->half;
    }
    uint64_t v = pcg64_next64(g);
    g->has_half = 1;
    g->half = (uint32_t)(v >> 32);
    return (uint32_t)v;
}

/* numpy buffered_bounded_lemire_uint32 with rng = L-1 (L >= 2). */
static inline uint32_t lemire32(pcg64_t *g, uint32_t L) {
    uint64_t m = (uint64_t)pcg64_next32(g) * L;
    uint32_t left = (uint32_t)m;
    if (left < L) {
        uint32_t thresh = (uint32_t)(-L) % L;
        while (left < thresh) {
            m = (uint64_t)pcg64_next32(g) * L;
            left = (uint32_t)m;
        }
    }
    return (uint32_t)(m >> 32);
}

/* numpy random_interval(max) for max <= 0xFFFFFFFF. */
static inline uint32_t interval32(pcg64_t *g, uint32_t max) {
    if (max == 0) return 0;
    uint32_t mask = max;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
    mask |= mask >> 8; mask |= mask >> 16;
    uint32_t v;
    while ((v = (pcg64_next32(g) & mask)) > max) {}
    return v;
}

/*
 * Returns 0 on success, -1 on bad arguments.
 * state/inc: numpy PCG64 .state["state"] as two 64-bit halves (hi, lo).
 * bucket: int64[in_dim]; sign: double[in_dim]; draws_out: number of 32-bit
 * draws consumed per phase {A, B, signs} (may be NULL).
 */
int oracle_countsketch_hash(uint64_t state_hi, uint64_t state_lo,
                            uint64_t inc_hi, uint64_t inc_lo,
                            int64_t in_dim, int64_t out_dim, int surjective,
                            int64_t *bucket, double *sign, int64_t *draws_out) {
    if (in_dim < 1 || out_dim < 1 || out_dim > 0xFFFFFFFFLL) return -1;
    if (in_dim > 0xFFFFFFFFLL) return -1; /* 64-bit interval path not restated */
    if (surjective && out_dim > in_dim) return -1;
    pcg64_t g;
    g.state = ((u128)state_hi << 64) | state_lo;
    g.inc = ((u128)inc_hi << 64) | inc_lo;
    g.has_half = 0;
    g.half = 0;
    g.n64 = 0;
    const uint32_t L = (uint32_t)out_dim;
    uint64_t d0 = 0, d1, d2, d3;
#define DRAWS32() (2 * g.n64 - (uint64_t)g.has_half)
    if (surjective) {
        for (int64_t t = 0; t < out_dim; ++t) bucket[t] = t;
        for (int64_t t = out_dim; t < in_dim; ++t)
            bucket[t] = (L == 1) ? 0 : (int64_t)lemire32(&g, L);
        d1 = DRAWS32();
        for (int64_t i = in_dim - 1; i >= 1; --i) {
            uint32_t j = interval32(&g, (uint32_t)i);
            int64_t tmp = bucket[j];
            bucket[j] = bucket[i];
            bucket[i] = tmp;
        }
        d2 = DRAWS32();
    } else {
        for (int64_t t = 0; t < in_dim; ++t)
            bucket[t] = (L == 1) ? 0 : (int64_t)lemire32(&g, L);
        d1 = DRAWS32();
        d2 = d1;
    }
    for (int64_t t = 0; t < in_dim; ++t)
        sign[t] = (pcg64_next32(&g) >> 31) ? 1.0 : -1.0;
    d3 = DRAWS32();
    if (draws_out) {
        draws_out[0] = (int64_t)(d1 - d0);
        draws_out[1] = (int64_t)(d2 - d1);
        draws_out[2] = (int64_t)(d3 - d2);
    }
#undef DRAWS32
    return 0;
}

/* Raw 32-bit draw stream from a fresh generator: out[d] for d < n. */
int oracle_pcg64_stream32(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                          uint64_t inc_lo, int64_t n, uint32_t *out) {
    pcg64_t g;
    g.state = ((u128)state_hi << 64) | state_lo;
    g.inc = ((u128)inc_hi << 64) | inc_lo;
    g.has_half = 0;
    g.half = 0;
    g.n64 = 0;
    for (int64_t d = 0; d < n; ++d) out[d] = pcg64_next32(&g);
    return 0;
}

/*
 * Sequential CountSketch restating scipy's csr_matvecs / csr_matmat order
 * (reference sketch.py:119 `self._matrix @ a`): for each bucket l, rows i
 * with h(i) = l in increasing i, Y[l, :] += sign(i) * A[i, :], Y starting at
 * +0.0.  A is row-major (rows x cols, leading dimension lda); Y row-major L x cols.
 */
int oracle_countsketch_dense(const double *A, int64_t rows, int64_t cols, int64_t lda,
                             const int64_t *bucket, const double *sign, int64_t L,
                             double *Y) {
    memset(Y, 0, sizeof(double) * (size_t)(L * cols));
    for (int64_t i = 0; i < rows; ++i) {
        double *y = Y + bucket[i] * cols;
        const double *a = A + i * lda;
        const double s = sign[i];
        for (int64_t c = 0; c < cols; ++c) y[c] += s * a[c];
    }
    return 0;
}
