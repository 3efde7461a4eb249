// Device helpers shared by the CPQR kernels (cpqr.cu, cpqr_dist.cu).
#pragma once

#include <float.h>
#include <math.h>
#include <stdint.h>

namespace {

struct ArgMax {
    double val;
    int64_t pos;
    int64_t col;
    int64_t col_at_next;  // column currently at position (step + 1), or -1
};

__device__ __forceinline__ bool better(double v, int64_t p, double bv, int64_t bp) {
    // larger value wins; equal values -> lower position (first max, idamax)
    return v > bv || (v == bv && p < bp);
}

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// LAPACK dlapy2: sqrt(x^2 + y^2) avoiding overflow.
__device__ __forceinline__ double dlapy2(double x, double y) {
    const double xa = fabs(x), ya = fabs(y);
    const double w = fmax(xa, ya), z = fmin(xa, ya);
    if (z == 0.0 || w > DBL_MAX) return w;
    const double r = z / w;
    return w * sqrt(1.0 + r * r);
}



// Warp 0 reduces the G per-CTA argmax partials (lane-parallel loads, then a
// shuffle tree); every CTA runs the same code, so all agree on the pivot.
__device__ ArgMax reduce_partials_warp(const ArgMax* __restrict__ part, int64_t G) {
    const int lane = threadIdx.x & 31;
    ArgMax best{-1.0, INT64_MAX, -1, -1};
    for (int64_t i0 = 0; i0 < G; i0 += 128) {  // four candidates per lane in flight
        ArgMax o[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + lane + 32 * u;
            if (i < G) o[u] = part[i];
            else o[u] = ArgMax{-1.0, INT64_MAX, -1, -1};
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (better(o[u].val, o[u].pos, best.val, best.pos)) {
                best.val = o[u].val;
                best.pos = o[u].pos;
                best.col = o[u].col;
            }
            if (o[u].col_at_next >= 0) best.col_at_next = o[u].col_at_next;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        ArgMax ot;
        ot.val = __shfl_xor_sync(0xffffffffu, best.val, o);
        ot.pos = __shfl_xor_sync(0xffffffffu, best.pos, o);
        ot.col = __shfl_xor_sync(0xffffffffu, best.col, o);
        ot.col_at_next = __shfl_xor_sync(0xffffffffu, best.col_at_next, o);
        if (better(ot.val, ot.pos, best.val, best.pos)) {
            best.val = ot.val;
            best.pos = ot.pos;
            best.col = ot.col;
        }
        if (ot.col_at_next >= 0) best.col_at_next = ot.col_at_next;
    }
    return best;
}

// Fixed-order sum of G partials strided by `stride`, by one warp (all lanes
// get the result); identical in every CTA.  Eight loads per lane in flight.
__device__ __forceinline__ double warp_sum_partials(const double* __restrict__ p, int64_t G,
                                                    int64_t stride) {
    const int lane = threadIdx.x & 31;
    double s = 0.0;
    for (int64_t i0 = 0; i0 < G; i0 += 256) {
        double t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t i = i0 + lane + 32 * u;
            t[u] = i < G ? p[i * stride] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) s += t[u];
    }
    return warp_sum(s);
}

// y - sum_q a[q*lda] * b[q*ldb] for q < n: eight loads of each operand in
// flight, four independent chains.
__device__ __forceinline__ double sub_dot(double y, const double* __restrict__ a, int64_t lda,
                                          const double* __restrict__ b, int64_t ldb, int64_t n) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int64_t q = 0;
    for (; q + 8 <= n; q += 8) {
        double x[8], w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x[u] = a[(q + u) * lda];
            w[u] = b[(q + u) * ldb];
        }
        s0 = fma(x[0], w[0], s0);
        s1 = fma(x[1], w[1], s1);
        s2 = fma(x[2], w[2], s2);
        s3 = fma(x[3], w[3], s3);
        s0 = fma(x[4], w[4], s0);
        s1 = fma(x[5], w[5], s1);
        s2 = fma(x[6], w[6], s2);
        s3 = fma(x[7], w[7], s3);
    }
    for (; q + 4 <= n; q += 4) {
        s0 = fma(a[q * lda], b[q * ldb], s0);
        s1 = fma(a[(q + 1) * lda], b[(q + 1) * ldb], s1);
        s2 = fma(a[(q + 2) * lda], b[(q + 2) * ldb], s2);
        s3 = fma(a[(q + 3) * lda], b[(q + 3) * ldb], s3);
    }
    for (; q < n; ++q) s0 = fma(a[q * lda], b[q * ldb], s0);
    return y - ((s0 + s1) + (s2 + s3));
}

// sum_{r = r0 + lane, step 32, r < m} a[r] * b[r] with four independent chains
// (one warp; result NOT yet reduced across lanes).
__device__ __forceinline__ double lane_dot(const double* __restrict__ a, const double* __restrict__ b,
                                           int64_t r0, int64_t m) {
    double s[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    // eight loads in flight per lane; the last batch is clamped and zero-weighted
    for (int64_t r = r0 + (threadIdx.x & 31); r < m; r += 256) {
        double x[8], y[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t rr = r + 32 * u;
            const int64_t rc = rr < m ? rr : m - 1;
            x[u] = a[rc];
            y[u] = rr < m ? b[rc] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) s[u] = fma(x[u], y[u], s[u]);
    }
    return ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
}

__device__ __forceinline__ int64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return (int64_t)t;
}

}  // namespace
