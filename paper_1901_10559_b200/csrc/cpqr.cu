// Truncated column-pivoted Householder QR + ID coefficients on B200.
//
// Replaces reference linalg.py:76-103 (cpqr: scipy.linalg.qr(pivoting=True)
// -> LAPACK dgeqp3/dorgqr, then truncation to k rows and numerical_rank) and
// matrix_id.py:56-84 (_coeffs_from_pivoted) + linalg.py:130-147
// (triangular_solve -> dtrtrs).
//
// Only k pivots are ever needed (k = rank <= sketch_dim), so the factorization
// runs k steps of LAPACK's pivoting rule and never touches the trailing
// matrix: like dlaqps it keeps the Householder vectors V (m x k) and the
// update factors F (n x k) so that the partially reduced matrix is
// Y - V F^T, and each step needs ONE streaming pass over Y (the GEMV
// Y^T v).  One persistent cooperative grid runs all k steps; column j is
// owned by one CTA for the whole factorization, rows are split across CTAs
// for the pivot-column work, and three grid-wide barriers separate the
// phases of a step (argmax -> pivot column -> GEMV -> downdate).
//
// Pivot rule (dgeqp3 / dlaqps): pivot = largest partial norm vn1 over the
// remaining columns, ties to the lowest current position (idamax); norms are
// downdated with LAPACK's formula and recomputed exactly when the downdate
// is untrustworthy (temp2 <= tol3z = sqrt(eps)).
#include <cooperative_groups.h>

#include <float.h>
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "cpqr_common.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kSeg = 512;                // GEMV unit: rows per (column, segment)
constexpr int kSegLoads = kSeg / 32;     // loads per lane per unit

struct CpqrArgs {
    const double* Y;
    int64_t m, n, ldy, k;
    int small;  // m small: pivot column and z computed redundantly by every CTA
    int64_t vwin;  // doubles of v kept in shared memory (all of it when small)
    const double* colnorm2;  // optional ||Y[:,j]||^2 (skips the initial norm pass)
    double rank_tol;
    int32_t* perm;
    double* Rtop;
    int32_t* numerical_rank;
    // workspace
    double *vn1, *vn2, *F, *Rcol, *W, *V, *tau, *beta, *a, *normpart, *zpart;
    int64_t* pos;
    int64_t* flag_list;
    ArgMax* amax;
    int64_t* tlog;  // debug: per-phase ns accumulated by CTA 0 (NULL: off)
};


// Block-wide sum of one double per thread; result valid in all threads.
__device__ double block_sum(double v, double* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < kWarps; ++i) s += red[i];
    return s;
}

__global__ void __launch_bounds__(kThreads, 1) cpqr_kernel(CpqrArgs g) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double vsm[];  // v (m), z (k), V[kk, :kk] (k)
    const int64_t mpad = (g.m + kSeg - 1) / kSeg * kSeg;  // v padded with zeros
    double* zsh = vsm + g.vwin;
    double* vrow = zsh + g.k;
    __shared__ int s_nflag;
    __shared__ double s_red0;
    __shared__ double red[kWarps];
    __shared__ ArgMax warp_best[kWarps];
    __shared__ int64_t s_piv[3];

    const int64_t G = gridDim.x, b = blockIdx.x;
    const int64_t m = g.m, n = g.n, k = g.k, ldy = g.ldy;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t c0 = n * b / G, c1 = n * (b + 1) / G;   // owned columns
    const int64_t r0 = m * b / G, r1 = m * (b + 1) / G;   // owned rows
    const double tol3z = sqrt(DBL_EPSILON);
    int64_t* flagged = g.flag_list + c0;  // this CTA's columns needing a norm recompute

    // local argmax over owned columns with pos >= pmin; reports column at pnext
    auto local_argmax = [&](int64_t pmin, int64_t pnext) {
        ArgMax best{-1.0, INT64_MAX, -1, -1};
        for (int64_t j = c0 + threadIdx.x; j < c1; j += kThreads) {
            const int64_t pj = g.pos[j];
            if (pj == pnext) best.col_at_next = j;
            if (pj >= pmin) {
                const double v = g.vn1[j];
                if (better(v, pj, best.val, best.pos)) {
                    best.val = v;
                    best.pos = pj;
                    best.col = j;
                }
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
        if (lane == 0) warp_best[wid] = best;
        __syncthreads();
        if (threadIdx.x == 0) {
            ArgMax r = warp_best[0];
            for (int i = 1; i < kWarps; ++i) {
                const ArgMax o = warp_best[i];
                if (better(o.val, o.pos, r.val, r.pos)) {
                    r.val = o.val;
                    r.pos = o.pos;
                    r.col = o.col;
                }
                if (o.col_at_next >= 0) r.col_at_next = o.col_at_next;
            }
            g.amax[b] = r;
        }
        __syncthreads();
    };

    // ---- prologue: column norms (dnrm2), positions; zero padding of a ----
    if (b == 0)
        for (int64_t r = m + threadIdx.x; r < mpad; r += kThreads) g.a[r] = 0.0;
    for (int64_t j = c0 + wid; j < c1; j += kWarps) {
        const double* y = g.Y + j * ldy;
        const double s = g.colnorm2 ? g.colnorm2[j] : warp_sum(lane_dot(y, y, 0, m));
        if (lane == 0) {
            g.vn1[j] = sqrt(s);
            g.vn2[j] = sqrt(s);
            g.pos[j] = j;
        }
    }
    __syncthreads();
    local_argmax(0, 0);
    grid.sync();

    const bool tl = g.tlog && b == 0 && threadIdx.x == 0;
    int64_t tprev = tl ? gtimer() : 0;
    auto stamp = [&](int phase) {
        if (tl) {
            const int64_t t = gtimer();
            g.tlog[phase] += t - tprev;
            tprev = t;
        }
    };
    for (int64_t kk = 0; kk < k; ++kk) {
        // ---- S1: global pivot, position swap, distributed pivot column ----
        if (wid == 0) {
            const ArgMax r = reduce_partials_warp(g.amax, G);
            if (lane == 0) {
                s_piv[0] = r.col;          // pivot column c*
                s_piv[1] = r.pos;          // its position p*
                s_piv[2] = r.col_at_next;  // column at position kk
            }
        }
        __syncthreads();
        int64_t cs = s_piv[0], ps = s_piv[1];
        const int64_t ck = s_piv[2];
        if (cs < 0) {  // every remaining norm is NaN (non-finite input): keep position kk
            cs = ck;
            ps = kk;
        }
        if (threadIdx.x == 0) {
            if (ck >= c0 && ck < c1 && ck != cs) g.pos[ck] = ps;
            if (cs >= c0 && cs < c1) g.pos[cs] = kk;
        }
        double alpha;
        if (g.small) {
            // short sketch: every CTA builds the whole pivot column itself
            const double* ycol = g.Y + cs * ldy;
            double ss = 0.0;
            for (int64_t r = kk + threadIdx.x; r < m; r += kThreads) {
                const double v = sub_dot(ycol[r], g.V + r, m, g.F + cs, n, kk);
                vsm[r] = v;
                if (r > kk) ss = fma(v, v, ss);
            }
            ss = block_sum(ss, red);
            if (threadIdx.x == 0) s_red0 = ss;
            __syncthreads();
            alpha = vsm[kk];
            __syncthreads();
        } else {
            const double* ycol = g.Y + cs * ldy;
            double ss = 0.0;
            for (int64_t r = r0 + threadIdx.x; r < r1; r += kThreads) {
                if (r < kk) {
                    g.a[r] = 0.0;  // rows above kk read as v = 0 by the GEMV
                    continue;
                }
                const double v = sub_dot(ycol[r], g.V + r, m, g.F + cs, n, kk);
                g.a[r] = v;
                if (r > kk) ss = fma(v, v, ss);
            }
            ss = block_sum(ss, red);
            if (threadIdx.x == 0) g.normpart[b] = ss;
            stamp(0);
            grid.sync();
            stamp(1);
            if (wid == 0) {
                const double xs = warp_sum_partials(g.normpart, G, 1);
                if (lane == 0) s_red0 = xs;
            }
            __syncthreads();
            alpha = g.a[kk];
        }

        // ---- S2: Householder vector (redundantly per CTA), z, GEMV ----
        const double xnorm = sqrt(s_red0);
        double tau, beta, scal;
        if (xnorm == 0.0) {
            tau = 0.0;
            beta = alpha;
            scal = 0.0;
        } else {
            beta = -copysign(dlapy2(alpha, xnorm), alpha);
            tau = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        // v = V[:, kk]: zero above kk, 1 at kk, a[r] * scal below (a[] holds
        // zeros above kk and in the padding).  Small sketches keep all of v
        // in shared memory; tall ones only the window of rows their GEMV
        // units touch, and read single entries from a[] elsewhere.
        auto vglob = [&](int64_t r) -> double { return r == kk ? 1.0 : g.a[r] * scal; };
        const int64_t nseg = (m + kSeg - 1) / kSeg, s0 = kk / kSeg, ns = nseg - s0;
        // tall: this CTA's contiguous range of units u = (sg - s0) * n + j
        const int64_t Ut = ns * n;
        const int64_t ub0 = g.small ? 0 : Ut * b / G, ub1 = g.small ? 0 : Ut * (b + 1) / G;
        const int64_t vlo = g.small ? 0 : (s0 + ub0 / n) * kSeg;
        const int64_t vhi = g.small ? mpad : (ub1 > ub0 ? (s0 + (ub1 - 1) / n + 1) * kSeg : vlo);
        if (g.small) {
            for (int64_t r = threadIdx.x; r < mpad; r += kThreads)
                vsm[r] = (r < kk || r >= m) ? 0.0 : (r == kk) ? 1.0 : vsm[r] * scal;
        } else {
            for (int64_t rb = vlo; rb < vhi; rb += 8 * kThreads) {  // 8 loads in flight
                double t[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int64_t r = rb + u * kThreads + threadIdx.x;
                    t[u] = r < vhi ? g.a[r] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int64_t r = rb + u * kThreads + threadIdx.x;
                    if (r < vhi) vsm[r - vlo] = (r == kk) ? 1.0 : t[u] * scal;
                }
            }
        }
        __syncthreads();
        // every CTA stores its own rows of V[:, kk] (identical values everywhere)
        for (int64_t r = r0 + threadIdx.x; r < r1; r += kThreads)
            g.V[kk * m + r] = r < kk ? 0.0 : (g.small ? vsm[r] : vglob(r));
        if (b == 0 && threadIdx.x == 0) {
            g.tau[kk] = tau;
            g.beta[kk] = beta;
        }
        if (threadIdx.x == 0 && cs >= c0 && cs < c1) g.Rcol[cs * k + kk] = beta;
        // z_q = V[:, q]^T v: whole columns (small) or owned-row partials
        for (int64_t q = wid; q < kk; q += kWarps) {
            if (g.small) {
                const double sz = warp_sum(lane_dot(g.V + q * m, vsm, kk, m));
                if (lane == 0) zsh[q] = sz;
            } else {
                double sz = 0.0;  // eight rows per lane in flight
                for (int64_t rb = tmax(r0, kk); rb < r1; rb += 256) {
                    double t[8], vv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int64_t r = rb + lane + 32 * u;
                        const bool ok = r < r1;
                        t[u] = ok ? g.V[q * m + r] : 0.0;
                        vv[u] = ok ? vglob(r) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) sz = fma(t[u], vv[u], sz);
                }
                sz = warp_sum(sz);
                if (lane == 0) g.zpart[b * k + q] = sz;
            }
        }
        stamp(8);
        // GEMV W_j = Y[kk:, j]^T v in units of (column j, kSeg-row segment),
        // two units per warp at a time (2 x 16 independent loads per lane);
        // partial dots go to W[sg * n + j] and are summed in fixed order in S3.
        // Small sketches: this CTA's columns; tall: this CTA's unit range,
        // walked backwards on odd steps (the tail of the previous pass is
        // still in L2 when Y does not fit there).
        {
            const int64_t cnt = g.small ? (c1 - c0) * ns : ub1 - ub0;
            const bool rev = !g.small && (kk & 1);
            const bool full = (m % kSeg) == 0;  // no clamping needed
            const int nl = (g.small && m < kSeg) ? (int)((m + 31) / 32) : kSegLoads;
            for (int64_t li = wid; li < cnt; li += 2 * kWarps) {
                int64_t j1, sg1, j2, sg2;
                const bool h2 = li + kWarps < cnt;
                if (g.small) {
                    j1 = c0 + li / ns;
                    sg1 = s0 + li % ns;
                    const int64_t l2 = h2 ? li + kWarps : li;
                    j2 = c0 + l2 / ns;
                    sg2 = s0 + l2 % ns;
                } else {
                    const uint32_t nn = (uint32_t)n;
                    const uint32_t ua = (uint32_t)(rev ? ub1 - 1 - li : ub0 + li);
                    const uint32_t l2 = (uint32_t)(h2 ? li + kWarps : li);
                    const uint32_t ub = (uint32_t)(rev ? ub1 - 1 - l2 : ub0 + l2);
                    j1 = ua % nn;
                    sg1 = s0 + ua / nn;
                    j2 = ub % nn;
                    sg2 = s0 + ub / nn;
                }
                const bool a1 = g.pos[j1] > kk, a2 = h2 && g.pos[j2] > kk;
                const double* p1 = g.Y + j1 * ldy;
                const double* p2 = g.Y + j2 * ldy;
                const int64_t b1 = sg1 * kSeg + lane, b2 = sg2 * kSeg + lane;
                double y1[kSegLoads], y2[kSegLoads];
                if (full) {
#pragma unroll
                    for (int t = 0; t < kSegLoads; ++t) {
                        y1[t] = p1[b1 + 32 * t];
                        y2[t] = p2[b2 + 32 * t];
                    }
                } else {  // clamped rows (v is zero there); a short sketch
                          // (m < kSeg) loads only its nl row groups
#pragma unroll
                    for (int t = 0; t < kSegLoads; ++t) {
                        y1[t] = t < nl ? p1[tmin(b1 + 32 * t, m - 1)] : 0.0;
                        y2[t] = t < nl ? p2[tmin(b2 + 32 * t, m - 1)] : 0.0;
                    }
                }
                const double* v1 = vsm + (b1 - vlo);
                const double* v2 = vsm + (b2 - vlo);
                double s1 = 0.0, s2 = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll
                for (int t = 0; t < kSegLoads; t += 2) {
                    if (t < nl) {
                        s1 = fma(y1[t], v1[32 * t], s1);
                        s2 = fma(y2[t], v2[32 * t], s2);
                    }
                    if (t + 1 < nl) {
                        t1 = fma(y1[t + 1], v1[32 * t + 32], t1);
                        t2 = fma(y2[t + 1], v2[32 * t + 32], t2);
                    }
                }
                const double w1 = warp_sum(s1 + t1), w2 = warp_sum(s2 + t2);
                if (lane == 0) {
                    if (a1) g.W[sg1 * n + j1] = w1;
                    if (a2) g.W[sg2 * n + j2] = w2;
                }
            }
        }
        stamp(2);
        if (g.small) __syncthreads();
        else grid.sync();
        stamp(3);

        // ---- S3: F column, row kk of R, norm downdate, next argmax ----
        // z = V[:, :kk]^T v (fixed-order sum of the per-CTA partials) and row kk of V
        for (int64_t q = wid; q < kk; q += kWarps) {
            const double zq = g.small ? 0.0 : warp_sum_partials(g.zpart + q, G, k);
            if (lane == 0) {
                if (!g.small) zsh[q] = zq;
                vrow[q] = g.V[q * m + kk];
            }
        }
        if (threadIdx.x == 0) s_nflag = 0;
        __syncthreads();
        stamp(9);
        // few owned columns: one warp per column (lanes split the segment
        // partials and the F dot products, lane 0 finishes the column); many
        // (short sketches): one thread per column
        const bool warp_cols = c1 - c0 <= 2 * kWarps;
        for (int64_t j = c0 + threadIdx.x; !warp_cols && j < c1; j += kThreads) {
            if (g.pos[j] <= kk) continue;
            double wj = 0.0;
            for (int64_t sg = kk / kSeg; sg < mpad / kSeg; ++sg) wj += g.W[sg * n + j];
            double f = sub_dot(wj, g.F + j, n, zsh, 1, kk);
            double rk = sub_dot(g.Y[j * ldy + kk], g.F + j, n, vrow, 1, kk);
            f *= tau;
            g.F[kk * n + j] = f;
            rk -= f;  // V[kk, kk] = 1
            g.Rcol[j * k + kk] = rk;
            const double vn1 = g.vn1[j];
            if (kk < m - 1 && vn1 != 0.0) {
                double temp = fabs(rk) / vn1;
                temp = fmax(0.0, (1.0 + temp) * (1.0 - temp));
                const double ratio = vn1 / g.vn2[j];
                const double temp2 = temp * ratio * ratio;
                if (temp2 <= tol3z) flagged[atomicAdd(&s_nflag, 1)] = j;
                else g.vn1[j] = vn1 * sqrt(temp);
            }
        }
        for (int64_t j = c0 + wid; warp_cols && j < c1; j += kWarps) {
            if (g.pos[j] <= kk) continue;
            const double ykk = lane == 0 ? g.Y[j * ldy + kk] : 0.0;
            const double vn1 = lane == 0 ? g.vn1[j] : 0.0;
            const double vn2 = lane == 0 ? g.vn2[j] : 1.0;
            double wj = 0.0, fz = 0.0, fv = 0.0;
            for (int64_t sg = kk / kSeg + lane; sg < mpad / kSeg; sg += 32) wj += g.W[sg * n + j];
            for (int64_t q = lane; q < kk; q += 32) {
                const double fq = g.F[q * n + j];
                fz = fma(fq, zsh[q], fz);
                fv = fma(fq, vrow[q], fv);
            }
            wj = warp_sum(wj);
            fz = warp_sum(fz);
            fv = warp_sum(fv);
            if (lane == 0) {
                const double f = (wj - fz) * tau;
                g.F[kk * n + j] = f;
                const double rk = (ykk - fv) - f;  // V[kk, kk] = 1
                g.Rcol[j * k + kk] = rk;
                if (kk < m - 1 && vn1 != 0.0) {
                    double temp = fabs(rk) / vn1;
                    temp = fmax(0.0, (1.0 + temp) * (1.0 - temp));
                    const double ratio = vn1 / vn2;
                    const double temp2 = temp * ratio * ratio;
                    if (temp2 <= tol3z) flagged[atomicAdd(&s_nflag, 1)] = j;
                    else g.vn1[j] = vn1 * sqrt(temp);
                }
            }
        }
        __syncthreads();
        stamp(4);
        // exact norms of the flagged columns below row kk (LAPACK's recompute)
        const int nflag = s_nflag;
        if (g.tlog && threadIdx.x == 0) atomicAdd((unsigned long long*)&g.tlog[15], (unsigned long long)nflag);
        for (int fi = wid; fi < nflag; fi += kWarps) {
            const int64_t j = flagged[fi];
            const double* y = g.Y + j * ldy;
            double s = 0.0;
            for (int64_t r = kk + 1 + lane; r < m; r += 32) {
                double v = sub_dot(y[r], g.V + r, m, g.F + j, n, kk);
                v = fma(-(g.small ? vsm[r] : vglob(r)), g.F[kk * n + j], v);
                s = fma(v, v, s);
            }
            s = warp_sum(s);
            if (lane == 0) {
                g.vn1[j] = sqrt(s);
                g.vn2[j] = sqrt(s);
            }
        }
        __syncthreads();
        stamp(5);
        local_argmax(kk + 1, kk + 1);
        stamp(6);
        grid.sync();
        stamp(7);
    }

    // ---- outputs: perm, Rtop, numerical rank ----
    for (int64_t j = c0 + threadIdx.x; j < c1; j += kThreads) {
        const int64_t p = g.pos[j];
        g.perm[p] = (int32_t)j;
        for (int64_t q = 0; q < k; ++q)
            g.Rtop[q * n + p] = (p >= q) ? g.Rcol[j * k + q] : 0.0;
    }
    if (b == 0 && threadIdx.x == 0) {
        const double lead = fabs(g.beta[0]);
        int32_t nr = 0;
        if (lead != 0.0)
            for (int64_t q = 0; q < k; ++q) nr += fabs(g.beta[q]) > g.rank_tol * lead ? 1 : 0;
        *g.numerical_rank = nr;
    }
}

// ---- short sketches: one thread-block CLUSTER, Y resident in shared memory --
// For L x R sketches small enough to split over the SMs of one cluster (the
// matrix configs: 40 x 1000, 100 x 2000), each CTA keeps its column slice of
// Y, its rows of F and R, and a private copy of V in shared memory.  A step
// then needs one hardware cluster barrier: the per-CTA argmax candidates are
// exchanged through distributed shared memory (double-buffered by step
// parity), the pivot column and its F row are read from the owner CTA's
// shared memory, and every CTA builds the Householder vector itself.

struct ClusterArgs {
    const double* Y;
    int64_t m, n, ldy, k;
    double rank_tol;
    int32_t* perm;
    double* Rtop;
    int32_t* numerical_rank;
    double* Vout;    // V (m x k) and tau for form_q_kernel, written by CTA 0
    double* tauout;
    int ncl;         // columns per CTA (max)
    int64_t* tlog;   // debug: per-phase ns accumulated by CTA 0 (NULL: off)
};

struct ClusterSmem {  // carve of the dynamic shared memory
    double *Ys, *Fs, *Rs, *V, *v, *z, *vn1, *vn2, *W, *tau, *beta;
    int* pos;
};

__device__ ClusterSmem carve_cluster(double* base, int64_t m, int64_t k, int ncl) {
    ClusterSmem c;
    c.Ys = base;
    c.Fs = c.Ys + (int64_t)m * ncl;  // F: k x ncl (q-major)
    c.Rs = c.Fs + k * ncl;           // R rows: k x ncl
    c.V = c.Rs + k * ncl;            // m x k col-major
    c.v = c.V + m * k;
    c.z = c.v + m;
    c.vn1 = c.z + k;
    c.vn2 = c.vn1 + ncl;
    c.W = c.vn2 + ncl;
    c.tau = c.W + ncl;
    c.beta = c.tau + k;
    c.pos = reinterpret_cast<int*>(c.beta + k);
    return c;
}

size_t cluster_smem_bytes(int64_t m, int64_t k, int ncl) {
    return sizeof(double) * ((size_t)m * ncl + 2 * k * ncl + m * k + m + k + 3 * ncl + 2 * k) +
           sizeof(int) * ncl + 64;
}

__global__ void __launch_bounds__(kThreads, 1) cpqr_cluster_kernel(ClusterArgs g) {
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ double dyn[];
    __shared__ ArgMax slot[2];           // this CTA's candidate, by step parity
    __shared__ ArgMax warp_best[kWarps];
    __shared__ double red[kWarps];
    __shared__ int64_t s_piv[3];
    __shared__ double s_ab[2];
    const int CS = (int)cluster.num_blocks();
    const int b = (int)cluster.block_rank();
    const int64_t m = g.m, n = g.n, k = g.k;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t c0 = n * b / CS, c1 = n * (b + 1) / CS;
    const int nc = (int)(c1 - c0);
    const ClusterSmem S = carve_cluster(dyn, m, k, g.ncl);
    const double tol3z = sqrt(DBL_EPSILON);

    // load the Y slice ROW-major (Ys[r * ncl + jj]: a thread per column walks
    // rows conflict-free), norms, positions
    for (int jj = wid; jj < nc; jj += kWarps) {  // a warp per column, coalesced rows
        const double* ycol = g.Y + (c0 + jj) * g.ldy;
        for (int64_t r = lane; r < m; r += 32) S.Ys[r * g.ncl + jj] = ycol[r];
    }
    __syncthreads();
    for (int jj = threadIdx.x; jj < nc; jj += kThreads) {
        double s2 = 0.0;
        for (int64_t r = 0; r < m; ++r) {
            const double y = S.Ys[r * g.ncl + jj];
            s2 = fma(y, y, s2);
        }
        S.vn1[jj] = sqrt(s2);
        S.vn2[jj] = sqrt(s2);
        S.pos[jj] = (int)(c0 + jj);
    }
    __syncthreads();

    auto local_argmax = [&](int64_t pmin, int64_t pnext, int par) {
        ArgMax best{-1.0, INT64_MAX, -1, -1};
        for (int jj = threadIdx.x; jj < nc; jj += kThreads) {
            const int64_t pj = S.pos[jj];
            if (pj == pnext) best.col_at_next = c0 + jj;
            if (pj >= pmin && better(S.vn1[jj], pj, best.val, best.pos)) {
                best.val = S.vn1[jj];
                best.pos = pj;
                best.col = c0 + jj;
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
        if (lane == 0) warp_best[wid] = best;
        __syncthreads();
        if (threadIdx.x == 0) {
            ArgMax r = warp_best[0];
            for (int i = 1; i < kWarps; ++i) {
                const ArgMax o = warp_best[i];
                if (better(o.val, o.pos, r.val, r.pos)) {
                    r.val = o.val;
                    r.pos = o.pos;
                    r.col = o.col;
                }
                if (o.col_at_next >= 0) r.col_at_next = o.col_at_next;
            }
            slot[par] = r;
        }
    };
    local_argmax(0, 0, 0);
    cluster.sync();

    const bool tl = g.tlog && b == 0 && threadIdx.x == 0;
    int64_t tprev = tl ? gtimer() : 0;
    auto stamp = [&](int phase) {
        if (tl) {
            const int64_t tn = gtimer();
            g.tlog[phase] += tn - tprev;
            tprev = tn;
        }
    };
    for (int64_t kk = 0; kk < k; ++kk) {
        const int par = (int)(kk & 1);
        // ---- pivot from every CTA's candidate (DSMEM), fixed rank order ----
        if (wid == 0) {  // lane q reads CTA q's candidate, then a shuffle tree
            ArgMax r{-1.0, INT64_MAX, -1, -1};
            if (lane < CS) r = *cluster.map_shared_rank(&slot[par], lane);
            for (int o = 16; o > 0; o >>= 1) {
                ArgMax ot;
                ot.val = __shfl_xor_sync(0xffffffffu, r.val, o);
                ot.pos = __shfl_xor_sync(0xffffffffu, r.pos, o);
                ot.col = __shfl_xor_sync(0xffffffffu, r.col, o);
                ot.col_at_next = __shfl_xor_sync(0xffffffffu, r.col_at_next, o);
                if (better(ot.val, ot.pos, r.val, r.pos)) {
                    r.val = ot.val;
                    r.pos = ot.pos;
                    r.col = ot.col;
                }
                if (ot.col_at_next >= 0) r.col_at_next = ot.col_at_next;
            }
            if (lane == 0) {
                if (r.col < 0) {  // all-NaN norms (non-finite input): keep position kk
                    r.col = r.col_at_next;
                    r.pos = kk;
                }
                s_piv[0] = r.col;
                s_piv[1] = r.pos;
                s_piv[2] = r.col_at_next;
            }
        }
        __syncthreads();
        const int64_t cs = s_piv[0], ps = s_piv[1], ck = s_piv[2];
        if (threadIdx.x == 0) {
            if (ck >= c0 && ck < c1 && ck != cs) S.pos[ck - c0] = (int)ps;
            if (cs >= c0 && cs < c1) S.pos[cs - c0] = (int)kk;
        }
        stamp(0);
        // ---- pivot column from the owner's shared memory, Householder ----
        // owner of column cs: the largest b with n * b / CS <= cs (one division)
        int owner = (int)tmin<int64_t>(CS - 1, (cs * CS) / n);
        while (owner > 0 && n * owner / CS > cs) --owner;
        while (owner + 1 < CS && n * (owner + 1) / CS <= cs) ++owner;
        const int64_t oc0 = n * owner / CS;
        {   // copy the pivot column and its F row from the owner (one remote read each)
            const double* ycol = cluster.map_shared_rank(S.Ys, owner) + (cs - oc0);
            const double* fown = cluster.map_shared_rank(S.Fs, owner) + (cs - oc0);
            for (int64_t r = kk + threadIdx.x; r < m; r += kThreads) S.v[r] = ycol[r * g.ncl];
            for (int64_t q = threadIdx.x; q < kk; q += kThreads) S.z[q] = fown[q * g.ncl];
        }
        __syncthreads();
        stamp(1);
        double ss = 0.0;
        for (int64_t r = kk + threadIdx.x; r < m; r += kThreads) {
            const double acc = sub_dot(S.v[r], S.V + r, m, S.z, 1, kk);
            S.v[r] = acc;
            if (r > kk) ss = fma(acc, acc, ss);
        }
        ss = block_sum(ss, red);
        if (threadIdx.x == 0) {
            s_ab[0] = S.v[kk];
            s_ab[1] = ss;
        }
        __syncthreads();
        const double alpha = s_ab[0], xnorm = sqrt(s_ab[1]);
        double tau, beta, scal;
        if (xnorm == 0.0) {
            tau = 0.0;
            beta = alpha;
            scal = 0.0;
        } else {
            beta = -copysign(dlapy2(alpha, xnorm), alpha);
            tau = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        for (int64_t r = threadIdx.x; r < m; r += kThreads) {
            const double vr = r < kk ? 0.0 : (r == kk ? 1.0 : S.v[r] * scal);
            S.v[r] = vr;
            S.V[kk * m + r] = vr;
        }
        if (threadIdx.x == 0) {
            S.tau[kk] = tau;
            S.beta[kk] = beta;
            if (cs >= c0 && cs < c1) S.Rs[kk * g.ncl + (cs - c0)] = beta;
        }
        __syncthreads();  // v complete; z (the F row copy) consumed, S.z reused below
        stamp(2);
        // GEMV over owned remaining columns, one thread per column (short m)
        for (int jj = threadIdx.x; jj < nc; jj += kThreads) {
            if (S.pos[jj] <= kk) continue;
            const double* yc = S.Ys + jj;
            const int64_t ld = g.ncl;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            int64_t r = kk;
            for (; r + 3 < m; r += 4) {
                a0 = fma(yc[r * ld], S.v[r], a0);
                a1 = fma(yc[(r + 1) * ld], S.v[r + 1], a1);
                a2 = fma(yc[(r + 2) * ld], S.v[r + 2], a2);
                a3 = fma(yc[(r + 3) * ld], S.v[r + 3], a3);
            }
            for (; r < m; ++r) a0 = fma(yc[r * ld], S.v[r], a0);
            S.W[jj] = (a0 + a1) + (a2 + a3);
        }
        // z = V[:, :kk]^T v
        for (int64_t q = wid; q < kk; q += kWarps) {
            const double zq = warp_sum(lane_dot(S.V + q * m, S.v, kk, m));
            if (lane == 0) S.z[q] = zq;
        }
        __syncthreads();
        stamp(3);
        // F, row kk of R, norm downdate (thread per column), flagged recompute (warp per column)
        int any_flag = 0;
        for (int jj = threadIdx.x; jj < nc; jj += kThreads) {
            if (S.pos[jj] <= kk) continue;
            double f = S.W[jj], rk = S.Ys[kk * g.ncl + jj];
            for (int64_t q = 0; q < kk; ++q) {
                const double fq = S.Fs[q * g.ncl + jj];
                f = fma(-fq, S.z[q], f);
                rk = fma(-S.V[q * m + kk], fq, rk);
            }
            f *= tau;
            S.Fs[kk * g.ncl + jj] = f;
            rk -= f;
            S.Rs[kk * g.ncl + jj] = rk;
            const double vn1 = S.vn1[jj];
            S.W[jj] = 0.0;  // recompute flag
            if (kk < m - 1 && vn1 != 0.0) {
                double temp = fabs(rk) / vn1;
                temp = fmax(0.0, (1.0 + temp) * (1.0 - temp));
                const double ratio = vn1 / S.vn2[jj];
                if (temp * ratio * ratio <= tol3z) {
                    S.W[jj] = 1.0;
                    any_flag = 1;
                } else {
                    S.vn1[jj] = vn1 * sqrt(temp);
                }
            }
        }
        any_flag = __syncthreads_or(any_flag);
        stamp(4);
        for (int jj = wid; any_flag && jj < nc; jj += kWarps) {
            if (S.pos[jj] <= kk || S.W[jj] == 0.0) continue;
            double s2 = 0.0;
            for (int64_t r = kk + 1 + lane; r < m; r += 32) {
                double v = S.Ys[r * g.ncl + jj];
                for (int64_t q = 0; q <= kk; ++q) v = fma(-S.V[q * m + r], S.Fs[q * g.ncl + jj], v);
                s2 = fma(v, v, s2);
            }
            s2 = warp_sum(s2);
            if (lane == 0) {
                S.vn1[jj] = sqrt(s2);
                S.vn2[jj] = sqrt(s2);
            }
        }
        if (any_flag) __syncthreads();
        stamp(5);
        local_argmax(kk + 1, kk + 1, par ^ 1);
        stamp(6);
        cluster.sync();
        stamp(7);
    }

    // ---- outputs ----
    for (int jj = threadIdx.x; jj < nc; jj += kThreads) {
        const int64_t p = S.pos[jj];
        g.perm[p] = (int32_t)(c0 + jj);
        for (int64_t q = 0; q < k; ++q) g.Rtop[q * n + p] = (p >= q) ? S.Rs[q * g.ncl + jj] : 0.0;
    }
    if (b == 0) {
        if (g.Vout) {
            for (int64_t e = threadIdx.x; e < m * k; e += kThreads) g.Vout[e] = S.V[e];
            for (int64_t q = threadIdx.x; q < k; q += kThreads) g.tauout[q] = S.tau[q];
        }
        if (threadIdx.x == 0) {
            const double lead = fabs(S.beta[0]);
            int32_t nr = 0;
            if (lead != 0.0)
                for (int64_t q = 0; q < k; ++q) nr += fabs(S.beta[q]) > g.rank_tol * lead ? 1 : 0;
            *g.numerical_rank = nr;
        }
    }
    cluster.sync();  // keep every CTA's shared memory alive until remote reads finish
}

// Q[:, c] = H_0 H_1 ... H_c e_c  (dorgqr's explicit Q, first k columns)
__global__ void __launch_bounds__(kThreads) form_q_kernel(const double* __restrict__ V,
                                                          const double* __restrict__ tau,
                                                          int64_t m, int64_t k, double* Q) {
    __shared__ double red[kWarps];
    const int64_t c = blockIdx.x;
    double* q = Q + c * m;
    for (int64_t r = threadIdx.x; r < m; r += kThreads) q[r] = (r == c) ? 1.0 : 0.0;
    __syncthreads();
    for (int64_t h = c; h >= 0; --h) {
        const double* v = V + h * m;
        double s = 0.0;
        for (int64_t r = h + threadIdx.x; r < m; r += kThreads) s = fma(v[r], q[r], s);
        s = block_sum(s, red);
        const double t = tau[h] * s;
        for (int64_t r = h + threadIdx.x; r < m; r += kThreads) q[r] = fma(-t, v[r], q[r]);
        __syncthreads();
    }
}

// One thread per non-selected position p >= k: T[:, p-k] = R11^{-1} R12[:, p-k]
// by back substitution in the order of reference BLAS dtrsm (column sweep
// from the last row up), with LAPACK-side diagonal flooring
// (matrix_id.py:68-79).  T: row-major k x (n - k) scratch.
__global__ void id_solve_kernel(const double* __restrict__ Rtop, int64_t k, int64_t n,
                                double rank_tol, const int32_t* __restrict__ numerical_rank,
                                double* __restrict__ T) {
    const int64_t nt = n - k;
    const double lead = fabs(Rtop[0]);
    const bool deficient = *numerical_rank < k;
    const double floorv = rank_tol * lead;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nt;
         p += (int64_t)gridDim.x * blockDim.x) {
        if (lead == 0.0) {
            for (int64_t q = 0; q < k; ++q) T[q * nt + p] = 0.0;
            continue;
        }
        for (int64_t q = 0; q < k; ++q) T[q * nt + p] = Rtop[q * n + k + p];
        for (int64_t q = k - 1; q >= 0; --q) {
            double d = Rtop[q * n + q];
            if (deficient && fabs(d) < floorv) d = d < 0.0 ? -floorv : floorv;
            double tq = T[q * nt + p];
            if (tq != 0.0) {
                tq = tq / d;
                T[q * nt + p] = tq;
                for (int64_t i = 0; i < q; ++i)
                    T[i * nt + p] = fma(-tq, Rtop[i * n + q], T[i * nt + p]);
            }
        }
    }
}

// id_solve_kernel for k <= kSolveRegs: each thread's column of T lives in
// registers and R11 in shared memory; the same operations in the same order
// (bit-identical results), without a global read-modify-write per update.
constexpr int kSolveRegs = 24;
__global__ void __launch_bounds__(128) id_solve_reg_kernel(const double* __restrict__ Rtop,
                                                           int64_t k, int64_t n, double rank_tol,
                                                           const int32_t* __restrict__ numerical_rank,
                                                           double* __restrict__ T) {
    __shared__ double r11[kSolveRegs * kSolveRegs];
    const int64_t nt = n - k;
    const double lead = fabs(Rtop[0]);
    const bool deficient = *numerical_rank < k;
    const double floorv = rank_tol * lead;
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int q = e / (int)k, i = e % (int)k;
        double d = Rtop[q * n + i];
        if (q == i && deficient && fabs(d) < floorv) d = d < 0.0 ? -floorv : floorv;
        r11[q * kSolveRegs + i] = d;
    }
    __syncthreads();
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nt;
         p += (int64_t)gridDim.x * blockDim.x) {
        double tv[kSolveRegs];
#pragma unroll
        for (int q = 0; q < kSolveRegs; ++q) tv[q] = (q < k && lead != 0.0) ? Rtop[q * n + k + p] : 0.0;
        if (lead != 0.0) {
#pragma unroll
            for (int q = kSolveRegs - 1; q >= 0; --q) {
                if (q < k && tv[q] != 0.0) {
                    const double tq = tv[q] / r11[q * kSolveRegs + q];
                    tv[q] = tq;
#pragma unroll
                    for (int i = 0; i < q; ++i) tv[i] = fma(-tq, r11[i * kSolveRegs + q], tv[i]);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < kSolveRegs; ++q)
            if (q < k) T[q * nt + p] = tv[q];
    }
}

// P[q, perm[c]] = (c < k) ? (q == c) : T[q, c - k]   (row-major k x n)
__global__ void id_scatter_kernel(const double* __restrict__ T, const int32_t* __restrict__ perm,
                                  int64_t k, int64_t n, double* __restrict__ P) {
    const int64_t nt = n - k;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < k * n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = e / n, c = e % n;
        const int64_t col = perm[c];
        P[q * n + col] = (c < k) ? (q == c ? 1.0 : 0.0) : T[q * nt + (c - k)];
    }
}

// Flags of the decomposition: bit 0 = numerically rank deficient; bit 1 =
// the solve met an exactly zero R11 diagonal (lead != 0, cols > k and a zero
// floor: rank_tol == 0 or rank_tol * |r00| underflowing), where the
// reference's triangular_solve raises SingularTriangleError (linalg.py:141-144)
// -- the first such index in bits 2.. .
__global__ void deficient_kernel(const int32_t* nr, const double* __restrict__ Rtop, int64_t k,
                                 int64_t cols, double rank_tol, int32_t* deficient) {
    const bool def = *nr < k;
    int32_t out = def ? 1 : 0;
    const double lead = fabs(Rtop[0]);
    const double floorv = rank_tol * lead;
    if (lead != 0.0 && cols > k && !(def && floorv > 0.0)) {
        for (int64_t q = 0; q < k; ++q)
            if (Rtop[q * cols + q] == 0.0) {
                out |= 2 | (int32_t)(q << 2);
                break;
            }
    }
    *deficient = out;
}

// Generic triangular solve r x = b (reference dtrsm loop order), one thread
// per right-hand-side column.  r row-major n x n, b/x row-major n x m.
__global__ void trsm_kernel(const double* __restrict__ r, const double* __restrict__ b,
                            int64_t n, int64_t m, int lower, double* __restrict__ x) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < m;
         c += (int64_t)gridDim.x * blockDim.x) {
        for (int64_t i = 0; i < n; ++i) x[i * m + c] = b[i * m + c];
        if (!lower) {
            for (int64_t q = n - 1; q >= 0; --q) {
                double t = x[q * m + c];
                if (t != 0.0) {
                    t /= r[q * n + q];
                    x[q * m + c] = t;
                    for (int64_t i = 0; i < q; ++i) x[i * m + c] = fma(-t, r[i * n + q], x[i * m + c]);
                }
            }
        } else {
            for (int64_t q = 0; q < n; ++q) {
                double t = x[q * m + c];
                if (t != 0.0) {
                    t /= r[q * n + q];
                    x[q * m + c] = t;
                    for (int64_t i = q + 1; i < n; ++i)
                        x[i * m + c] = fma(-t, r[i * n + q], x[i * m + c]);
                }
            }
        }
    }
}

template <class W>
void carve_cpqr(W& ws, int64_t m, int64_t n, int64_t k, int64_t G, CpqrArgs& a) {
    a.vn1 = ws.template take<double>(n);
    a.vn2 = ws.template take<double>(n);
    a.F = ws.template take<double>(n * k);
    a.Rcol = ws.template take<double>(n * k);
    a.W = ws.template take<double>(n * ceil_div(m, (int64_t)kSeg));
    a.V = ws.template take<double>(m * k);
    a.tau = ws.template take<double>(k);
    a.beta = ws.template take<double>(k);
    a.a = ws.template take<double>(ceil_div(m, (int64_t)kSeg) * kSeg);
    a.normpart = ws.template take<double>(G);
    a.zpart = ws.template take<double>(G * k);
    a.pos = ws.template take<int64_t>(n);
    a.flag_list = ws.template take<int64_t>(n);
    a.amax = ws.template take<ArgMax>(G);
}

struct CountCarve {
    size_t off = 0;
    template <class T>
    T* take(size_t cnt) {
        off = align_up(off, 256) + cnt * sizeof(T);
        return nullptr;
    }
};

int grid_size(int64_t m, int64_t n, size_t smem) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cpqr_kernel, kThreads, smem);
    if (per_sm < 1) per_sm = 1;
    // about one warp per owned column; tiny problems use few CTAs (cheap barriers)
    // (tall sketches: the whole GPU, the GEMV units are spread over every warp)
    const int64_t want = m > 1024 ? (int64_t)sms
                                  : tmax<int64_t>(1, tmin<int64_t>(ceil_div(n, kWarps), (int64_t)sms));
    const int64_t by_size = tmax<int64_t>(1, ceil_div(m * n, 2048));
    return (int)tmin<int64_t>((int64_t)sms * per_sm, tmin(want, by_size));
}

constexpr int64_t kMaxG = 148;



int64_t* g_cpqr_tlog = nullptr;  // debug: per-phase timing of the cooperative kernel

}  // namespace

// Debug hook: accumulate per-phase ns of cpqr_kernel into `buf` (device
// int64[16], [15] = flagged-column count); NULL disables.
extern "C" void ids_debug_cpqr_timing(int64_t* buf) { g_cpqr_tlog = buf; }

extern "C" size_t ids_cpqr_workspace_bytes(int64_t rows, int64_t cols, int64_t k) {
    CountCarve c;
    CpqrArgs a{};
    carve_cpqr(c, rows, cols, k, kMaxG, a);
    return c.off + 256;
}

extern "C" int ids_cpqr_trunc_f64(const double* Y, int64_t rows, int64_t cols, int64_t ldy,
                                  int64_t k, double rank_tol, int32_t* perm, double* Rtop,
                                  double* Q, int32_t* numerical_rank, void* workspace,
                                  size_t ws_bytes, void* stream) {
    return ids_cpqr_trunc_norms_f64(Y, rows, cols, ldy, k, rank_tol, nullptr, perm, Rtop, Q,
                                    numerical_rank, workspace, ws_bytes, stream);
}

extern "C" int ids_cpqr_trunc_norms_f64(const double* Y, int64_t rows, int64_t cols, int64_t ldy,
                                        int64_t k, double rank_tol, const double* colnorm2,
                                        int32_t* perm, double* Rtop, double* Q,
                                        int32_t* numerical_rank, void* workspace,
                                        size_t ws_bytes, void* stream) {
    if (rows < 1 || cols < 1 || k < 1 || k > rows || k > cols || ldy < rows || k > 64 * 1024) {
        ids_set_last_error("cpqr: bad arguments (need 1 <= k <= min(rows, cols))");
        return IDS_EINVAL;
    }
    cudaStream_t st = as_stream(stream);
    {   // short sketch: one cluster with Y in shared memory
        for (int csz : {8, 16}) {
            const int ncl = (int)ceil_div(cols, csz);
            const size_t cs_smem = cluster_smem_bytes(rows, k, ncl);
            if (cols < 2 * csz || cs_smem > 200 * 1024) continue;
            if (rows * cols < 4096) break;  // tiny: the cooperative kernel is fine
            ClusterArgs ca{};
            ca.Y = Y;
            ca.m = rows;
            ca.n = cols;
            ca.ldy = ldy;
            ca.k = k;
            ca.rank_tol = rank_tol;
            ca.perm = perm;
            ca.Rtop = Rtop;
            ca.numerical_rank = numerical_rank;
            ca.ncl = ncl;
            ca.tlog = g_cpqr_tlog;
            WsCarve wsc(workspace, ws_bytes);
            ca.Vout = wsc.take<double>((size_t)rows * k);
            ca.tauout = wsc.take<double>((size_t)k);
            if (!wsc.ok()) break;
            IDS_CUDA_TRY(cudaFuncSetAttribute(cpqr_cluster_kernel,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)cs_smem));
            if (csz > 8)
                IDS_CUDA_TRY(cudaFuncSetAttribute(cpqr_cluster_kernel,
                                                  cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(csz);
            cfg.blockDim = dim3(kThreads);
            cfg.dynamicSmemBytes = cs_smem;
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = csz;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            int clusters = 0;
            if (cudaOccupancyMaxActiveClusters(&clusters, cpqr_cluster_kernel, &cfg) != cudaSuccess ||
                clusters < 1) {
                cudaGetLastError();
                continue;
            }
            IDS_CUDA_TRY(cudaLaunchKernelEx(&cfg, cpqr_cluster_kernel, ca));
            ids_count_launch();
            if (Q) {
                form_q_kernel<<<(unsigned)k, kThreads, 0, st>>>(ca.Vout, ca.tauout, rows, k, Q);
                IDS_LAUNCH_CHECK();
            }
            return IDS_OK;
        }
    }
    // shared memory: v (whole, short sketches) or the window of v rows this
    // CTA's GEMV units touch (tall sketches), then z and row kk of V
    const int64_t mpad = ceil_div(rows, (int64_t)kSeg) * kSeg;
    const bool small = rows <= 1024;
    const int G = (int)tmin<int64_t>(
        grid_size(rows, cols, (size_t)((small ? mpad : 0) + 2 * k) * sizeof(double)), kMaxG);
    const int64_t nseg = mpad / kSeg;
    const int64_t vwin = small ? mpad : (ceil_div(nseg * cols, G) / cols + 2) * kSeg;
    const size_t smem = (size_t)(vwin + 2 * k) * sizeof(double);
    if (smem > 200 * 1024) {
        ids_set_last_error("cpqr: rank too large for the shared-memory z buffer");
        return IDS_EINVAL;
    }
    if (smem > 40 * 1024)
        IDS_CUDA_TRY(cudaFuncSetAttribute(cpqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
    CpqrArgs a{};
    a.Y = Y;
    a.m = rows;
    a.n = cols;
    a.ldy = ldy;
    a.k = k;
    a.rank_tol = rank_tol;
    a.small = small ? 1 : 0;
    a.vwin = vwin;
    a.colnorm2 = colnorm2;
    a.perm = perm;
    a.Rtop = Rtop;
    a.numerical_rank = numerical_rank;
    a.tlog = g_cpqr_tlog;
    WsCarve ws(workspace, ws_bytes);
    carve_cpqr(ws, rows, cols, k, kMaxG, a);
    if (!ws.ok()) {
        ids_set_last_error("cpqr: workspace too small");
        return IDS_EWORKSPACE;
    }
    void* args[] = {&a};
    IDS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)cpqr_kernel, dim3(G), dim3(kThreads),
                                             args, smem, st));
    ids_count_launch();
    if (Q) {
        form_q_kernel<<<(unsigned)k, kThreads, 0, st>>>(a.V, a.tau, rows, k, Q);
        IDS_LAUNCH_CHECK();
    }
    return IDS_OK;
}

extern "C" size_t ids_id_coeffs_workspace_bytes(int64_t k, int64_t cols) {
    return (size_t)k * (size_t)(cols > k ? cols - k : 0) * sizeof(double) + 256;
}

extern "C" int ids_id_coeffs_f64(const double* Rtop, const int32_t* perm, int64_t k, int64_t cols,
                                 double rank_tol, const int32_t* numerical_rank, double* P,
                                 int32_t* deficient, void* workspace, size_t ws_bytes,
                                 void* stream) {
    if (k < 1 || cols < k) {
        ids_set_last_error("id coeffs: bad arguments");
        return IDS_EINVAL;
    }
    cudaStream_t st = as_stream(stream);
    // T = R11^{-1} R12 in position order (k x (cols - k)), then scattered into P
    WsCarve ws(workspace, ws_bytes);
    const int64_t nt = cols - k;
    double* T = nt > 0 ? ws.take<double>((size_t)k * nt) : nullptr;
    if (!ws.ok()) {
        ids_set_last_error("id coeffs: workspace too small");
        return IDS_EWORKSPACE;
    }
    if (nt > 0) {
        const unsigned g = (unsigned)tmin<int64_t>(ceil_div(nt, 128), 148 * 8);
        if (k <= kSolveRegs)
            id_solve_reg_kernel<<<g, 128, 0, st>>>(Rtop, k, cols, rank_tol, numerical_rank, T);
        else
            id_solve_kernel<<<g, 128, 0, st>>>(Rtop, k, cols, rank_tol, numerical_rank, T);
        IDS_LAUNCH_CHECK();
    }
    const unsigned g2 = (unsigned)tmin<int64_t>(ceil_div(k * cols, 256), 148 * 8);
    id_scatter_kernel<<<g2, 256, 0, st>>>(T, perm, k, cols, P);
    IDS_LAUNCH_CHECK();
    if (deficient) {
        deficient_kernel<<<1, 1, 0, st>>>(numerical_rank, Rtop, k, cols, rank_tol, deficient);
        IDS_LAUNCH_CHECK();
    }
    return IDS_OK;
}

extern "C" int ids_triangular_solve_f64(const double* r, const double* b, int64_t n, int64_t m,
                                        int lower, double* x, int64_t* bad_index, void* stream) {
    if (n < 1 || m < 0) {
        ids_set_last_error("triangular solve: bad shape");
        return IDS_EINVAL;
    }
    cudaStream_t st = as_stream(stream);
    // diagonal to the host (strided copy), checked there (linalg.py:141-144)
    double* diag = static_cast<double*>(malloc(sizeof(double) * n));
    if (!diag) return IDS_EINVAL;
    cudaError_t e = cudaMemcpy2DAsync(diag, sizeof(double), r, sizeof(double) * (n + 1),
                                      sizeof(double), n, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        free(diag);
        ids_set_last_error(cudaGetErrorString(e));
        return IDS_ECUDA;
    }
    int64_t h = -1;
    for (int64_t i = 0; i < n; ++i)
        if (diag[i] == 0.0) {
            h = i;
            break;
        }
    free(diag);
    if (h != -1) {
        if (bad_index) *bad_index = h;
        ids_set_last_error("zero diagonal entry");
        return IDS_ESINGULAR;
    }
    if (m == 0) return IDS_OK;
    const unsigned g = (unsigned)tmin<int64_t>(ceil_div(m, 128), 148 * 8);
    trsm_kernel<<<g, 128, 0, st>>>(r, b, n, m, lower, x);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}
