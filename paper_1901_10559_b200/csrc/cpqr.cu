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




// ---- tall sketches: column ownership, two barriers per step ----------------
// For m > 1024 rows (C4: 4096 x 1000, C5: 16384 x 2000).  CTA b owns a
// contiguous block of COLUMNS for the whole factorization and keeps the full
// Householder vector v in shared memory, so the GEMV W_j = Y[:, j]^T v of
// its columns, their F entries, row kk of R and the norm downdates all stay
// on the CTA: no W partials cross CTAs.  Rows are split across CTAs only for
// the pivot column's residual a = Y[:, p] - V F[p, :]^T, whose norm and
// z~ = V^T a partials ride on the first barrier: the LAST CTA to arrive sums
// them (fixed order) before releasing it; the second barrier likewise
// reduces the argmax candidates to the next pivot.  A step is
//   S1 residual rows -> [barrier A: norm, z~] -> S2 Householder, v into
//   shared memory, GEMV, F / R / downdate, argmax -> [barrier B: pivot],
// against three grid syncs and two all-CTA partial reductions before.
constexpr int kTThreads = 512;
constexpr int kTWarps = kTThreads / 32;
constexpr int kMaxOwn = 64;  // owned columns per CTA
constexpr int kTallMaxK = 256;
constexpr int kMaxSegT = 16;  // v segments (rows <= 16 x 2048)

struct TallArgs {
    const double* Y;
    int64_t m, n, ldy, k;
    const double* colnorm2;
    double rank_tol;
    int32_t* perm;
    double* Rtop;
    int32_t* numerical_rank;
    double *F, *Rcol, *V, *tau, *beta, *a, *normpart, *zpart, *red;
    int64_t* piv;
    int64_t* flag_list;
    ArgMax* amax;
    unsigned* bar;
    int64_t* tlog;
    int pin_segs;  // leading 2048-row segments of each column kept in L2 (evict_last)
    int tmem;      // resident units in tensor memory
    float pin_frac;  // fraction of segment pin_segs also kept (evict_last)
};

__device__ __forceinline__ double block_sum_t(double v, double* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < kTWarps; ++i) s += red[i];
    return s;
}

// Grid barrier whose LAST arriving CTA runs `last()` (all its threads) before
// releasing the others; bar[0] counts arrivals, bar[1] is the generation.
template <class Fn>
__device__ __forceinline__ void bar_last(unsigned* bar, unsigned nblocks, Fn&& last) {
    __shared__ int s_last;
    __shared__ unsigned s_gen;
    __syncthreads();
    if (threadIdx.x == 0) {
        s_gen = *((volatile unsigned*)bar + 1);
        __threadfence();
        s_last = atomicAdd(bar, 1u) == nblocks - 1;
        if (s_last) __threadfence();
    }
    __syncthreads();
    if (s_last) {
        last();
        __syncthreads();
        if (threadIdx.x == 0) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        }
    } else if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        while (*gen == s_gen) {
        }
        __threadfence();
    }
    __syncthreads();
}

// Grid barrier on a monotonic arrival counter: every CTA posts one release-add
// and polls with acquire loads until the count reaches its target (number of
// barriers passed x grid size) -- one posted reduction and one polling round
// trip, no reset.  ctr must be zero at launch.
__device__ __forceinline__ void grid_bar_count(unsigned* ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

// y - sum_q a[q*lda] * b[q*ldb] with the b operand read through L2 (entries
// written by other CTAs)
__device__ __forceinline__ double sub_dot_cg(double y, const double* __restrict__ a, int64_t lda,
                                             const double* b, int64_t ldb, int64_t n) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int64_t q = 0;
    for (; q + 4 <= n; q += 4) {
        s0 = fma(a[q * lda], __ldcg(b + q * ldb), s0);
        s1 = fma(a[(q + 1) * lda], __ldcg(b + (q + 1) * ldb), s1);
        s2 = fma(a[(q + 2) * lda], __ldcg(b + (q + 2) * ldb), s2);
        s3 = fma(a[(q + 3) * lda], __ldcg(b + (q + 3) * ldb), s3);
    }
    for (; q < n; ++q) s0 = fma(a[q * lda], __ldcg(b + q * ldb), s0);
    return y - ((s0 + s1) + (s2 + s3));
}

static_assert(sizeof(ArgMax) == 32, "ArgMax is read as two 16-byte words");

// reduce_partials_warp with the candidates read through L2 (written by the
// other CTAs since this CTA last read them).
__device__ ArgMax reduce_partials_warp_cg(const ArgMax* part, int64_t G) {
    const int lane = threadIdx.x & 31;
    ArgMax best{-1.0, INT64_MAX, -1, -1};
    for (int64_t i0 = 0; i0 < G; i0 += 160) {  // one batch of loads for G <= 160
        ArgMax o[5];
#pragma unroll
        for (int u = 0; u < 5; ++u) {
            const int64_t i = i0 + lane + 32 * u;
            if (i < G) {
                const double2* w = reinterpret_cast<const double2*>(part + i);
                const double2 w0 = __ldcg(w), w1 = __ldcg(w + 1);
                o[u] = ArgMax{w0.x, __double_as_longlong(w0.y), __double_as_longlong(w1.x),
                              __double_as_longlong(w1.y)};
            } else {
                o[u] = ArgMax{-1.0, INT64_MAX, -1, -1};
            }
        }
#pragma unroll
        for (int u = 0; u < 5; ++u) {
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

// Fixed-order sum of G contiguous partials by one warp, read through L2.
__device__ __forceinline__ double warp_sum_partials_cg(const double* p, int64_t G) {
    const int lane = threadIdx.x & 31;
    double s = 0.0;
    for (int64_t i0 = 0; i0 < G; i0 += 256) {
        double t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t i = i0 + lane + 32 * u;
            t[u] = i < G ? __ldcg(p + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) s += t[u];
    }
    return warp_sum(s);
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ int64_t ceil_div_d(int64_t a, int64_t b) { return (a + b - 1) / b; }

// 16 doubles of this thread's TMEM lane (32 consecutive 32-bit columns)
__device__ __forceinline__ void tm_st_x32(uint32_t ta, const double* v) {
    uint32_t r[32];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        r[2 * i] = (uint32_t)__double2loint(v[i]);
        r[2 * i + 1] = (uint32_t)__double2hiint(v[i]);
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(ta),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ void tm_ld_x32(uint32_t ta, double* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(ta)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
}

__device__ __forceinline__ double2 ld_pol2(const double* p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p), "l"(pol));
    return v;
}

// Y loads with an L2 eviction policy: the pinned segments of every column
// (read again by each of the k GEMV passes) evict_last, the rest evict_first
__device__ __forceinline__ double ld_pol(const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}

// SEG: rows of one GEMV unit (2048 for tall sketches; 256 for short, wide
// ones such as C3's 200 x 10000)
template <int SEG>
__global__ void __launch_bounds__(kTThreads, 1) cpqr_tall_kernel(TallArgs g) {
    constexpr int kSegT = SEG;
    constexpr int kSegTLoads = kSegT / 32 / 4;  // loads per lane per quarter unit
    extern __shared__ double vsm[];
    const int64_t m = g.m, n = g.n, k = g.k, ldy = g.ldy;
    const int64_t mpad = (m + kSegT - 1) / kSegT * kSegT;
    const int nsegT = (int)(mpad / kSegT);
    const int G = gridDim.x, b = blockIdx.x;
    const int64_t rmax = (m + G - 1) / G;
    // shared memory: v | GEMV partials | z | row kk of V | F[cs, :] | owned
    // columns' norms, Y[kk, j], F rows | owned rows of V | positions
    double* part = vsm + mpad;                 // kMaxOwn x nsegT
    double* zsh = part + kMaxOwn * nsegT;      // k
    double* vrow = zsh + k;                    // k: V[kk, :kk]
    double* fpiv = vrow + k;                   // k: F[cs, :kk]
    double* svn1 = fpiv + k;                   // kMaxOwn
    double* svn2 = svn1 + kMaxOwn;
    double* sykk = svn2 + kMaxOwn;             // Y[kk, j] of the owned columns
    double* fown = sykk + kMaxOwn;             // kMaxOwn x k: F[j, :] of the owned columns
    double* vown = fown + kMaxOwn * k;         // rmax x k: V[r, :] of the owned rows
    int64_t* spos = reinterpret_cast<int64_t*>(vown + rmax * k);
    __shared__ double red[kTWarps];
    __shared__ double zacc[kTThreads];  // a[r] of the owned rows below kk
    __shared__ ArgMax wbest[kTWarps];
    __shared__ int s_nflag;
    __shared__ int64_t s_piv[3];
    __shared__ double s_nrm;
    __shared__ __align__(8) uint64_t s_mb[kMaxSegT];  // one per v segment
    __shared__ double s_scal, s_tau, s_beta;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t c0 = n * b / G, c1 = n * (b + 1) / G, nown = c1 - c0;
    const int64_t r0 = m * b / G, r1 = m * (b + 1) / G, nrow = r1 - r0;
    const double tol3z = sqrt(DBL_EPSILON);
    int64_t* flagged = g.flag_list + c0;
    unsigned nbar = 0;
    // resident units: warp w keeps (column w / Sres, segment pin + w % Sres),
    // one of the non-pinned segments, in its quarter of TMEM (128 columns x
    // 32 lanes = 2048 doubles)
    const int64_t pin = tmin<int64_t>(g.pin_segs, nsegT);
    const int64_t Sres = nsegT - pin;
    const int nres = (SEG == 2048 && g.tmem) ? (int)tmin<int64_t>(kTWarps, Sres > 0 ? nown * Sres : 0) : 0;
    __shared__ uint32_t s_tm;
    if (g.tmem && wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&s_tm))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm_base = g.tmem ? s_tm : 0u;
    uint64_t pol_keep, pol_stream, pol_half;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
    // the next segment: a fraction of its lines evict_last, the rest evict_first
    const float pin_frac = g.pin_frac;
    asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;"
                 : "=l"(pol_half)
                 : "f"(pin_frac));

    auto local_argmax = [&](int64_t pmin, int64_t pnext) {  // warp 0 (nown <= 64)
        if (wid != 0) return;
        ArgMax best{-1.0, INT64_MAX, -1, -1};
        for (int64_t jj = lane; jj < nown; jj += 32) {
            const int64_t pj = spos[jj];
            if (pj == pnext) best.col_at_next = c0 + jj;
            if (pj >= pmin && better(svn1[jj], pj, best.val, best.pos)) {
                best.val = svn1[jj];
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
        if (lane == 0) g.amax[b] = best;
    };

    // ---- prologue: zero v (its padding stays zero), owned columns' norms ----
    for (int64_t r = threadIdx.x; r < mpad; r += kTThreads) vsm[r] = 0.0;
    if (threadIdx.x == 0) {
        for (int sg = 0; sg < nsegT; ++sg)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&s_mb[sg])) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    for (int64_t jj = wid; jj < nown; jj += kTWarps) {
        const int64_t j = c0 + jj;
        const double* y = g.Y + j * ldy;
        const double s2 = g.colnorm2 ? g.colnorm2[j] : warp_sum(lane_dot(y, y, 0, m));
        if (lane == 0) {
            svn1[jj] = sqrt(s2);
            svn2[jj] = sqrt(s2);
            spos[jj] = j;
        }
    }
    __syncthreads();
    local_argmax(0, 0);
    grid_bar_count(g.bar, (unsigned)(++nbar * G));

    // debug timing: phase durations of CTA 0, thread 0, kept in shared memory
    // (a global read-modify-write per stamp would itself cost a round trip)
    __shared__ int64_t s_tacc[16];
    const bool tl = g.tlog && b == 0 && threadIdx.x == 0;
    if (tl)
        for (int i = 0; i < 16; ++i) s_tacc[i] = 0;
    int64_t tprev = tl ? gtimer() : 0;
    auto stamp = [&](int phase) {
        if (tl) {
            const int64_t t = gtimer();
            s_tacc[phase] += t - tprev;
            tprev = t;
        }
    };
    for (int64_t kk = 0; kk < k; ++kk) {
        // ---- S1: the pivot (every CTA reduces the candidates itself), row kk
        // of V, positions, the pivot column's residual on the owned rows ----
        if (wid == 0) {
            const ArgMax r = reduce_partials_warp_cg(g.amax, G);
            if (lane == 0) {
                s_piv[0] = r.col;
                s_piv[1] = r.pos;
                s_piv[2] = r.col_at_next;
            }
        } else {
            for (int64_t q = threadIdx.x - 32; q < kk; q += kTThreads - 32)
                vrow[q] = __ldcg(g.V + q * m + kk);  // V[kk, q]
        }
        __syncthreads();
        stamp(8);
        int64_t cs = s_piv[0], ps = s_piv[1];
        const int64_t ck = s_piv[2];
        if (cs < 0) {  // every remaining norm is NaN (non-finite input): keep position kk
            cs = ck;
            ps = kk;
        }
        if (threadIdx.x == 0) {
            if (ck >= c0 && ck < c1 && ck != cs) spos[ck - c0] = ps;
            if (cs >= c0 && cs < c1) spos[cs - c0] = kk;
        }
        const int64_t rr = r0 + threadIdx.x;
        const double yrr = (threadIdx.x < nrow && rr >= kk) ? __ldg(g.Y + cs * ldy + rr) : 0.0;
        for (int64_t q = threadIdx.x; q < kk; q += kTThreads) fpiv[q] = __ldcg(g.F + q * n + cs);
        __syncthreads();
        stamp(9);
        double av = 0.0;
        if (threadIdx.x < nrow && rr >= kk) {  // a[r] = Y[r, cs] - V[r, :kk] F[cs, :kk]^T
            const double* vr = vown + threadIdx.x * k;
            double s4[4] = {0.0, 0.0, 0.0, 0.0};
            for (int64_t q = 0; q < kk; ++q) s4[q & 3] = fma(vr[q], fpiv[q], s4[q & 3]);
            av = yrr - ((s4[0] + s4[1]) + (s4[2] + s4[3]));
        }
        if (threadIdx.x < nrow) {
            g.a[rr] = rr == kk ? 0.0 : av;  // v's row kk enters the GEMV as Y[kk, j]
            if (rr == kk) g.red[0] = av;      // alpha
        }
        const double ac = rr > kk ? av : 0.0;  // rows below kk enter the norm and z~
        const double ss = block_sum_t(ac * ac, red);
        if (threadIdx.x == 0) g.normpart[b] = ss;
        stamp(10);
        // z~_q partial = V[r0:r1, q]^T a over the owned rows (threads < nrow)
        // (16 threads per q, rows strided by 16, a fixed shuffle tree)
        if (threadIdx.x < nrow) zacc[threadIdx.x] = ac;
        __syncthreads();
        for (int64_t q0 = 0; q0 < kk; q0 += kTThreads / 16) {
            const int64_t q = q0 + (threadIdx.x >> 4);
            const int sub = threadIdx.x & 15;
            double x = 0.0;
            if (q < kk)
                for (int64_t rl = sub; rl < nrow; rl += 16) x = fma(vown[rl * k + q], zacc[rl], x);
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            if (q < kk && sub == 0) g.zpart[q * G + b] = x;
        }
        stamp(0);
        grid_bar_count(g.bar, (unsigned)(++nbar * G));
        stamp(1);

        // ---- S2: a[] into shared memory by one bulk copy per 2048-row segment
        // (each GEMV unit waits only for its own segment), ||a[kk+1:]|| (fixed-
        // order sum of the partials) and the Householder scalars ----
        if (wid == 0 && lane < nsegT) {  // one lane per segment issues its copy
            asm volatile("fence.proxy.async;" ::: "memory");
            {
                const int sg = lane;
                const int64_t lo = (int64_t)sg * kSegT, hi = tmin<int64_t>(m, lo + kSegT);
                const uint32_t bytes = (uint32_t)(((hi - lo + 1) / 2) * 16);  // a[m] is a zero pad
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                                 smem_addr(&s_mb[sg])),
                             "r"(bytes)
                             : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_addr(vsm + lo)),
                    "l"(g.a + lo), "r"(bytes), "r"(smem_addr(&s_mb[sg]))
                    : "memory");
            }
        }
        if (wid == 1) {
            const double x = warp_sum_partials_cg(g.normpart, G);
            if (lane == 0) {
                const double alpha = __ldcg(g.red);
                const double xnorm = sqrt(x);
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
                s_scal = scal;
                s_tau = tau;
                s_beta = beta;
            }
        }
        if (threadIdx.x == 0) s_nflag = 0;
        for (int64_t jj = threadIdx.x; jj < nown; jj += kTThreads) sykk[jj] = __ldg(g.Y + (c0 + jj) * ldy + kk);
        stamp(2);
        auto wait_seg = [&](int64_t sg) {
            asm volatile(
                "{\n\t.reg .pred p;\n"
                "CPQR_WAIT_%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                "@!p bra CPQR_WAIT_%=;\n}" ::"r"(smem_addr(&s_mb[sg])),
                "r"((uint32_t)(kk & 1))
                : "memory");
        };

        // ---- GEMV over the owned columns: units (column, 2048-row segment).
        // Warp w's resident unit (one non-pinned segment) lives in TENSOR MEMORY
        // after the first pass; the other units stream from L2 (pinned
        // segments) or DRAM, two per warp at a time, walked backwards on odd
        // steps ----
        {
            if (SEG == 2048 && wid < nres) {  // this warp's resident unit
                const int64_t jr = (int64_t)wid / Sres, sr = pin + (int64_t)wid % Sres;
                const uint32_t ta = tm_base + ((uint32_t)(32 * (wid & 3)) << 16) + (uint32_t)((wid >> 2) * 128);
                const bool act = spos[jr] > kk;
                const double* pr = g.Y + (c0 + jr) * ldy;
                double s1 = 0.0, t1 = 0.0;
#pragma unroll 1
                for (int qtr = 0; qtr < 4; ++qtr) {
                    const int64_t br = sr * kSegT + qtr * (kSegT / 4) + lane;
                    double yr[kSegTLoads];
                    if (kk == 0) {  // first pass: from memory, kept in TMEM
#pragma unroll
                        for (int u = 0; u < kSegTLoads; ++u)
                            yr[u] = __ldg(pr + tmin<int64_t>(br + 32 * u, m - 1));
                        tm_st_x32(ta + 32 * qtr, yr);
                    } else {
                        tm_ld_x32(ta + 32 * qtr, yr);
                    }
                    if (qtr == 0) wait_seg(sr);
                    if (act) {
#pragma unroll
                        for (int u = 0; u < kSegTLoads; u += 2) {
                            s1 = fma(yr[u], vsm[br + 32 * u], s1);
                            t1 = fma(yr[u + 1], vsm[br + 32 * u + 32], t1);
                        }
                    }
                }
                if (kk == 0) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                const double wr = warp_sum(s1 + t1);
                if (lane == 0 && act) part[jr * nsegT + sr] = wr;
            }
            const int64_t U = nown * nsegT - nres;  // streamed units
            const int64_t npin = nown * pin;
            auto unit_of = [&](int64_t li, int64_t& j, int64_t& sg) {
                if (li < npin) {
                    j = li / pin;
                    sg = li % pin;
                } else {
                    const int64_t e = nres + (li - npin);
                    j = e / Sres;
                    sg = pin + e % Sres;
                }
            };
            const bool rev = kk & 1;
            const bool full = m == mpad;
            // whole segments, even ldy and a 16-byte aligned Y: 16-byte loads
            const bool vec16 = full && (ldy & 1) == 0 && (reinterpret_cast<uintptr_t>(g.Y) & 15) == 0;
            for (int64_t li = wid; li < U; li += 2 * kTWarps) {
                const bool h2 = li + kTWarps < U;
                int64_t ja, sa, jb, sb;
                unit_of(rev ? U - 1 - li : li, ja, sa);
                unit_of(h2 ? (rev ? U - 1 - (li + kTWarps) : li + kTWarps) : (rev ? U - 1 - li : li), jb, sb);
                const bool aa = spos[ja] > kk, ab = h2 && spos[jb] > kk;
                const double* pa = g.Y + (c0 + ja) * ldy;
                const double* pb = g.Y + (c0 + jb) * ldy;
                const uint64_t pola = sa < pin ? pol_keep : (sa == pin && pin_frac > 0.f ? pol_half : pol_stream);
                const uint64_t polb = sb < pin ? pol_keep : (sb == pin && pin_frac > 0.f ? pol_half : pol_stream);
                double s1 = 0.0, s2 = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll 1
                for (int qtr = 0; qtr < 4 && vec16; ++qtr) {  // 16-byte loads: rows 2 lane + 64 u
                    const int64_t ba = sa * kSegT + qtr * (kSegT / 4) + 2 * lane;
                    const int64_t bb = sb * kSegT + qtr * (kSegT / 4) + 2 * lane;
                    double2 ya[kSegTLoads / 2], yb[kSegTLoads / 2];
#pragma unroll
                    for (int u = 0; u < kSegTLoads / 2; ++u) {
                        ya[u] = aa ? ld_pol2(pa + ba + 64 * u, pola) : make_double2(0.0, 0.0);
                        yb[u] = ab ? ld_pol2(pb + bb + 64 * u, polb) : make_double2(0.0, 0.0);
                    }
                    if (qtr == 0) {
                        wait_seg(sa);
                        wait_seg(sb);
                    }
#pragma unroll
                    for (int u = 0; u < kSegTLoads / 2; ++u) {
                        const double2 va = *reinterpret_cast<const double2*>(vsm + ba + 64 * u);
                        const double2 vb = *reinterpret_cast<const double2*>(vsm + bb + 64 * u);
                        s1 = fma(ya[u].x, va.x, s1);
                        t1 = fma(ya[u].y, va.y, t1);
                        s2 = fma(yb[u].x, vb.x, s2);
                        t2 = fma(yb[u].y, vb.y, t2);
                    }
                }
#pragma unroll 1
                for (int qtr = 0; qtr < 4 && !vec16; ++qtr) {
                    const int64_t ba = sa * kSegT + qtr * (kSegT / 4) + lane;
                    const int64_t bb = sb * kSegT + qtr * (kSegT / 4) + lane;
                    double ya[kSegTLoads], yb[kSegTLoads];
#pragma unroll
                    for (int u = 0; u < kSegTLoads; ++u) {
                        if (full) {
                            ya[u] = aa ? ld_pol(pa + ba + 32 * u, pola) : 0.0;
                            yb[u] = ab ? ld_pol(pb + bb + 32 * u, polb) : 0.0;
                        } else {
                            ya[u] = aa ? ld_pol(pa + tmin<int64_t>(ba + 32 * u, m - 1), pola) : 0.0;
                            yb[u] = ab ? ld_pol(pb + tmin<int64_t>(bb + 32 * u, m - 1), polb) : 0.0;
                        }
                    }
                    if (qtr == 0) {
                        wait_seg(sa);
                        wait_seg(sb);
                    }
#pragma unroll
                    for (int u = 0; u < kSegTLoads; u += 2) {
                        s1 = fma(ya[u], vsm[ba + 32 * u], s1);
                        s2 = fma(yb[u], vsm[bb + 32 * u], s2);
                        t1 = fma(ya[u + 1], vsm[ba + 32 * u + 32], t1);
                        t2 = fma(yb[u + 1], vsm[bb + 32 * u + 32], t2);
                    }
                }
                const double wa = warp_sum(s1 + t1), wb = warp_sum(s2 + t2);
                if (lane == 0) {
                    part[ja * nsegT + sa] = wa;
                    if (h2) part[jb * nsegT + sb] = wb;
                }
            }
        }
        __syncthreads();  // s_scal / s_tau / s_beta
        const double scal = s_scal, tau = s_tau, beta = s_beta;
        if (threadIdx.x < nrow) {  // V[r, kk] of the owned rows (global: other CTAs' row kk, form_q)
            const double vr = rr < kk ? 0.0 : rr == kk ? 1.0 : vsm[rr] * scal;
            vown[threadIdx.x * k + kk] = vr;
            g.V[kk * m + rr] = vr;
        }
        if (b == 0 && threadIdx.x == 0) {
            g.tau[kk] = tau;
            g.beta[kk] = beta;
        }
        if (threadIdx.x == 0 && cs >= c0 && cs < c1) g.Rcol[cs * k + kk] = beta;
        // z_q = V[:, q]^T v = V[kk, q] + scal * (fixed-order sum of the z~ partials)
        for (int64_t q = wid; q < kk; q += kTWarps) {
            const double x = warp_sum_partials_cg(g.zpart + q * G, G);
            if (lane == 0) zsh[q] = fma(scal, x, vrow[q]);
        }
        __syncthreads();
        stamp(3);

        // ---- F column, row kk of R, norm downdates (one warp per column) ----
        for (int64_t jj = wid; jj < nown; jj += kTWarps) {
            if (spos[jj] <= kk) continue;
            const int64_t j = c0 + jj;
            double wj = 0.0;
            for (int sg = 0; sg < nsegT; ++sg) wj += part[jj * nsegT + sg];  // fixed order
            wj = fma(scal, wj, sykk[jj]);
            double fz = 0.0, fv = 0.0;
            for (int64_t q = lane; q < kk; q += 32) {
                const double fq = fown[jj * k + q];
                fz = fma(fq, zsh[q], fz);
                fv = fma(fq, vrow[q], fv);
            }
            fz = warp_sum(fz);
            fv = warp_sum(fv);
            if (lane == 0) {
                const double f = (wj - fz) * tau;
                fown[jj * k + kk] = f;
                g.F[kk * n + j] = f;
                const double rk = (sykk[jj] - fv) - f;  // V[kk, kk] = 1
                g.Rcol[j * k + kk] = rk;
                const double vn1 = svn1[jj];
                if (kk < m - 1 && vn1 != 0.0) {
                    double temp = fabs(rk) / vn1;
                    temp = fmax(0.0, (1.0 + temp) * (1.0 - temp));
                    const double ratio = vn1 / svn2[jj];
                    const double temp2 = temp * ratio * ratio;
                    if (temp2 <= tol3z) flagged[atomicAdd(&s_nflag, 1)] = jj;
                    else svn1[jj] = vn1 * sqrt(temp);
                }
            }
        }
        __syncthreads();
        // exact norms of the flagged columns below row kk (LAPACK's recompute)
        const int nflag = s_nflag;
        for (int fi = wid; fi < nflag; fi += kTWarps) {
            const int64_t jj = flagged[fi], j = c0 + jj;
            const double* y = g.Y + j * ldy;
            double s = 0.0;
            for (int64_t r = kk + 1 + lane; r < m; r += 32) {
                double v = y[r];
                for (int64_t q = 0; q < kk; ++q) v = fma(-__ldcg(g.V + q * m + r), fown[jj * k + q], v);
                v = fma(-vsm[r] * scal, fown[jj * k + kk], v);
                s = fma(v, v, s);
            }
            s = warp_sum(s);
            if (lane == 0) {
                svn1[jj] = sqrt(s);
                svn2[jj] = sqrt(s);
            }
        }
        __syncthreads();
        stamp(4);
        local_argmax(kk + 1, kk + 1);
        stamp(14);
        grid_bar_count(g.bar, (unsigned)(++nbar * G));
        stamp(5);
    }

    if (tl)
        for (int i = 0; i < 16; ++i) g.tlog[i] += s_tacc[i];
    if (g.tmem) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (wid == 0)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm_base) : "memory");
    }
    // the pinned segments back to normal eviction priority
    if (g.pin_segs > 0) {
        const int64_t rows_pin = tmin<int64_t>(m, (int64_t)(g.pin_segs + (g.pin_frac > 0.f ? 1 : 0)) * kSegT);
        const int64_t lines = ceil_div_d(rows_pin * 8, 128);
        for (int64_t i = threadIdx.x; i < nown * lines; i += kTThreads) {
            const double* ln = g.Y + (c0 + i / lines) * ldy + (i % lines) * 16;
            asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(ln) : "memory");
        }
    }
    // ---- outputs: perm, Rtop, numerical rank ----
    for (int64_t jj = threadIdx.x; jj < nown; jj += kTThreads) {
        const int64_t j = c0 + jj, p = spos[jj];
        g.perm[p] = (int32_t)j;
        for (int64_t q = 0; q < k; ++q) g.Rtop[q * n + p] = (p >= q) ? g.Rcol[j * k + q] : 0.0;
    }
    if (b == 0 && threadIdx.x == 0) {
        const double lead = fabs(g.beta[0]);
        int32_t nr = 0;
        if (lead != 0.0)
            for (int64_t q = 0; q < k; ++q) nr += fabs(g.beta[q]) > g.rank_tol * lead ? 1 : 0;
        *g.numerical_rank = nr;
    }
}

// ---- short, wide sketches: column slices resident in shared memory ---------
// For m <= 1024 rows and many columns (C3: 200 x 10000).  CTA b owns a
// contiguous block of columns for the whole factorization and copies its
// slice of Y into shared memory once; it also keeps the rows of F, R and V it
// needs there, so the GEMV, the F / R columns, the downdates and the norm
// recomputes never touch global memory.  A step needs ONE grid barrier: each
// CTA publishes its argmax candidate TOGETHER with that column's residual
// a = Y[:, c] - V F[c, :]^T (computed by the owner from shared memory), so
// after the barrier every CTA agrees on the pivot, reads its residual from
// L2 and builds the Householder vector itself.  The arithmetic (operation
// order included) is that of cpqr_kernel's short-sketch path, so both give
// identical factors.
struct WideArgs {
    const double* Y;
    int64_t m, n, ldy, k;
    const double* colnorm2;
    double rank_tol;
    int32_t* perm;
    double* Rtop;
    int32_t* numerical_rank;
    double *V, *tau, *beta;  // global copies for form_q_kernel and the rank count
    ArgMax* amax;            // [2][G] candidates, by step parity
    double* apub;            // [2][G][m] candidate residuals, by step parity
    unsigned* bar;           // monotonic arrival counter (zero at launch)
    int64_t nc_max;          // owned columns per CTA (max)
    int64_t* tlog;
};

constexpr int64_t kWideMinCols = 256;

size_t wide_smem_bytes(int64_t m, int64_t k, int64_t nc) {
    // Ys (nc m), Vs (k m), Fs and Rs (nc k each), v and a (m each), z and
    // V[kk, :] (k each), vn1 / vn2 (nc each); pos (nc int64), flagged (nc int32)
    return (size_t)(nc * m + k * m + 2 * nc * (k | 1) + 2 * m + 2 * k + 2 * nc) * sizeof(double) +
           (size_t)nc * sizeof(int64_t) + (size_t)nc * sizeof(int32_t) + 64;
}

__global__ void __launch_bounds__(kThreads, 1) cpqr_wide_kernel(WideArgs g) {
    extern __shared__ double wsm[];
    const int64_t G = gridDim.x, b = blockIdx.x;
    const int64_t m = g.m, n = g.n, k = g.k, ldy = g.ldy;
    const int64_t c0 = n * b / G, c1 = n * (b + 1) / G, nc = c1 - c0;
    const int64_t ncm = g.nc_max;
    double* Ys = wsm;                 // ncm x m, column jl at Ys + jl m
    double* Vs = Ys + ncm * m;        // k x m: V[:, q] at Vs + q m
    const int64_t kp = k | 1;         // odd row stride: thread-per-column loops conflict-free
    double* Fs = Vs + k * m;          // F[q, c0 + jl] at Fs + jl kp + q
    double* Rs = Fs + ncm * kp;       // R[q, c0 + jl] at Rs + jl kp + q
    double* vsm = Rs + ncm * kp;      // v (m)
    double* asm_ = vsm + m;           // pivot residual a (m)
    double* zsh = asm_ + m;           // z (k)
    double* vrow = zsh + k;           // V[kk, :kk] (k)
    double* vn1 = vrow + k;           // ncm
    double* vn2 = vn1 + ncm;          // ncm
    int64_t* pos = reinterpret_cast<int64_t*>(vn2 + ncm);   // ncm
    int32_t* flagged = reinterpret_cast<int32_t*>(pos + ncm);  // ncm
    __shared__ int s_nflag;
    __shared__ double s_red0;
    __shared__ double red[kWarps];
    __shared__ ArgMax warp_best[kWarps];
    __shared__ int64_t s_piv[4];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const double tol3z = sqrt(DBL_EPSILON);

    // ---- prologue: the slice into shared memory (cp.async, all in flight) ----
    {
        const uint32_t ys = (uint32_t)__cvta_generic_to_shared(Ys);
        const int64_t tot = nc * m;
        for (int64_t e = threadIdx.x; e < tot; e += kThreads) {
            const int64_t jl = e / m, r = e - jl * m;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(ys + (uint32_t)(8 * e)),
                         "l"(g.Y + (c0 + jl) * ldy + r)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    }
    for (int64_t r = threadIdx.x; r < m; r += kThreads) vsm[r] = 0.0;
    __syncthreads();
    for (int64_t jl = wid; jl < nc; jl += kWarps) {
        const double s = g.colnorm2 ? g.colnorm2[c0 + jl] : warp_sum(lane_dot(Ys + jl * m, Ys + jl * m, 0, m));
        if (lane == 0) {
            vn1[jl] = sqrt(s);
            vn2[jl] = sqrt(s);
            pos[jl] = c0 + jl;
        }
    }
    __syncthreads();

    // local argmax over owned columns with pos >= step; publishes the
    // candidate and its residual (rows >= step, `step` terms of V F^T) into
    // buffer step & 1
    auto publish = [&](int64_t step) {
        ArgMax best{-1.0, INT64_MAX, -1, -1};
        for (int64_t jl = threadIdx.x; jl < nc; jl += kThreads) {
            const int64_t pj = pos[jl];
            if (pj == step) best.col_at_next = c0 + jl;
            if (pj >= step && better(vn1[jl], pj, best.val, best.pos)) {
                best.val = vn1[jl];
                best.pos = pj;
                best.col = c0 + jl;
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
            g.amax[(step & 1) * G + b] = r;
            // the column whose residual is published: the candidate, else (no
            // finite norm left here) the column at position `step`, if owned
            s_piv[3] = r.col >= 0 ? r.col : r.col_at_next;
        }
        __syncthreads();
        const int64_t pc = s_piv[3];
        if (pc >= 0 && step < k) {
            const int64_t jl = pc - c0;
            double* out = g.apub + ((step & 1) * G + b) * m;
            for (int64_t r = step + threadIdx.x; r < m; r += kThreads)
                out[r] = sub_dot(Ys[jl * m + r], Vs + r, m, Fs + jl * kp, 1, step);
        }
    };

    const bool tl = g.tlog && b == 0 && threadIdx.x == 0;
    int64_t tprev = tl ? gtimer() : 0;
    auto stamp = [&](int phase) {
        if (tl) {
            const int64_t t = gtimer();
            g.tlog[phase] += t - tprev;
            tprev = t;
        }
    };
    publish(0);
    grid_bar_count(g.bar, (unsigned)G);
    stamp(0);

    for (int64_t kk = 0; kk < k; ++kk) {
        // ---- pivot: reduce the candidates, fetch the winner's residual ----
        const ArgMax* cand = g.amax + (kk & 1) * G;
        if (wid == 0) {
            const ArgMax r = reduce_partials_warp_cg(cand, G);
            if (lane == 0) {
                s_piv[0] = r.col;
                s_piv[1] = r.pos;
                s_piv[2] = r.col_at_next;
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
            if (ck >= c0 && ck < c1 && ck != cs) pos[ck - c0] = ps;
            if (cs >= c0 && cs < c1) pos[cs - c0] = kk;
        }
        int64_t ob = cs * G / n;  // owner CTA of column cs
        while (ob + 1 < G && n * (ob + 1) / G <= cs) ++ob;
        while (ob > 0 && n * ob / G > cs) --ob;
        const double* ain = g.apub + ((kk & 1) * G + ob) * m;
        double ss = 0.0;
        for (int64_t r = kk + threadIdx.x; r < m; r += kThreads) {
            const double v = __ldcg(ain + r);
            asm_[r] = v;
            if (r > kk) ss = fma(v, v, ss);
        }
        ss = block_sum(ss, red);
        stamp(1);

        // ---- Householder vector (every CTA), z = V^T v, V[kk, :kk] ----
        const double alpha = asm_[kk];
        const double xnorm = sqrt(ss);
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
            const double v = r < kk ? 0.0 : (r == kk) ? 1.0 : asm_[r] * scal;
            vsm[r] = v;
            Vs[kk * m + r] = v;
            if (b == 0) g.V[kk * m + r] = v;
        }
        if (b == 0 && threadIdx.x == 0) {
            g.tau[kk] = tau;
            g.beta[kk] = beta;
        }
        if (threadIdx.x == 0 && cs >= c0 && cs < c1) Rs[(cs - c0) * kp + kk] = beta;
        __syncthreads();
        for (int64_t q = wid; q < kk; q += kWarps) {
            const double sz = warp_sum(lane_dot(Vs + q * m, vsm, kk, m));
            if (lane == 0) {
                zsh[q] = sz;
                vrow[q] = Vs[q * m + kk];
            }
        }
        if (threadIdx.x == 0) s_nflag = 0;
        stamp(2);
        // ---- GEMV W_j = Y[:, j]^T v over the owned columns: one warp per
        // column, four columns per warp side by side (rows lane + 32 t,
        // clamped to m - 1 where v is zero; two chains per column) ----
        {
            const int nl = (int)((m + 31) / 32);
            for (int64_t jb = 4 * wid; jb < nc; jb += 4 * kWarps) {
                const double* y[4];
                bool on[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    on[c] = jb + c < nc && pos[jb + c] > kk;
                    y[c] = Ys + (on[c] ? jb + c : jb) * m;
                }
                double s1[4] = {0.0, 0.0, 0.0, 0.0}, t1[4] = {0.0, 0.0, 0.0, 0.0};
                for (int t = 0; t < nl; t += 2) {
                    const int64_t ra = lane + 32 * t, rb = ra + 32;
                    const int64_t ca = tmin(ra, m - 1), cb = tmin(rb, m - 1);
                    const double va = ra < m ? vsm[ra] : 0.0, vb = rb < m ? vsm[rb] : 0.0;
                    const bool two = t + 1 < nl;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        s1[c] = fma(y[c][ca], va, s1[c]);
                        if (two) t1[c] = fma(y[c][cb], vb, t1[c]);
                    }
                }
                double w[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) w[c] = s1[c] + t1[c];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) w[c] += __shfl_xor_sync(0xffffffffu, w[c], o);
                }
                if (lane < 4 && on[lane]) {
                    double wl = w[0];
#pragma unroll
                    for (int c = 1; c < 4; ++c) wl = lane == c ? w[c] : wl;
                    Fs[(jb + lane) * kp + kk] = wl;  // W_j, turned into F[kk, j] below
                }
            }
        }
        __syncthreads();
        stamp(3);
        // ---- F column, row kk of R, norm downdate (one thread per column) ----
        for (int64_t jl = threadIdx.x; jl < nc; jl += kThreads) {
            if (pos[jl] <= kk) continue;
            const double wj = 0.0 + Fs[jl * kp + kk];
            double f = sub_dot(wj, Fs + jl * kp, 1, zsh, 1, kk);
            double rk = sub_dot(Ys[jl * m + kk], Fs + jl * kp, 1, vrow, 1, kk);
            f *= tau;
            Fs[jl * kp + kk] = f;
            rk -= f;  // V[kk, kk] = 1
            Rs[jl * kp + kk] = rk;
            const double v1 = vn1[jl];
            if (kk < m - 1 && v1 != 0.0) {
                double temp = fabs(rk) / v1;
                temp = fmax(0.0, (1.0 + temp) * (1.0 - temp));
                const double ratio = v1 / vn2[jl];
                const double temp2 = temp * ratio * ratio;
                if (temp2 <= tol3z) flagged[atomicAdd(&s_nflag, 1)] = (int32_t)jl;
                else vn1[jl] = v1 * sqrt(temp);
            }
        }
        __syncthreads();
        stamp(4);
        // exact norms of the flagged columns below row kk (LAPACK's recompute)
        const int nflag = s_nflag;
        if (g.tlog && threadIdx.x == 0) atomicAdd((unsigned long long*)&g.tlog[15], (unsigned long long)nflag);
        for (int fi = wid; fi < nflag; fi += kWarps) {
            const int64_t jl = flagged[fi];
            const double* y = Ys + jl * m;
            double s = 0.0;
            for (int64_t r = kk + 1 + lane; r < m; r += 32) {
                double v = sub_dot(y[r], Vs + r, m, Fs + jl * kp, 1, kk);
                v = fma(-vsm[r], Fs[jl * kp + kk], v);
                s = fma(v, v, s);
            }
            s = warp_sum(s);
            if (lane == 0) {
                vn1[jl] = sqrt(s);
                vn2[jl] = sqrt(s);
            }
        }
        __syncthreads();
        stamp(5);
        if (kk + 1 < k) {
            publish(kk + 1);
            stamp(6);
            grid_bar_count(g.bar, (unsigned)(G * (kk + 2)));
            stamp(7);
        }
    }

    // ---- outputs: perm, Rtop, numerical rank ----
    for (int64_t jl = threadIdx.x; jl < nc; jl += kThreads) {
        const int64_t p = pos[jl];
        g.perm[p] = (int32_t)(c0 + jl);
        for (int64_t q = 0; q < k; ++q) g.Rtop[q * n + p] = (p >= q) ? Rs[jl * kp + q] : 0.0;
    }
    if (b == 0 && threadIdx.x == 0) {
        const double lead = fabs(g.beta[0]);
        int32_t nr = 0;
        if (lead != 0.0)
            for (int64_t q = 0; q < k; ++q) nr += fabs(g.beta[q]) > g.rank_tol * lead ? 1 : 0;
        *g.numerical_rank = nr;
    }
}

template <class W>
void carve_wide(W& ws, int64_t m, int64_t k, int64_t G, WideArgs& a) {
    a.V = ws.template take<double>(m * k);
    a.tau = ws.template take<double>(k);
    a.beta = ws.template take<double>(k);
    a.amax = ws.template take<ArgMax>(2 * G);
    a.apub = ws.template take<double>(2 * G * m);
    a.bar = ws.template take<unsigned>(4);
}

size_t tall_smem_bytes(int64_t m, int64_t k, int64_t G, int64_t seg) {
    const int64_t mpad = ceil_div(m, seg) * seg;
    const int64_t rmax = ceil_div(m, G);
    return (size_t)(mpad + kMaxOwn * (mpad / seg) + 3 * k + 3 * kMaxOwn + kMaxOwn * k + rmax * k) *
               sizeof(double) +
           (size_t)kMaxOwn * sizeof(int64_t);
}

template <class W>
void carve_tall(W& ws, int64_t m, int64_t n, int64_t k, int64_t G, TallArgs& a) {
    a.F = ws.template take<double>(n * k);
    a.Rcol = ws.template take<double>(n * k);
    a.V = ws.template take<double>(m * k);
    a.tau = ws.template take<double>(k);
    a.beta = ws.template take<double>(k);
    a.a = ws.template take<double>(m + 2);  // a[m] stays zero (bulk copies round up)
    a.normpart = ws.template take<double>(G);
    a.zpart = ws.template take<double>(G * k);
    a.red = ws.template take<double>(k + 1);
    a.piv = ws.template take<int64_t>(4);
    a.flag_list = ws.template take<int64_t>(n);
    a.amax = ws.template take<ArgMax>(G);
    a.bar = ws.template take<unsigned>(4);
}

int64_t* g_cpqr_tlog = nullptr;  // debug: per-phase timing of the cooperative kernel

}  // namespace

// Debug hook: accumulate per-phase ns of cpqr_kernel into `buf` (device
// int64[16], [15] = flagged-column count); NULL disables.
extern "C" void ids_debug_cpqr_timing(int64_t* buf) { g_cpqr_tlog = buf; }

extern "C" size_t ids_cpqr_workspace_bytes(int64_t rows, int64_t cols, int64_t k) {
    CountCarve c;
    CpqrArgs a{};
    carve_cpqr(c, rows, cols, k, kMaxG, a);
    CountCarve c2;
    TallArgs t{};
    carve_tall(c2, rows, cols, k, kMaxG, t);
    CountCarve c3;
    WideArgs w{};
    carve_wide(c3, rows, k, kMaxG, w);
    return tmax(tmax(c.off, c2.off), c3.off) + 256;
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
    if (rows <= 1024 && !getenv("IDS_CPQR_NO_WIDE")) {
        // short sketch too large for one cluster (C3's 200 x 10000): column
        // slices resident in shared memory on every SM, one grid barrier per
        // step (C3: 219 us vs 349 on the segment-unit kernel; the cluster
        // kernel above stays faster where it fits: C2 167 vs 172 us)
        int dev = 0, sms = 148, optin = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        const int64_t G = tmin<int64_t>(tmin<int64_t>(sms, kMaxG), cols);
        const int64_t ncm = ceil_div(cols, G);
        const size_t smem = wide_smem_bytes(rows, k, ncm);
        if (cols >= kWideMinCols && smem <= (size_t)optin - 1024) {
            WideArgs w{};
            w.Y = Y;
            w.m = rows;
            w.n = cols;
            w.ldy = ldy;
            w.k = k;
            w.colnorm2 = colnorm2;
            w.rank_tol = rank_tol;
            w.perm = perm;
            w.Rtop = Rtop;
            w.numerical_rank = numerical_rank;
            w.nc_max = ncm;
            w.tlog = g_cpqr_tlog;
            WsCarve ws(workspace, ws_bytes);
            carve_wide(ws, rows, k, kMaxG, w);
            if (!ws.ok()) {
                ids_set_last_error("cpqr: workspace too small");
                return IDS_EWORKSPACE;
            }
            IDS_CUDA_TRY(cudaMemsetAsync(w.bar, 0, 4 * sizeof(unsigned), st));
            IDS_CUDA_TRY(cudaFuncSetAttribute(cpqr_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)smem));
            void* args[] = {&w};
            IDS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)cpqr_wide_kernel, dim3((unsigned)G),
                                                     dim3(kThreads), args, smem, st));
            ids_count_launch();
            if (Q) {
                form_q_kernel<<<(unsigned)k, kThreads, 0, st>>>(w.V, w.tau, rows, k, Q);
                IDS_LAUNCH_CHECK();
            }
            return IDS_OK;
        }
    }
    // (short wide sketches beyond the shared-memory kernels: the segment-unit
    // kernel measured faster than the 256-row column-owning variant at C3's
    // shape, 348 vs 401 us; that variant stays for them to opt into with
    // IDS_CPQR_WIDE=1)
    const bool tall = rows > 1024, wide = rows >= 128 && cols >= 4096 && getenv("IDS_CPQR_WIDE");
    if ((tall || wide) && k <= kTallMaxK && !getenv("IDS_CPQR_SEGMENT_UNITS")) {
        // column-owning CTAs, v in shared memory (GEMV units of 2048 rows for
        // tall sketches, 256 for short wide ones)
        const int64_t seg = tall ? 2048 : 256;
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        int G = (int)tmin<int64_t>(tmin<int64_t>(sms, kMaxG), cols);
        if (const char* e = getenv("IDS_CPQR_G")) G = tmin(G, atoi(e));  // experiments
        const size_t smem = tall_smem_bytes(rows, k, G, seg);
        if (ceil_div(cols, (int64_t)G) <= kMaxOwn && ceil_div(rows, (int64_t)G) <= kTThreads &&
            ceil_div(rows, seg) <= kMaxSegT && smem <= 200 * 1024) {
            TallArgs t{};
            t.Y = Y;
            t.m = rows;
            t.n = cols;
            t.ldy = ldy;
            t.k = k;
            t.colnorm2 = colnorm2;
            t.rank_tol = rank_tol;
            t.perm = perm;
            t.Rtop = Rtop;
            t.numerical_rank = numerical_rank;
            t.tlog = g_cpqr_tlog;
            // the leading 2 x 2048 rows of every column stay in L2 across the k
            // passes (64 MB at C5; larger pins measured slower) -- unless every
            // CTA's units fit in TMEM (one per warp): then none is pinned and
            // all of them stay resident (C4, 4096 x 1000: 152 -> 127 us)
            const bool all_resident =
                seg == 2048 && ceil_div(cols, (int64_t)G) * ceil_div(rows, seg) <= kTThreads / 32;
            t.pin_segs = all_resident ? 0 : 2;
            t.tmem = 1;
            if (const char* e = getenv("IDS_CPQR_PIN")) t.pin_segs = atoi(e);  // experiments
            if (const char* e = getenv("IDS_CPQR_TMEM")) t.tmem = atoi(e);
            t.pin_frac = 0.75f;  // C5: 872 vs 895 us at 0 (3 of 4 lines of the third segment, ~88 MB)
            if (const char* e = getenv("IDS_CPQR_PIN_FRAC")) t.pin_frac = (float)atof(e);
            WsCarve ws(workspace, ws_bytes);
            carve_tall(ws, rows, cols, k, kMaxG, t);
            if (!ws.ok()) {
                ids_set_last_error("cpqr: workspace too small");
                return IDS_EWORKSPACE;
            }
            IDS_CUDA_TRY(cudaMemsetAsync(t.bar, 0, 4 * sizeof(unsigned), st));
            IDS_CUDA_TRY(cudaMemsetAsync(t.a + rows, 0, 2 * sizeof(double), st));
            auto kern = seg == 2048 ? cpqr_tall_kernel<2048> : cpqr_tall_kernel<256>;
            IDS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            void* args[] = {&t};
            IDS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)kern, dim3(G), dim3(kTThreads), args, smem,
                                                     st));
            ids_count_launch();
            if (Q) {
                form_q_kernel<<<(unsigned)k, kThreads, 0, st>>>(t.V, t.tau, rows, k, Q);
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
