// Column-distributed truncated CPQR: the k-step pivoted
// Householder QR of linalg.py:76-103 (dgeqp3's pivot rule, as in cpqr.cu)
// with the COLUMNS of the sketch split across ranks -- the tensor path's term
// blocks, so the L x R/G sketch blocks never have to be gathered.
//
// Each rank keeps its columns' partial norms, positions, update factors F and
// R rows; the Householder vectors V (L x k) are replicated.  One step, driven
// by the host (paper_1901_10559_b200/distributed.py) around two tiny
// collectives:
//   host:   all-gather the per-rank pivot candidates, pick the global pivot
//           (largest partial norm, ties to the lowest position -- fixed order);
//   owner:  ids_dcpqr_pivot_f64 -- position swap, residual pivot column
//           a = Y[:, c*] - V F[:, c*] (rows >= kk); the others only swap;
//   host:   broadcast a (L doubles) from the owner;
//   all:    ids_dcpqr_step_f64 -- Householder vector from a (identical on
//           every rank), z = V^T v, the GEMV Y_local^T v, F row, R row,
//           LAPACK norm downdate / recompute, next local candidate.
// Candidates travel as 4 doubles (value, position, column, column at the next
// position), exact for indices < 2^53.
#include <float.h>
#include <math.h>

#include "common.cuh"
#include "cpqr_common.cuh"

namespace {

constexpr int kT = 256;
constexpr int kW = kT / 32;
constexpr int kSeg = 512;          // GEMV unit: rows per (column, segment)
constexpr int kSegLoads = kSeg / 32;

// kSeg-padded row count (device code)
__device__ __forceinline__ int64_t ceil_div_dev(int64_t m) { return (m + kSeg - 1) / kSeg * kSeg; }

struct DState {  // carve of the workspace
    double *vn1, *vn2, *F, *R, *V, *tau, *beta, *z, *hh, *W;
    int64_t* pos;
    int64_t* flag_list;
    int* nflag;
};

template <class Carve>
DState carve(Carve& ws, int64_t m, int64_t n, int64_t k) {
    DState s;
    const int64_t mpad = ceil_div(m, (int64_t)kSeg) * kSeg;
    s.vn1 = ws.template take<double>(n);
    s.vn2 = ws.template take<double>(n);
    s.F = ws.template take<double>(k * n);
    s.R = ws.template take<double>(k * n);
    s.V = ws.template take<double>(mpad * k);
    s.tau = ws.template take<double>(k);
    s.beta = ws.template take<double>(k);
    s.z = ws.template take<double>(k);
    s.hh = ws.template take<double>(4);
    s.W = ws.template take<double>(n * (mpad / kSeg));
    s.pos = ws.template take<int64_t>(n);
    s.flag_list = ws.template take<int64_t>(n);
    s.nflag = ws.template take<int>(1);
    return s;
}

struct Count {
    size_t off = 0;
    template <class T>
    T* take(size_t cnt) {
        off = align_up(off, 256) + cnt * sizeof(T);
        return nullptr;
    }
};

__device__ double block_reduce(double v, double* red) {  // fixed order, all threads get it
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    return s;
}

// norms and positions of the local columns (warp per column)
__global__ void __launch_bounds__(kT) dc_init_kernel(const double* __restrict__ Y, int64_t m,
                                                     int64_t n, int64_t ldy, int64_t col0,
                                                     DState s) {
    const int lane = threadIdx.x & 31;
    for (int64_t j = ((int64_t)blockIdx.x * kT + threadIdx.x) >> 5; j < n;
         j += ((int64_t)gridDim.x * kT) >> 5) {
        const double nrm = sqrt(warp_sum(lane_dot(Y + j * ldy, Y + j * ldy, 0, m)));
        if (lane == 0) {
            s.vn1[j] = nrm;
            s.vn2[j] = nrm;
            s.pos[j] = col0 + j;
        }
    }
}

// local pivot candidate over columns with pos >= pmin (one CTA)
__global__ void __launch_bounds__(kT) dc_candidate_kernel(int64_t n, int64_t col0, int64_t pmin,
                                                          DState s, double* __restrict__ cand) {
    __shared__ ArgMax wb[kW];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    ArgMax best{-1.0, INT64_MAX, -1, -1};
    for (int64_t j = threadIdx.x; j < n; j += kT) {
        const int64_t pj = s.pos[j];
        if (pj == pmin) best.col_at_next = col0 + j;
        if (pj >= pmin && better(s.vn1[j], pj, best.val, best.pos)) {
            best.val = s.vn1[j];
            best.pos = pj;
            best.col = col0 + j;
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
    if (lane == 0) wb[w] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        ArgMax r = wb[0];
        for (int i = 1; i < kW; ++i) {
            const ArgMax o = wb[i];
            if (better(o.val, o.pos, r.val, r.pos)) {
                r.val = o.val;
                r.pos = o.pos;
                r.col = o.col;
            }
            if (o.col_at_next >= 0) r.col_at_next = o.col_at_next;
        }
        cand[0] = r.val;
        cand[1] = (double)(r.col < 0 ? -1 : r.pos);
        cand[2] = (double)r.col;
        cand[3] = (double)r.col_at_next;
    }
}

// Global pivot from the gathered per-shard candidates (shard order, 4
// doubles each: value, position, column, column at position kk): largest
// value, ties to the lowest position; all-NaN norms keep position kk.  The
// device twin of distributed.pick_pivot -- piv = (c*, p*, column at kk).
__global__ void dc_select_kernel(const double* __restrict__ cands, int64_t nshards, int64_t kk,
                                 int64_t* __restrict__ piv) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    bool have = false;
    double bv = 0.0;
    int64_t bp = 0, bc = -1, ck = -1;
    for (int64_t q = 0; q < nshards; ++q) {
        const double val = cands[4 * q], pos = cands[4 * q + 1];
        const double col = cands[4 * q + 2], nxt = cands[4 * q + 3];
        if (nxt >= 0.0) ck = (int64_t)nxt;
        if (col < 0.0) continue;
        if (!have || val > bv || (val == bv && (int64_t)pos < bp)) {
            have = true;
            bv = val;
            bp = (int64_t)pos;
            bc = (int64_t)col;
        }
    }
    piv[0] = have ? bc : ck;
    piv[1] = have ? bp : kk;
    piv[2] = ck;
}

// position swap (CTA 0) and, on the owner, the residual pivot column.  With
// piv (device) the pivot comes from dc_select_kernel and the non-owners fill
// a with -0.0, the identity of IEEE addition: an all-reduce(SUM) of a over
// the ranks then reproduces the owner's column bit for bit.
__global__ void __launch_bounds__(kT) dc_pivot_kernel(const double* __restrict__ Y, int64_t m,
                                                      int64_t n, int64_t ldy, int64_t k,
                                                      int64_t col0, int64_t kk, int64_t cs,
                                                      int64_t ps, int64_t ck,
                                                      const int64_t* __restrict__ piv, DState s,
                                                      double* __restrict__ a) {
    if (piv) {
        cs = piv[0];
        ps = piv[1];
        ck = piv[2];
    }
    const int64_t csl = cs - col0, ckl = ck - col0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (ckl >= 0 && ckl < n && ck != cs) s.pos[ckl] = ps;
        if (csl >= 0 && csl < n) s.pos[csl] = kk;
    }
    if (csl < 0 || csl >= n) {
        if (piv)
            for (int64_t r = (int64_t)blockIdx.x * kT + threadIdx.x; r < m;
                 r += (int64_t)gridDim.x * kT)
                a[r] = -0.0;
        return;
    }
    const int64_t mpad = ceil_div_dev(m);
    const double* ycol = Y + csl * ldy;
    for (int64_t r = (int64_t)blockIdx.x * kT + threadIdx.x; r < m; r += (int64_t)gridDim.x * kT)
        a[r] = r < kk ? 0.0 : sub_dot(ycol[r], s.V + r, mpad, s.F + csl, n, kk);
}

// Householder vector v = V[:, kk] from the broadcast pivot column (one CTA,
// identical arithmetic on every rank); the owner records R[kk, c*] = beta
__global__ void __launch_bounds__(1024) dc_householder_kernel(int64_t m, int64_t n, int64_t col0,
                                                              int64_t kk, int64_t cs,
                                                              const int64_t* __restrict__ piv,
                                                              DState s,
                                                              const double* __restrict__ a) {
    __shared__ double red[32];
    if (piv) cs = piv[0];
    const int64_t mpad = ceil_div_dev(m);
    double ss = 0.0;
    for (int64_t r = kk + 1 + threadIdx.x; r < m; r += blockDim.x) ss = fma(a[r], a[r], ss);
    ss = block_reduce(ss, red);
    const double alpha = a[kk], xnorm = sqrt(ss);
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
    double* v = s.V + kk * mpad;
    for (int64_t r = threadIdx.x; r < mpad; r += blockDim.x)
        v[r] = (r < kk || r >= m) ? 0.0 : (r == kk ? 1.0 : a[r] * scal);
    if (threadIdx.x == 0) {
        s.tau[kk] = tau;
        s.beta[kk] = beta;
        s.hh[0] = tau;
        *s.nflag = 0;
        const int64_t csl = cs - col0;
        if (csl >= 0 && csl < n) s.R[kk * n + csl] = beta;
    }
}

// z_q = V[:, q]^T v (CTA q)
__global__ void __launch_bounds__(kT) dc_z_kernel(int64_t m, int64_t kk, DState s) {
    __shared__ double red[kW];
    const int64_t mpad = ceil_div_dev(m);
    const int64_t q = blockIdx.x;
    const double* vq = s.V + q * mpad;
    const double* v = s.V + kk * mpad;
    double acc = 0.0;
    for (int64_t r = kk + threadIdx.x; r < m; r += kT) acc = fma(vq[r], v[r], acc);
    acc = block_reduce(acc, red);
    if (threadIdx.x == 0) s.z[q] = acc;
}

// GEMV units (column j, kSeg-row segment): W[sg * n + j] = Y[seg, j]^T v
__global__ void __launch_bounds__(kT) dc_gemv_kernel(const double* __restrict__ Y, int64_t m,
                                                     int64_t n, int64_t ldy, int64_t kk, DState s) {
    const int lane = threadIdx.x & 31;
    const int64_t mpad = ceil_div_dev(m);
    const int64_t nseg = mpad / kSeg, s0 = kk / kSeg, ns = nseg - s0;
    const double* v = s.V + kk * mpad;
    const int64_t units = n * ns;
    for (int64_t u = ((int64_t)blockIdx.x * kT + threadIdx.x) >> 5; u < units;
         u += ((int64_t)gridDim.x * kT) >> 5) {
        const int64_t j = u / ns, sg = s0 + u % ns;
        if (s.pos[j] <= kk) continue;
        const double* y = Y + j * ldy;
        const int64_t b0 = sg * kSeg + lane;
        double yv[kSegLoads];
#pragma unroll
        for (int t = 0; t < kSegLoads; ++t) yv[t] = y[tmin(b0 + 32 * t, m - 1)];
        double s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int t = 0; t < kSegLoads; t += 2) {  // v is zero above kk and past m
            s1 = fma(yv[t], v[b0 + 32 * t], s1);
            s2 = fma(yv[t + 1], v[b0 + 32 * t + 32], s2);
        }
        const double w = warp_sum(s1 + s2);
        if (lane == 0) s.W[sg * n + j] = w;
    }
}

// F row, R row, norm downdate; flagged columns listed for the recompute
__global__ void __launch_bounds__(kT) dc_update_kernel(const double* __restrict__ Y, int64_t m,
                                                       int64_t n, int64_t ldy, int64_t kk,
                                                       DState s) {
    const double tol3z = sqrt(DBL_EPSILON);
    const int64_t mpad = ceil_div_dev(m);
    const int64_t nseg = mpad / kSeg;
    const double tau = s.tau[kk];
    for (int64_t j = (int64_t)blockIdx.x * kT + threadIdx.x; j < n; j += (int64_t)gridDim.x * kT) {
        if (s.pos[j] <= kk) continue;
        double wj = 0.0;
        for (int64_t sg = kk / kSeg; sg < nseg; ++sg) wj += s.W[sg * n + j];
        double f = sub_dot(wj, s.F + j, n, s.z, 1, kk);
        double rk = sub_dot(Y[j * ldy + kk], s.F + j, n, s.V + kk, mpad, kk);
        f *= tau;
        s.F[kk * n + j] = f;
        rk -= f;  // V[kk, kk] = 1
        s.R[kk * n + j] = rk;
        const double vn1 = s.vn1[j];
        if (kk < m - 1 && vn1 != 0.0) {
            double temp = fabs(rk) / vn1;
            temp = fmax(0.0, (1.0 + temp) * (1.0 - temp));
            const double ratio = vn1 / s.vn2[j];
            if (temp * ratio * ratio <= tol3z) s.flag_list[atomicAdd(s.nflag, 1)] = j;
            else s.vn1[j] = vn1 * sqrt(temp);
        }
    }
}

// exact partial norms of the flagged columns (warp per column)
__global__ void __launch_bounds__(kT) dc_recompute_kernel(const double* __restrict__ Y, int64_t m,
                                                          int64_t n, int64_t ldy, int64_t kk,
                                                          DState s) {
    const int lane = threadIdx.x & 31;
    const int64_t mpad = ceil_div_dev(m);
    const int nf = *s.nflag;
    for (int64_t fi = ((int64_t)blockIdx.x * kT + threadIdx.x) >> 5; fi < nf;
         fi += ((int64_t)gridDim.x * kT) >> 5) {
        const int64_t j = s.flag_list[fi];
        const double* y = Y + j * ldy;
        double acc = 0.0;
        for (int64_t r = kk + 1 + lane; r < m; r += 32) {
            const double v = sub_dot(y[r], s.V + r, mpad, s.F + j, n, kk + 1);
            acc = fma(v, v, acc);
        }
        acc = warp_sum(acc);
        if (lane == 0) {
            s.vn1[j] = sqrt(acc);
            s.vn2[j] = sqrt(acc);
        }
    }
}

// ---- fused device-driven steps (one launch each side of the pivot all-reduce) ----

// Pivot selection (dc_select_kernel's rule, redundantly per CTA) fused with
// the position swap and the residual pivot column (dc_pivot_kernel's with
// -0.0 from non-owners); CTA 0 publishes piv for the fused step.
__global__ void __launch_bounds__(kT) dc_select_pivot_kernel(
    const double* __restrict__ Y, int64_t m, int64_t n, int64_t ldy, int64_t col0, int64_t kk,
    const double* __restrict__ cands, int64_t nshards, int64_t* __restrict__ piv, DState s,
    double* __restrict__ a) {
    __shared__ int64_t sp[3];
    if (threadIdx.x == 0) {
        bool have = false;
        double bv = 0.0;
        int64_t bp = 0, bc = -1, ck = -1;
        for (int64_t q = 0; q < nshards; ++q) {
            const double val = cands[4 * q], pos = cands[4 * q + 1];
            const double col = cands[4 * q + 2], nxt = cands[4 * q + 3];
            if (nxt >= 0.0) ck = (int64_t)nxt;
            if (col < 0.0) continue;
            if (!have || val > bv || (val == bv && (int64_t)pos < bp)) {
                have = true;
                bv = val;
                bp = (int64_t)pos;
                bc = (int64_t)col;
            }
        }
        sp[0] = have ? bc : ck;
        sp[1] = have ? bp : kk;
        sp[2] = ck;
        if (blockIdx.x == 0) {
            piv[0] = sp[0];
            piv[1] = sp[1];
            piv[2] = sp[2];
        }
    }
    __syncthreads();
    const int64_t cs = sp[0], ps = sp[1], ck = sp[2];
    const int64_t csl = cs - col0, ckl = ck - col0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (ckl >= 0 && ckl < n && ck != cs) s.pos[ckl] = ps;
        if (csl >= 0 && csl < n) s.pos[csl] = kk;
    }
    const int64_t mpad = ceil_div_dev(m);
    const bool own = csl >= 0 && csl < n;
    const double* ycol = own ? Y + csl * ldy : nullptr;
    for (int64_t r = (int64_t)blockIdx.x * kT + threadIdx.x; r < m; r += (int64_t)gridDim.x * kT)
        a[r] = !own ? -0.0 : (r < kk ? 0.0 : sub_dot(ycol[r], s.V + r, mpad, s.F + csl, n, kk));
}

int sm_count() { return ids_sm_count(); }

bool bad_args(int64_t m, int64_t n, int64_t ldy, int64_t k) {
    return m < 1 || n < 0 || k < 1 || k > m || ldy < m;
}

}  // namespace

extern "C" size_t ids_dcpqr_workspace_bytes(int64_t rows, int64_t ncols, int64_t k) {
    Count c;
    carve(c, rows, ncols, k);
    return c.off + 256;
}

extern "C" int ids_dcpqr_init_f64(const double* Y, int64_t rows, int64_t ncols, int64_t ldy,
                                  int64_t k, int64_t col0, double* cand, void* workspace,
                                  size_t ws_bytes, void* stream) {
    if (bad_args(rows, ncols, ldy, k) || col0 < 0) {
        ids_set_last_error("dcpqr: bad arguments");
        return IDS_EINVAL;
    }
    WsCarve ws(workspace, ws_bytes);
    const DState s = carve(ws, rows, ncols, k);
    if (!ws.ok()) {
        ids_set_last_error("dcpqr: workspace too small");
        return IDS_EWORKSPACE;
    }
    cudaStream_t st = as_stream(stream);
    IDS_CUDA_TRY(cudaMemsetAsync(workspace, 0, ws.off, st));  // F, R, V start at zero
    if (ncols > 0) {
        const unsigned g = (unsigned)tmax<int64_t>(1, tmin<int64_t>(ceil_div(ncols, kW), sm_count() * 8));
        dc_init_kernel<<<g, kT, 0, st>>>(Y, rows, ncols, ldy, col0, s);
        IDS_LAUNCH_CHECK();
    }
    dc_candidate_kernel<<<1, kT, 0, st>>>(ncols, col0, 0, s, cand);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}

extern "C" int ids_dcpqr_pivot_f64(const double* Y, int64_t rows, int64_t ncols, int64_t ldy,
                                   int64_t k, int64_t col0, int64_t kk, int64_t cs, int64_t ps,
                                   int64_t ck, double* a, void* workspace, size_t ws_bytes,
                                   void* stream) {
    if (bad_args(rows, ncols, ldy, k) || kk < 0 || kk >= k) {
        ids_set_last_error("dcpqr: bad arguments");
        return IDS_EINVAL;
    }
    WsCarve ws(workspace, ws_bytes);
    const DState s = carve(ws, rows, ncols, k);
    if (!ws.ok()) {
        ids_set_last_error("dcpqr: workspace too small");
        return IDS_EWORKSPACE;
    }
    const unsigned g = (unsigned)tmax<int64_t>(1, tmin<int64_t>(ceil_div(rows, kT), sm_count()));
    dc_pivot_kernel<<<g, kT, 0, as_stream(stream)>>>(Y, rows, ncols, ldy, k, col0, kk, cs, ps, ck,
                                                     nullptr, s, a);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}

static int dcpqr_step(const double* Y, int64_t rows, int64_t ncols, int64_t ldy, int64_t k,
                      int64_t col0, int64_t kk, int64_t cs, const int64_t* piv, const double* a,
                      double* cand, void* workspace, size_t ws_bytes, void* stream) {
    if (bad_args(rows, ncols, ldy, k) || kk < 0 || kk >= k) {
        ids_set_last_error("dcpqr: bad arguments");
        return IDS_EINVAL;
    }
    WsCarve ws(workspace, ws_bytes);
    const DState s = carve(ws, rows, ncols, k);
    if (!ws.ok()) {
        ids_set_last_error("dcpqr: workspace too small");
        return IDS_EWORKSPACE;
    }
    cudaStream_t st = as_stream(stream);
    const int sms = sm_count();
    dc_householder_kernel<<<1, 1024, 0, st>>>(rows, ncols, col0, kk, cs, piv, s, a);
    IDS_LAUNCH_CHECK();
    if (kk > 0) {
        dc_z_kernel<<<(unsigned)kk, kT, 0, st>>>(rows, kk, s);
        IDS_LAUNCH_CHECK();
    }
    if (ncols > 0) {
        const int64_t units = ncols * (ceil_div(rows, (int64_t)kSeg) - kk / kSeg);
        const unsigned gg = (unsigned)tmax<int64_t>(1, tmin<int64_t>(ceil_div(units, kW), sms * 8));
        dc_gemv_kernel<<<gg, kT, 0, st>>>(Y, rows, ncols, ldy, kk, s);
        IDS_LAUNCH_CHECK();
        const unsigned gu = (unsigned)tmax<int64_t>(1, tmin<int64_t>(ceil_div(ncols, kT), sms));
        dc_update_kernel<<<gu, kT, 0, st>>>(Y, rows, ncols, ldy, kk, s);
        IDS_LAUNCH_CHECK();
        const unsigned gr = (unsigned)tmax<int64_t>(1, tmin<int64_t>(ceil_div(ncols, kW), sms * 2));
        dc_recompute_kernel<<<gr, kT, 0, st>>>(Y, rows, ncols, ldy, kk, s);
        IDS_LAUNCH_CHECK();
    }
    dc_candidate_kernel<<<1, kT, 0, st>>>(ncols, col0, kk + 1, s, cand);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}

extern "C" int ids_dcpqr_step_f64(const double* Y, int64_t rows, int64_t ncols, int64_t ldy,
                                  int64_t k, int64_t col0, int64_t kk, int64_t cs, const double* a,
                                  double* cand, void* workspace, size_t ws_bytes, void* stream) {
    return dcpqr_step(Y, rows, ncols, ldy, k, col0, kk, cs, nullptr, a, cand, workspace, ws_bytes,
                      stream);
}

extern "C" int ids_dcpqr_select_f64(const double* cands, int64_t nshards, int64_t kk, int64_t* piv,
                                    void* stream) {
    if (nshards < 1 || kk < 0) {
        ids_set_last_error("dcpqr: bad arguments");
        return IDS_EINVAL;
    }
    dc_select_kernel<<<1, 32, 0, as_stream(stream)>>>(cands, nshards, kk, piv);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}

extern "C" int ids_dcpqr_pivot_dev_f64(const double* Y, int64_t rows, int64_t ncols, int64_t ldy,
                                       int64_t k, int64_t col0, int64_t kk, const int64_t* piv,
                                       double* a, void* workspace, size_t ws_bytes, void* stream) {
    if (bad_args(rows, ncols, ldy, k) || kk < 0 || kk >= k || !piv) {
        ids_set_last_error("dcpqr: bad arguments");
        return IDS_EINVAL;
    }
    WsCarve ws(workspace, ws_bytes);
    const DState s = carve(ws, rows, ncols, k);
    if (!ws.ok()) {
        ids_set_last_error("dcpqr: workspace too small");
        return IDS_EWORKSPACE;
    }
    const unsigned g = (unsigned)tmax<int64_t>(1, tmin<int64_t>(ceil_div(rows, kT), sm_count()));
    dc_pivot_kernel<<<g, kT, 0, as_stream(stream)>>>(Y, rows, ncols, ldy, k, col0, kk, -1, kk, -1,
                                                     piv, s, a);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}

extern "C" int ids_dcpqr_step_dev_f64(const double* Y, int64_t rows, int64_t ncols, int64_t ldy,
                                      int64_t k, int64_t col0, int64_t kk, const int64_t* piv,
                                      const double* a, double* cand, void* workspace,
                                      size_t ws_bytes, void* stream) {
    if (!piv) {
        ids_set_last_error("dcpqr: bad arguments");
        return IDS_EINVAL;
    }
    return dcpqr_step(Y, rows, ncols, ldy, k, col0, kk, -1, piv, a, cand, workspace, ws_bytes,
                      stream);
}

extern "C" int ids_dcpqr_select_pivot_f64(const double* Y, int64_t rows, int64_t ncols,
                                          int64_t ldy, int64_t k, int64_t col0, int64_t kk,
                                          const double* cands, int64_t nshards, int64_t* piv,
                                          double* a, void* workspace, size_t ws_bytes,
                                          void* stream) {
    if (bad_args(rows, ncols, ldy, k) || kk < 0 || kk >= k || nshards < 1 || !piv) {
        ids_set_last_error("dcpqr: bad arguments");
        return IDS_EINVAL;
    }
    WsCarve ws(workspace, ws_bytes);
    const DState s = carve(ws, rows, ncols, k);
    if (!ws.ok()) {
        ids_set_last_error("dcpqr: workspace too small");
        return IDS_EWORKSPACE;
    }
    const unsigned g = (unsigned)tmax<int64_t>(1, tmin<int64_t>(ceil_div(rows, kT), sm_count()));
    dc_select_pivot_kernel<<<g, kT, 0, as_stream(stream)>>>(Y, rows, ncols, ldy, col0, kk, cands,
                                                            nshards, piv, s, a);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}

extern "C" int ids_dcpqr_results_f64(int64_t rows, int64_t ncols, int64_t k, int64_t* pos,
                                     double* R, double* beta, void* workspace, size_t ws_bytes,
                                     void* stream) {
    WsCarve ws(workspace, ws_bytes);
    const DState s = carve(ws, rows, ncols, k);
    if (!ws.ok() || rows < 1 || k < 1 || ncols < 0) {
        ids_set_last_error("dcpqr: bad arguments or workspace");
        return IDS_EINVAL;
    }
    cudaStream_t st = as_stream(stream);
    if (ncols > 0) {
        IDS_CUDA_TRY(cudaMemcpyAsync(pos, s.pos, sizeof(int64_t) * ncols, cudaMemcpyDeviceToDevice, st));
        IDS_CUDA_TRY(cudaMemcpyAsync(R, s.R, sizeof(double) * k * ncols, cudaMemcpyDeviceToDevice, st));
    }
    IDS_CUDA_TRY(cudaMemcpyAsync(beta, s.beta, sizeof(double) * k, cudaMemcpyDeviceToDevice, st));
    return IDS_OK;
}
