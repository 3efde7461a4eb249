// Operator applications for the error metric: y = A x and
// y = A^T x on device-resident A, dense in either layout or CSR -- the passes
// est_spectral_norm makes through id_residual_operator / matrix_operator
// (reference pkg/src/idsketch/estimators.py:91-121, bench.py:137-145).
//
// Every pass streams A once from HBM, so each kernel is built for memory-level
// parallelism: 16 independent loads in flight per lane, branch-free (clamped
// addresses, zero weights past the end).  Sums are in a fixed order (per-lane
// strips, shuffle tree, segment partials reduced in index order), so results
// are deterministic run to run.
#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kLoads = 16;          // independent loads per lane per batch
constexpr int64_t kSegLen = 8192;   // elements of a dot unit (output, segment)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// "dot" form: unit (o, s) -> sum over t in segment s of M[o * ld + t] * x[t];
// written to out[o] (one segment) or part[s * nout + o].
__global__ void __launch_bounds__(kThreads) gemv_dot_kernel(const double* __restrict__ M,
                                                            int64_t nout, int64_t nin, int64_t ld,
                                                            const double* __restrict__ x,
                                                            int64_t nseg, double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * kThreads) >> 5;
    const int64_t units = nout * nseg;
    for (int64_t u = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5; u < units; u += nw) {
        const int64_t o = u / nseg, sg = u - o * nseg;
        const double* row = M + o * ld;
        const int64_t t1 = tmin(nin, (sg + 1) * kSegLen);
        double acc0 = 0.0, acc1 = 0.0;
        for (int64_t t = sg * kSegLen + lane; t < t1; t += 32 * kLoads) {
            double a[kLoads], b[kLoads];
#pragma unroll
            for (int i = 0; i < kLoads; ++i) {
                const int64_t ti = t + 32 * i;
                const int64_t tc = ti < t1 ? ti : t1 - 1;
                a[i] = row[tc];
                b[i] = ti < t1 ? x[tc] : 0.0;
            }
#pragma unroll
            for (int i = 0; i < kLoads; i += 2) {
                acc0 = fma(a[i], b[i], acc0);
                acc1 = fma(a[i + 1], b[i + 1], acc1);
            }
        }
        const double s = warp_sum(acc0 + acc1);
        if (lane == 0) out[sg * nout + o] = s;
    }
}

// "axpy" form: thread o of tile tb -> sum over t in the tile of M[t * ld + o] * x[t]
// (coalesced across o); written to out[o] (one tile) or part[tb * nout + o].
__global__ void __launch_bounds__(kThreads) gemv_axpy_kernel(const double* __restrict__ M,
                                                             int64_t nout, int64_t nin, int64_t ld,
                                                             const double* __restrict__ x,
                                                             int64_t tile, double* __restrict__ out) {
    const int64_t o = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (o >= nout) return;
    const int64_t tb = blockIdx.y;
    const int64_t t0 = tb * tile, t1 = tmin(nin, t0 + tile);
    double acc[kLoads];
#pragma unroll
    for (int i = 0; i < kLoads; ++i) acc[i] = 0.0;
    for (int64_t t = t0; t < t1; t += kLoads) {
        double a[kLoads];
#pragma unroll
        for (int i = 0; i < kLoads; ++i) a[i] = M[tmin(t + i, t1 - 1) * ld + o];
#pragma unroll
        for (int i = 0; i < kLoads; ++i) acc[i] = fma(a[i], t + i < t1 ? x[t + i] : 0.0, acc[i]);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kLoads; ++i) s += acc[i];
    out[tb * nout + o] = s;
}

// out[o] = sum_{p < np} part[p * n + o], in order
__global__ void partials_reduce_kernel(const double* __restrict__ part, int64_t np, int64_t n,
                                       double* __restrict__ out) {
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n;
         o += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int64_t p = 0; p < np; ++p) s += part[p * n + o];
        out[o] = s;
    }
}

// CSR y = A x: GL lanes per row (GL | 32), strided over the row's nonzeros,
// then a shuffle tree inside the lane group.
template <class IP, int GL>
__global__ void __launch_bounds__(kThreads) csr_spmv_kernel(const IP* __restrict__ indptr,
                                                            const int32_t* __restrict__ indices,
                                                            const double* __restrict__ data,
                                                            int64_t rows, const double* __restrict__ x,
                                                            double* __restrict__ y) {
    constexpr int kRowsPerWarp = 32 / GL;
    const int lane = threadIdx.x & 31, li = lane % GL;
    const int64_t w = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * kThreads) >> 5;
    for (int64_t rb = w * kRowsPerWarp; rb < rows; rb += nw * kRowsPerWarp) {
        const int64_t r = rb + lane / GL;
        double s = 0.0;
        if (r < rows) {
            const int64_t p0 = (int64_t)indptr[r], p1 = (int64_t)indptr[r + 1];
            double s1 = 0.0;
            int64_t p = p0 + li;
            for (; p + GL < p1; p += 2 * GL) {
                s = fma(data[p], x[indices[p]], s);
                s1 = fma(data[p + GL], x[indices[p + GL]], s1);
            }
            if (p < p1) s = fma(data[p], x[indices[p]], s);
            s += s1;
        }
#pragma unroll
        for (int o = GL / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (r < rows && li == 0) y[r] = s;
    }
}

int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// Work split of one dense pass: dot form with `nseg` segments, or axpy form
// with `ntile` tiles of `tile` elements; `parts` partial doubles when > 1.
struct GemvPlan {
    bool dot;
    int64_t nout, nin, nseg, ntile, tile, parts;
};

GemvPlan plan_gemv(int64_t rows, int64_t cols, int layout, int trans) {
    GemvPlan p{};
    // row-major A x and col-major A^T x are dots along contiguous vectors
    p.dot = (layout == IDS_ROW_MAJOR) == (trans == 0);
    p.nout = trans ? cols : rows;
    p.nin = trans ? rows : cols;
    const int64_t threads_wanted = (int64_t)148 * 2048 * 2;
    if (p.dot) {
        p.nseg = ceil_div(p.nin, kSegLen);
        p.parts = p.nseg > 1 ? p.nseg * p.nout : 0;
    } else {
        p.ntile = tmax<int64_t>(1, tmin<int64_t>(ceil_div(threads_wanted, p.nout),
                                                 ceil_div(p.nin, 256)));
        p.tile = ceil_div(p.nin, p.ntile);
        p.ntile = ceil_div(p.nin, p.tile);
        p.parts = p.ntile > 1 ? p.ntile * p.nout : 0;
    }
    return p;
}

template <class IP>
int launch_spmv(const IP* indptr, const int32_t* indices, const double* data, int64_t rows,
                int64_t nnz, const double* x, double* y, cudaStream_t st) {
    const double avg = rows > 0 ? (double)nnz / (double)rows : 0.0;
    const int64_t blocks_cap = (int64_t)sm_count() * 8;
    auto grid = [&](int gl) {
        return (unsigned)tmax<int64_t>(1, tmin(ceil_div(rows * gl, kThreads), blocks_cap));
    };
    if (avg <= 2.0) csr_spmv_kernel<IP, 1><<<grid(1), kThreads, 0, st>>>(indptr, indices, data, rows, x, y);
    else if (avg <= 6.0) csr_spmv_kernel<IP, 4><<<grid(4), kThreads, 0, st>>>(indptr, indices, data, rows, x, y);
    else if (avg <= 24.0) csr_spmv_kernel<IP, 8><<<grid(8), kThreads, 0, st>>>(indptr, indices, data, rows, x, y);
    else csr_spmv_kernel<IP, 32><<<grid(32), kThreads, 0, st>>>(indptr, indices, data, rows, x, y);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}

}  // namespace

extern "C" size_t ids_dense_gemv_workspace_bytes(int64_t rows, int64_t cols, int layout, int trans) {
    if (rows < 1 || cols < 1) return 256;
    const GemvPlan p = plan_gemv(rows, cols, layout, trans);
    return (size_t)p.parts * sizeof(double) + 256;
}

extern "C" int ids_dense_gemv_f64(const double* A, int64_t rows, int64_t cols, int64_t ld,
                                  int layout, int trans, const double* x, double* y,
                                  void* workspace, size_t ws_bytes, void* stream) {
    if (rows < 0 || cols < 0 || (layout != IDS_ROW_MAJOR && layout != IDS_COL_MAJOR) ||
        (layout == IDS_ROW_MAJOR ? ld < cols : ld < rows) || ld < 1) {
        ids_set_last_error("dense gemv: bad arguments");
        return IDS_EINVAL;
    }
    cudaStream_t st = as_stream(stream);
    const int64_t nout = trans ? cols : rows;
    if (nout == 0) return IDS_OK;
    if ((trans ? rows : cols) == 0) {
        IDS_CUDA_TRY(cudaMemsetAsync(y, 0, sizeof(double) * nout, st));
        return IDS_OK;
    }
    const GemvPlan p = plan_gemv(rows, cols, layout, trans);
    double* part = nullptr;
    if (p.parts) {
        WsCarve ws(workspace, ws_bytes);
        part = ws.take<double>(p.parts);
        if (!ws.ok()) {
            ids_set_last_error("dense gemv: workspace too small");
            return IDS_EWORKSPACE;
        }
    }
    double* out = p.parts ? part : y;
    const int64_t blocks_cap = (int64_t)sm_count() * 8;
    if (p.dot) {
        const unsigned g = (unsigned)tmax<int64_t>(1, tmin(ceil_div(p.nout * p.nseg * 32, kThreads),
                                                           blocks_cap));
        gemv_dot_kernel<<<g, kThreads, 0, st>>>(A, p.nout, p.nin, ld, x, p.nseg, out);
    } else {
        const dim3 g((unsigned)ceil_div(p.nout, kThreads), (unsigned)p.ntile);
        gemv_axpy_kernel<<<g, kThreads, 0, st>>>(A, p.nout, p.nin, ld, x, p.tile, out);
    }
    IDS_LAUNCH_CHECK();
    if (p.parts) {
        const int64_t np = p.dot ? p.nseg : p.ntile;
        partials_reduce_kernel<<<(unsigned)tmin<int64_t>(ceil_div(p.nout, kThreads), blocks_cap),
                                 kThreads, 0, st>>>(part, np, p.nout, y);
        IDS_LAUNCH_CHECK();
    }
    return IDS_OK;
}

extern "C" int ids_csr_spmv_f64(const void* indptr, int indptr64, const int32_t* indices,
                                const double* data, int64_t rows, int64_t cols, int64_t nnz,
                                const double* x, double* y, void* stream) {
    if (rows < 0 || cols < 0 || nnz < 0) {
        ids_set_last_error("csr spmv: bad arguments");
        return IDS_EINVAL;
    }
    if (rows == 0) return IDS_OK;
    cudaStream_t st = as_stream(stream);
    if (indptr64)
        return launch_spmv(static_cast<const int64_t*>(indptr), indices, data, rows, nnz, x, y, st);
    return launch_spmv(static_cast<const int32_t*>(indptr), indices, data, rows, nnz, x, y, st);
}
