// Dense CountSketch Y = S @ A on B200 (replaces reference sketch.py:119 for
// dense A: scipy csr_matvecs over the CSR operator built at sketch.py:108-114).
//
// Row-major A (the numpy default):  bucket-gather kernel.  One warp owns one
// (bucket l, 64-column chunk) unit and walks the rows of bucket l in
// increasing row order (the bucket index), streaming each row segment with
// 16-byte loads and accumulating in registers.  A is read exactly once, with
// no atomics and no shared memory; the per-entry summation order is scipy's,
// so Y is bit-identical to the reference when each bucket is one segment.
//
// Col-major A (Fortran order, what the reference's as_dense produces):
// column-stream kernel.  One warp owns NC columns and a row segment; lanes
// read 32 consecutive rows (coalesced) and scatter into a per-warp L x NC
// shared-memory accumulator.  Lanes that hit the same bucket are ordered by
// row with __match_any_sync ranks, so the sum order is again increasing row.
//
// Both paths are HBM-streaming kernels (algorithmic traffic = bytes of A);
// tensor cores have nothing to do here.
#include "common.cuh"

namespace {

constexpr int kWarpsPerBlock = 8;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ int64_t lower_bound_rows(const int32_t* __restrict__ order,
                                                    int64_t lo, int64_t hi, int64_t row) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)dec_row(order[mid]) < row) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <int VEC>
struct VecT;
template <>
struct VecT<1> {
    typedef double T;
    static __device__ __forceinline__ void load(const double* p, double* v) { v[0] = __ldcs(p); }
};
template <>
struct VecT<2> {
    typedef double2 T;
    static __device__ __forceinline__ void load(const double* p, double* v) {
        const double2 x = __ldcs(reinterpret_cast<const double2*>(p));
        v[0] = x.x;
        v[1] = x.y;
    }
};

// unit = ((l * nseg + seg) * nchunks + chunk); one warp per unit.
template <int VEC, int UNR>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    cs_rowmajor_kernel(const double* __restrict__ A, int64_t ld, int64_t cols, int64_t row0,
                       int64_t rows, int restrict_rows, const int32_t* __restrict__ order,
                       const int64_t* __restrict__ bstart, int64_t L, int nchunks, int nseg,
                       double* __restrict__ out, int64_t seg_stride, int init_from_out) {
    const int64_t gw = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (gw >= L * nchunks * nseg) return;
    const int chunk = (int)(gw % nchunks);
    const int64_t t = gw / nchunks;
    const int seg = (int)(t % nseg);
    const int64_t l = t / nseg;

    int64_t k0 = bstart[l], k1 = bstart[l + 1];
    if (restrict_rows) {
        const int64_t a = lower_bound_rows(order, k0, k1, row0);
        k1 = lower_bound_rows(order, a, k1, row0 + rows);
        k0 = a;
    }
    const int64_t len = k1 - k0;
    const int64_t s0 = k0 + len * seg / nseg, s1 = k0 + len * (seg + 1) / nseg;

    const int64_t c = (int64_t)chunk * 32 * VEC + (int64_t)lane * VEC;
    const bool valid = c < cols;
    double acc[VEC];
    double* o = out + (int64_t)seg * seg_stride;
#pragma unroll
    for (int v = 0; v < VEC; ++v)
        acc[v] = (init_from_out && valid && c + v < cols) ? o[(c + v) * L + l] : 0.0;

    // lanes past the last column read a valid column (results discarded) so
    // that the hot loop is branch-free and all loads of a batch are in flight
    const int64_t cl = valid ? c : (cols - VEC);
    const double* Abase = A + cl - row0 * ld;
    int64_t kb = s0;
    for (; kb + 32 <= s1; kb += 32) {  // full batches: 32 rows, two rounds of 16 loads
        const int32_t e = __ldg(order + kb + lane);
#pragma unroll
        for (int h = 0; h < 32; h += UNR) {
            double x[UNR][VEC];
            int32_t ev[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                ev[u] = __shfl_sync(kFull, e, h + u);
                VecT<VEC>::load(Abase + (int64_t)dec_row(ev[u]) * ld, x[u]);
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
#pragma unroll
                for (int v = 0; v < VEC; ++v)
                    acc[v] = ev[u] >= 0 ? acc[v] + x[u][v] : acc[v] - x[u][v];
            }
        }
    }
    if (kb < s1) {  // tail batch (< 32 rows), in order
        const int n = (int)(s1 - kb);
        const int32_t e = lane < n ? __ldg(order + kb + lane) : 0;
        for (int u = 0; u < n; ++u) {
            const int32_t ev = __shfl_sync(kFull, e, u);
            double x[VEC];
            VecT<VEC>::load(Abase + (int64_t)dec_row(ev) * ld, x);
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[v] = ev >= 0 ? acc[v] + x[v] : acc[v] - x[v];
        }
    }
    if (valid) {
#pragma unroll
        for (int v = 0; v < VEC; ++v)
            if (c + v < cols) o[(c + v) * L + l] = acc[v];
    }
}

// unit = seg * ngroups + group; one warp per unit; per-warp acc NC x L.
template <int NC, int UNR>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    cs_colmajor_kernel(const double* __restrict__ A, int64_t ld, int64_t rows, int64_t cols,
                       int64_t row0, const int32_t* __restrict__ bucket,
                       const int8_t* __restrict__ sign, int64_t L, int ngroups, int nseg,
                       int warps_per_block, double* __restrict__ out, int64_t seg_stride,
                       int init_from_out, double* __restrict__ gacc) {
    extern __shared__ double smem_acc[];
    const int wib = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (wib >= warps_per_block) return;
    const int64_t gw = (int64_t)blockIdx.x * warps_per_block + wib;
    if (gw >= (int64_t)ngroups * nseg) return;
    const int group = (int)(gw % ngroups);
    const int seg = (int)(gw / ngroups);
    double* acc = gacc ? gacc + gw * (int64_t)NC * L : smem_acc + (int64_t)wib * NC * L;
    const int64_t c0 = (int64_t)group * NC;
    const int nc = (int)tmin<int64_t>(NC, cols - c0);
    double* o = out + (int64_t)seg * seg_stride;
    for (int64_t q = lane; q < (int64_t)NC * L; q += 32) {
        const int64_t qc = q / L, ql = q % L;
        acc[q] = (init_from_out && qc < nc) ? o[(c0 + qc) * L + ql] : 0.0;
    }
    __syncwarp();
    const int64_t r0 = rows * seg / nseg, r1 = rows * (seg + 1) / nseg;
    const uint32_t lt = (1u << lane) - 1u;
    for (int64_t rb = r0; rb < r1; rb += 32 * UNR) {
        int32_t h[UNR];
        int8_t s[UNR];
        double x[UNR][NC];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int64_t i = rb + u * 32 + lane;
            const bool act = i < r1;
            h[u] = act ? __ldg(bucket + row0 + i) : -1;
            s[u] = act ? __ldg(sign + row0 + i) : (int8_t)1;
#pragma unroll
            for (int q = 0; q < NC; ++q)
                x[u][q] = (act && q < nc) ? __ldcs(A + (c0 + q) * ld + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint32_t peers = __match_any_sync(kFull, h[u]);
            const int rank = __popc(peers & lt);
            const int maxr = (int)__reduce_max_sync(kFull, (unsigned)(h[u] >= 0 ? rank : 0));
            for (int rr = 0; rr <= maxr; ++rr) {
                if (h[u] >= 0 && rank == rr) {
#pragma unroll
                    for (int q = 0; q < NC; ++q) {
                        double* p = acc + (int64_t)q * L + h[u];
                        *p = s[u] > 0 ? *p + x[u][q] : *p - x[u][q];
                    }
                }
                __syncwarp();
            }
        }
    }
    __syncwarp();
    for (int64_t q = lane; q < (int64_t)nc * L; q += 32) {
        const int64_t qc = q / L, ql = q % L;
        o[(c0 + qc) * L + ql] = acc[q];
    }
}

// Y[e] = (accumulate ? Y[e] : 0) + sum_s part[s][e], s in order.
__global__ void seg_reduce_kernel(const double* __restrict__ part, int nseg, int64_t n,
                                  int64_t seg_stride, double* __restrict__ Y, int accumulate) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        double acc = accumulate ? Y[e] : 0.0;
        for (int s = 0; s < nseg; ++s) acc += part[(int64_t)s * seg_stride + e];
        Y[e] = acc;
    }
}

__global__ void nonfinite_scan_kernel(const double* __restrict__ Y, int64_t n, int32_t* flag) {
    bool bad = false;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(Y[e]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
}

__global__ void dense_nonfinite_kernel(const double* __restrict__ A, int64_t outer,
                                       int64_t inner, int64_t ld, int32_t* flag) {
    bool bad = false;
    const int64_t n = outer * inner;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = e / inner, in = e % inner;
        bad |= !isfinite(A[o * ld + in]);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
}

struct DensePlan {
    int layout;
    int vec, nchunks;   // row-major
    int nc, ngroups;    // col-major
    int wpb;            // col-major warps per block
    bool global_acc;
    int nseg;
    int64_t units;
    size_t smem;
};

constexpr int64_t kTargetWarps = 148 * 16;
constexpr int64_t kMinWarps = 148 * 8;

DensePlan plan_dense(int64_t rows, int64_t cols, int64_t L, int layout, int flags,
                     bool aligned2, int64_t bucket_rows) {
    DensePlan p{};
    p.layout = layout;
    p.nseg = 1;
    if (layout == IDS_ROW_MAJOR) {
        p.vec = aligned2 ? 2 : 1;
        p.nchunks = (int)ceil_div(cols, 32 * p.vec);
        p.units = L * p.nchunks;
        if (!(flags & IDS_FLAG_ORDERED) && p.units < kMinWarps) {
            int64_t ns = ceil_div(kTargetWarps, p.units);
            const int64_t cap = tmax<int64_t>(1, bucket_rows / 256);
            p.nseg = (int)tmax<int64_t>(1, tmin<int64_t>(ns, cap));
        }
        p.units *= p.nseg;
    } else {
        p.nc = cols >= 2 * kTargetWarps ? 2 : 1;
        p.ngroups = (int)ceil_div(cols, p.nc);
        p.units = p.ngroups;
        if (!(flags & IDS_FLAG_ORDERED) && p.units < kMinWarps) {
            int64_t ns = ceil_div(kTargetWarps, p.units);
            const int64_t cap = tmax<int64_t>(1, rows / 1024);
            p.nseg = (int)tmax<int64_t>(1, tmin<int64_t>(ns, cap));
        }
        p.units *= p.nseg;
        const size_t per_warp = (size_t)p.nc * L * sizeof(double);
        const size_t budget = 160 * 1024;
        p.wpb = (int)tmin<size_t>(kWarpsPerBlock, budget / per_warp);
        if (p.wpb < 1) {
            p.wpb = kWarpsPerBlock;
            p.global_acc = true;
            p.smem = 0;
        } else {
            p.global_acc = false;
            p.smem = per_warp * p.wpb;
        }
    }
    return p;
}

}  // namespace

extern "C" size_t ids_countsketch_dense_workspace_bytes(int64_t rows, int64_t cols,
                                                        int64_t out_dim, int layout) {
    // worst case over the plans the kernel may choose
    const DensePlan p = plan_dense(rows, cols, out_dim, layout, 0, true, rows);
    const DensePlan p1 = plan_dense(rows, cols, out_dim, layout, 0, false, rows);
    const int nseg = max(p.nseg, p1.nseg);
    WsCount c;
    c.take<double>((size_t)nseg * out_dim * cols);
    if (layout == IDS_COL_MAJOR && p.global_acc) c.take<double>((size_t)p.units * p.nc * out_dim);
    return c.off + 256;
}

extern "C" int ids_countsketch_dense_f64(const double* A, int64_t rows, int64_t cols,
                                         int64_t ld, int layout, int64_t row0, int64_t in_dim,
                                         const int32_t* bucket, const int8_t* sign,
                                         const int32_t* order_signed, const int64_t* bstart,
                                         int64_t out_dim, double* Y, int accumulate, int flags,
                                         int32_t* nonfinite, void* workspace, size_t ws_bytes,
                                         void* stream) {
    if (rows < 1 || cols < 1 || out_dim < 1 || row0 < 0 || row0 + rows > in_dim ||
        (layout != IDS_ROW_MAJOR && layout != IDS_COL_MAJOR) ||
        ld < (layout == IDS_ROW_MAJOR ? cols : rows) || in_dim > 0x7fffffffLL) {
        ids_set_last_error("dense countsketch: bad arguments");
        return IDS_EINVAL;
    }
    cudaStream_t st = as_stream(stream);
    const bool aligned2 = ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && (ld % 2 == 0) &&
                          (cols % 2 == 0);
    const DensePlan p = plan_dense(rows, cols, out_dim, layout, flags, aligned2,
                                   tmax<int64_t>(1, rows / out_dim));
    WsCarve ws(workspace, ws_bytes);
    double* part = p.nseg > 1 ? ws.take<double>((size_t)p.nseg * out_dim * cols) : nullptr;
    double* gacc = (layout == IDS_COL_MAJOR && p.global_acc)
                       ? ws.take<double>((size_t)p.units * p.nc * out_dim)
                       : nullptr;
    if (!ws.ok()) {
        ids_set_last_error("dense countsketch: workspace too small");
        return IDS_EWORKSPACE;
    }
    double* out = p.nseg > 1 ? part : Y;
    const int64_t seg_stride = out_dim * cols;
    const int init_from_out = (p.nseg == 1 && accumulate) ? 1 : 0;
    if (layout == IDS_ROW_MAJOR) {
        const int restrict_rows = (row0 != 0 || rows != in_dim) ? 1 : 0;
        const unsigned grid = (unsigned)ceil_div(p.units, kWarpsPerBlock);
        if (p.vec == 2)
            cs_rowmajor_kernel<2, 8><<<grid, kWarpsPerBlock * 32, 0, st>>>(
                A, ld, cols, row0, rows, restrict_rows, order_signed, bstart, out_dim,
                p.nchunks, p.nseg, out, seg_stride, init_from_out);
        else
            cs_rowmajor_kernel<1, 8><<<grid, kWarpsPerBlock * 32, 0, st>>>(
                A, ld, cols, row0, rows, restrict_rows, order_signed, bstart, out_dim,
                p.nchunks, p.nseg, out, seg_stride, init_from_out);
        IDS_LAUNCH_CHECK();
    } else {
        const unsigned grid = (unsigned)ceil_div(p.units, p.wpb);
        if (p.smem > 40 * 1024) {
            if (p.nc == 2)
                IDS_CUDA_TRY(cudaFuncSetAttribute(cs_colmajor_kernel<2, 4>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)p.smem));
            else
                IDS_CUDA_TRY(cudaFuncSetAttribute(cs_colmajor_kernel<1, 4>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)p.smem));
        }
        if (p.nc == 2)
            cs_colmajor_kernel<2, 4><<<grid, p.wpb * 32, p.smem, st>>>(
                A, ld, rows, cols, row0, bucket, sign, out_dim, p.ngroups, p.nseg, p.wpb, out,
                seg_stride, init_from_out, gacc);
        else
            cs_colmajor_kernel<1, 4><<<grid, p.wpb * 32, p.smem, st>>>(
                A, ld, rows, cols, row0, bucket, sign, out_dim, p.ngroups, p.nseg, p.wpb, out,
                seg_stride, init_from_out, gacc);
        IDS_LAUNCH_CHECK();
    }
    if (p.nseg > 1) {
        const unsigned g = (unsigned)tmin<int64_t>(ceil_div(seg_stride, 256), 148 * 8);
        seg_reduce_kernel<<<g, 256, 0, st>>>(part, p.nseg, seg_stride, seg_stride, Y, accumulate);
        IDS_LAUNCH_CHECK();
    }
    if (nonfinite) {
        const unsigned g = (unsigned)tmin<int64_t>(ceil_div(seg_stride, 256), 148 * 4);
        nonfinite_scan_kernel<<<g, 256, 0, st>>>(Y, seg_stride, nonfinite);
        IDS_LAUNCH_CHECK();
    }
    return IDS_OK;
}

extern "C" int ids_dense_has_nonfinite(const double* A, int64_t rows, int64_t cols, int64_t ld,
                                       int layout, int32_t* flag, void* stream) {
    if (rows < 0 || cols < 0) return IDS_EINVAL;
    if (rows == 0 || cols == 0) return IDS_OK;
    const int64_t outer = layout == IDS_ROW_MAJOR ? rows : cols;
    const int64_t inner = layout == IDS_ROW_MAJOR ? cols : rows;
    const unsigned g = (unsigned)tmin<int64_t>(ceil_div(outer * inner, 256), 148 * 16);
    dense_nonfinite_kernel<<<g, 256, 0, as_stream(stream)>>>(A, outer, inner, ld, flag);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}
