// Sparse CountSketch Y = S @ A (replaces reference sketch.py:119 on sparse A:
// as_csc canonicalization, linalg.py:39-53, then scipy csr_matmat).
//
// CSC kernel (the reference's canonical format): one warp per column walks
// the column's stored entries in storage (= increasing row) order, looks up
// each row's bucket and sign, and adds into a per-warp L-entry shared-memory
// accumulator.  Lanes of one 32-entry window that hit the same bucket are
// serialized in row order via __match_any_sync ranks, so every Y entry is
// summed exactly in scipy's order: Y is bit-identical to the reference for
// canonical input.
//
// CSR input is transposed to CSC on the device first (stable radix sort of
// column ids, so rows stay increasing within each column), then sketched by
// the CSC kernel.
#include <cub/cub.cuh>

#include "common.cuh"

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kWpb = 8;

template <class IP>
__global__ void __launch_bounds__(kWpb * 32)
    cs_csc_kernel(const IP* __restrict__ colptr, const int32_t* __restrict__ rowidx,
                  const double* __restrict__ data, int64_t cols, int64_t row0,
                  const int32_t* __restrict__ bucket, const int8_t* __restrict__ sign,
                  int64_t L, int wpb, double* __restrict__ Y, int accumulate,
                  double* __restrict__ gacc) {
    extern __shared__ double smem_acc[];
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (wib >= wpb) return;
    const int64_t c = (int64_t)blockIdx.x * wpb + wib;
    if (c >= cols) return;
    double* acc = gacc ? gacc + c * L : smem_acc + (int64_t)wib * L;
    double* y = Y + c * L;
    for (int64_t l = lane; l < L; l += 32) acc[l] = accumulate ? y[l] : 0.0;
    __syncwarp();
    const int64_t p0 = (int64_t)colptr[c], p1 = (int64_t)colptr[c + 1];
    const uint32_t lt = (1u << lane) - 1u;
    for (int64_t pb = p0; pb < p1; pb += 32) {
        const int64_t p = pb + lane;
        const bool act = p < p1;
        int32_t h = -1;
        double v = 0.0;
        if (act) {
            const int64_t i = row0 + __ldg(rowidx + p);
            h = __ldg(bucket + i);
            v = __ldcs(data + p);
            if (__ldg(sign + i) < 0) v = -v;
        }
        const uint32_t peers = __match_any_sync(kFull, h);
        const int rank = __popc(peers & lt);
        const int maxr = (int)__reduce_max_sync(kFull, (unsigned)(act ? rank : 0));
        for (int rr = 0; rr <= maxr; ++rr) {
            if (act && rank == rr) acc[h] = acc[h] + v;
            __syncwarp();
        }
    }
    for (int64_t l = lane; l < L; l += 32) y[l] = acc[l];
}

template <class IP>
__global__ void row_of_entry_kernel(const IP* __restrict__ indptr, int64_t rows,
                                    int32_t* __restrict__ row_of, int32_t* __restrict__ iota) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p0 = (int64_t)indptr[r], p1 = (int64_t)indptr[r + 1];
        for (int64_t p = p0; p < p1; ++p) {
            row_of[p] = (int32_t)r;
            iota[p] = (int32_t)p;
        }
    }
}

__global__ void gather_csc_kernel(const int32_t* __restrict__ perm,
                                  const int32_t* __restrict__ row_of,
                                  const double* __restrict__ data, int64_t nnz,
                                  int32_t* __restrict__ crow, double* __restrict__ cval) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = perm[q];
        crow[q] = row_of[p];
        cval[q] = data[p];
    }
}

__global__ void colptr_kernel(const int32_t* __restrict__ keys, int64_t nnz, int64_t cols,
                              int64_t* __restrict__ colptr) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c <= cols;
         c += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)keys[mid] < c) lo = mid + 1;
            else hi = mid;
        }
        colptr[c] = lo;
    }
}

__global__ void nonfinite_values_kernel(const double* __restrict__ v, int64_t n, int32_t* flag) {
    bool bad = false;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(v[e]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
}

int key_bits(int64_t n) {
    int b = 0;
    while ((1LL << b) < n) ++b;
    return b < 1 ? 1 : b;
}

size_t sort_bytes(int64_t nnz, int64_t cols) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const int32_t*)nullptr, (int32_t*)nullptr, (int)nnz, 0,
                                    key_bits(cols));
    return bytes;
}

struct CscLaunch {
    int wpb;
    size_t smem;
    bool global_acc;
};

CscLaunch csc_launch(int64_t L) {
    CscLaunch c;
    const size_t per = (size_t)L * sizeof(double);
    c.wpb = (int)tmin<size_t>(kWpb, (160 * 1024) / per);
    if (c.wpb < 1) {
        c.wpb = kWpb;
        c.global_acc = true;
        c.smem = 0;
    } else {
        c.global_acc = false;
        c.smem = per * c.wpb;
    }
    return c;
}

template <class IP>
int launch_csc(const IP* colptr, const int32_t* rowidx, const double* data, int64_t cols,
               int64_t row0, const int32_t* bucket, const int8_t* sign, int64_t L, double* Y,
               int accumulate, double* gacc, cudaStream_t st) {
    const CscLaunch cl = csc_launch(L);
    if (cl.smem > 48 * 1024)
        IDS_CUDA_TRY(cudaFuncSetAttribute(cs_csc_kernel<IP>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)cl.smem));
    const unsigned grid = (unsigned)ceil_div(cols, cl.wpb);
    cs_csc_kernel<IP><<<grid, cl.wpb * 32, cl.smem, st>>>(colptr, rowidx, data, cols, row0,
                                                          bucket, sign, L, cl.wpb, Y, accumulate,
                                                          cl.global_acc ? gacc : nullptr);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}

}  // namespace

extern "C" size_t ids_countsketch_csc_workspace_bytes(int64_t cols, int64_t out_dim) {
    WsCount c;
    if (csc_launch(out_dim).global_acc) c.take<double>((size_t)cols * out_dim);
    return c.off + 256;
}

extern "C" int ids_countsketch_csc_f64(const void* colptr, int colptr64, const int32_t* rowidx,
                                       const double* data, int64_t rows, int64_t cols,
                                       int64_t nnz, int64_t row0, int64_t in_dim,
                                       const int32_t* bucket, const int8_t* sign,
                                       int64_t out_dim, double* Y, int accumulate,
                                       int32_t* nonfinite, void* workspace, size_t ws_bytes,
                                       void* stream) {
    if (rows < 1 || cols < 1 || nnz < 0 || out_dim < 1 || row0 < 0 || row0 + rows > in_dim) {
        ids_set_last_error("csc countsketch: bad arguments");
        return IDS_EINVAL;
    }
    cudaStream_t st = as_stream(stream);
    WsCarve ws(workspace, ws_bytes);
    double* gacc = csc_launch(out_dim).global_acc ? ws.take<double>((size_t)cols * out_dim) : nullptr;
    if (!ws.ok()) {
        ids_set_last_error("csc countsketch: workspace too small");
        return IDS_EWORKSPACE;
    }
    int rc = colptr64 ? launch_csc(static_cast<const int64_t*>(colptr), rowidx, data, cols, row0,
                                   bucket, sign, out_dim, Y, accumulate, gacc, st)
                      : launch_csc(static_cast<const int32_t*>(colptr), rowidx, data, cols, row0,
                                   bucket, sign, out_dim, Y, accumulate, gacc, st);
    if (rc != IDS_OK) return rc;
    if (nonfinite) {
        // a stored NaN/Inf always leaves a NaN/Inf in Y; the host confirms
        // with ids_values_has_nonfinite before raising
        const unsigned g = (unsigned)tmin<int64_t>(ceil_div(out_dim * cols, 256), 148 * 4);
        nonfinite_values_kernel<<<g, 256, 0, st>>>(Y, out_dim * cols, nonfinite);
        IDS_LAUNCH_CHECK();
    }
    return IDS_OK;
}

extern "C" size_t ids_countsketch_csr_workspace_bytes(int64_t rows, int64_t cols, int64_t nnz,
                                                      int64_t out_dim) {
    (void)rows;
    WsCount c;
    c.take<int32_t>(nnz);  // row_of
    c.take<int32_t>(nnz);  // iota
    c.take<int32_t>(nnz);  // sorted keys
    c.take<int32_t>(nnz);  // perm
    c.take<int32_t>(nnz);  // csc rows
    c.take<double>(nnz);   // csc values
    c.take<int64_t>(cols + 1);
    c.take<char>(sort_bytes(nnz, cols));
    if (csc_launch(out_dim).global_acc) c.take<double>((size_t)cols * out_dim);
    return c.off + 256;
}

extern "C" int ids_countsketch_csr_f64(const void* indptr, int indptr64, const int32_t* indices,
                                       const double* data, int64_t rows, int64_t cols,
                                       int64_t nnz, int64_t row0, int64_t in_dim,
                                       const int32_t* bucket, const int8_t* sign,
                                       const int32_t* order_signed, const int64_t* bstart,
                                       int64_t out_dim, double* Y, int accumulate, int flags,
                                       int32_t* nonfinite, void* workspace, size_t ws_bytes,
                                       void* stream) {
    (void)order_signed;
    (void)bstart;
    (void)flags;
    if (rows < 1 || cols < 1 || nnz < 0 || nnz > 0x7fffffffLL || out_dim < 1 || row0 < 0 ||
        row0 + rows > in_dim) {
        ids_set_last_error("csr countsketch: bad arguments");
        return IDS_EINVAL;
    }
    cudaStream_t st = as_stream(stream);
    WsCarve ws(workspace, ws_bytes);
    int32_t* row_of = ws.take<int32_t>(nnz);
    int32_t* iota = ws.take<int32_t>(nnz);
    int32_t* keys = ws.take<int32_t>(nnz);
    int32_t* perm = ws.take<int32_t>(nnz);
    int32_t* crow = ws.take<int32_t>(nnz);
    double* cval = ws.take<double>(nnz);
    int64_t* colptr = ws.take<int64_t>(cols + 1);
    const size_t sb = sort_bytes(nnz, cols);
    void* tmp = ws.take<char>(sb);
    double* gacc = csc_launch(out_dim).global_acc ? ws.take<double>((size_t)cols * out_dim) : nullptr;
    if (!ws.ok()) {
        ids_set_last_error("csr countsketch: workspace too small");
        return IDS_EWORKSPACE;
    }
    if (nnz > 0) {
        const unsigned g = (unsigned)tmin<int64_t>(ceil_div(rows, 256), 148 * 16);
        if (indptr64)
            row_of_entry_kernel<<<g, 256, 0, st>>>(static_cast<const int64_t*>(indptr), rows,
                                                   row_of, iota);
        else
            row_of_entry_kernel<<<g, 256, 0, st>>>(static_cast<const int32_t*>(indptr), rows,
                                                   row_of, iota);
        IDS_LAUNCH_CHECK();
        size_t b = sb;
        IDS_CUDA_TRY(cub::DeviceRadixSort::SortPairs(
            tmp, b, reinterpret_cast<const uint32_t*>(indices), reinterpret_cast<uint32_t*>(keys),
            iota, perm, (int)nnz, 0, key_bits(cols), st));
        const unsigned g2 = (unsigned)tmin<int64_t>(ceil_div(nnz, 256), 148 * 16);
        gather_csc_kernel<<<g2, 256, 0, st>>>(perm, row_of, data, nnz, crow, cval);
        IDS_LAUNCH_CHECK();
        colptr_kernel<<<(unsigned)tmin<int64_t>(ceil_div(cols + 1, 256), 1024), 256, 0, st>>>(
            keys, nnz, cols, colptr);
        IDS_LAUNCH_CHECK();
    } else {
        IDS_CUDA_TRY(cudaMemsetAsync(colptr, 0, sizeof(int64_t) * (cols + 1), st));
    }
    int rc = launch_csc(colptr, crow, cval, cols, row0, bucket, sign, out_dim, Y, accumulate,
                        gacc, st);
    if (rc != IDS_OK) return rc;
    if (nonfinite) {
        // a stored NaN/Inf always leaves a NaN/Inf in Y; the host confirms
        // with ids_values_has_nonfinite before raising
        const unsigned g = (unsigned)tmin<int64_t>(ceil_div(out_dim * cols, 256), 148 * 4);
        nonfinite_values_kernel<<<g, 256, 0, st>>>(Y, out_dim * cols, nonfinite);
        IDS_LAUNCH_CHECK();
    }
    return IDS_OK;
}

extern "C" int ids_values_has_nonfinite(const double* v, int64_t n, int32_t* flag, void* stream) {
    if (n < 0) return IDS_EINVAL;
    if (n == 0) return IDS_OK;
    const unsigned g = (unsigned)tmin<int64_t>(ceil_div(n, 256), 148 * 16);
    nonfinite_values_kernel<<<g, 256, 0, as_stream(stream)>>>(v, n, flag);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}
