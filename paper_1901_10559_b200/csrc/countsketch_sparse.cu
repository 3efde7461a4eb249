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
    if (cl.smem > 40 * 1024)
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

static size_t csr_transpose_ws(int64_t cols, int64_t nnz, int64_t out_dim) {
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

// CSR -> CSC on the device: stable radix sort of the entries by column (row
// order kept inside each column), then gather rows/values and column starts.
static int build_csc(const void* indptr, int indptr64, const int32_t* indices, const double* data,
                     int64_t rows, int64_t cols, int64_t nnz, int32_t* row_of, int32_t* iota,
                     int32_t* keys, int32_t* perm, void* tmp, size_t sb, int32_t* crow,
                     double* cval, int64_t* colptr, cudaStream_t st) {
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
    return IDS_OK;
}

static int csr_transpose_path(const void* indptr, int indptr64, const int32_t* indices,
                              const double* data, int64_t rows, int64_t cols, int64_t nnz,
                              int64_t row0, int64_t in_dim, const int32_t* bucket,
                              const int8_t* sign, int64_t out_dim, double* Y, int accumulate,
                              int32_t* nonfinite, void* workspace, size_t ws_bytes,
                              cudaStream_t st) {
    if (rows < 1 || cols < 1 || nnz < 0 || nnz > 0x7fffffffLL || out_dim < 1 || row0 < 0 ||
        row0 + rows > in_dim) {
        ids_set_last_error("csr countsketch: bad arguments");
        return IDS_EINVAL;
    }
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
    {
        const int rc = build_csc(indptr, indptr64, indices, data, rows, cols, nnz, row_of, iota, keys,
                                 perm, tmp, sb, crow, cval, colptr, st);
        if (rc != IDS_OK) return rc;
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

// ---- direct CSR kernel ------------------------------------------------------
// One CTA per (bucket l, segment of the bucket's rows).  The CTA walks its
// rows in increasing order (the bucket index) in batches, gathers their
// nonzeros (coalesced within a row), and accumulates into an R-wide fp64
// accumulator in shared memory.  Determinism without atomics: the column
// range is split into 8 tiles, each owned by one warp; a stable block-wide
// counting sort routes every staged nonzero to its tile's list in row order,
// and the owner warp adds them with same-column lanes serialized by
// __match_any_sync rank.  Each Y entry therefore sums its rows in increasing
// row order (scipy's order: bit-identical with one segment per bucket).
constexpr int kCsrThreads = 256;
constexpr int kCsrOwners = 8;
constexpr int kCsrRows = 256;
constexpr int kCsrCap = 2048;  // staged nonzeros per sub-batch (8 per thread)
constexpr int64_t kCsrMaxCols = 16384;

__device__ __forceinline__ int64_t lower_bound_rows_csr(const int32_t* __restrict__ order,
                                                        int64_t lo, int64_t hi, int64_t row) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)dec_row(order[mid]) < row) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <class IP>
__global__ void __launch_bounds__(kCsrThreads) cs_csr_bucket_kernel(
    const IP* __restrict__ indptr, const int32_t* __restrict__ indices,
    const double* __restrict__ data, int64_t cols, int64_t row0, int64_t rows,
    int restrict_rows, const int32_t* __restrict__ order, const int64_t* __restrict__ bstart,
    int64_t L, int nseg, double* __restrict__ out, int64_t seg_stride, int init_from_out,
    int rpb) {
    extern __shared__ double acc[];  // cols
    __shared__ int64_t s_p0[kCsrRows];
    __shared__ int s_off[kCsrRows + 1];
    __shared__ int8_t s_sg[kCsrRows];
    __shared__ int s_col[kCsrCap];
    __shared__ uint8_t s_rowof[kCsrCap];  // batch row of each staged entry
    __shared__ double s_val[kCsrCap];
    __shared__ int s_base[kCsrOwners * 8 * kCsrOwners];  // [owner][q][warp]
    __shared__ int s_ostart[kCsrOwners + 1];
    typedef cub::BlockScan<int, kCsrThreads> BS;
    __shared__ typename BS::TempStorage scan_tmp;

    const int t = threadIdx.x, w = t >> 5, lane = t & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const int64_t l = blockIdx.x / nseg;
    const int seg = (int)(blockIdx.x % nseg);
    int64_t k0 = bstart[l], k1 = bstart[l + 1];
    if (restrict_rows) {
        const int64_t a = lower_bound_rows_csr(order, k0, k1, row0);
        k1 = lower_bound_rows_csr(order, a, k1, row0 + rows);
        k0 = a;
    }
    const int64_t len = k1 - k0;
    const int64_t s0 = k0 + len * seg / nseg, s1 = k0 + len * (seg + 1) / nseg;
    const int tw = (int)((cols + kCsrOwners - 1) / kCsrOwners);
    const float inv_tw = 1.0f / (float)tw;
    double* o = out + (int64_t)seg * seg_stride;
    for (int64_t c = t; c < cols; c += kCsrThreads) acc[c] = init_from_out ? o[c * L + l] : 0.0;

    // rpb rows per batch; the row pointers of batch b + 1 and the order entries
    // of batch b + 2 are loaded while batch b is processed
    auto batch_rows = [&](int64_t kb) { return kb < s1 ? (int)tmin<int64_t>(rpb, s1 - kb) : 0; };
    int32_t e_cur = t < batch_rows(s0) ? __ldg(order + s0 + t) : 0;
    int64_t q0 = 0, q1 = 0;
    if (t < batch_rows(s0)) {
        const int64_t row = (int64_t)dec_row(e_cur) - row0;
        q0 = (int64_t)indptr[row];
        q1 = (int64_t)indptr[row + 1];
    }
    int32_t e_nxt = t < batch_rows(s0 + rpb) ? __ldg(order + s0 + rpb + t) : 0;
    for (int64_t kb = s0; kb < s1; kb += rpb) {
        const int nr = batch_rows(kb);
        int cnt = 0;
        if (t < nr) {
            s_p0[t] = q0;
            s_sg[t] = e_cur >= 0 ? 1 : -1;
            cnt = (int)(q1 - q0);
        }
        int64_t n0 = 0, n1 = 0;
        if (t < batch_rows(kb + rpb)) {
            const int64_t row = (int64_t)dec_row(e_nxt) - row0;
            n0 = (int64_t)indptr[row];
            n1 = (int64_t)indptr[row + 1];
        }
        const int32_t e_nn = t < batch_rows(kb + 2 * rpb) ? __ldg(order + kb + 2 * rpb + t) : 0;
        e_cur = e_nxt;
        e_nxt = e_nn;
        int off, E;
        BS(scan_tmp).ExclusiveSum(cnt, off, E);
        if (t < nr) s_off[t] = off;
        if (t == 0) s_off[nr] = E;
        __syncthreads();
        for (int f0 = 0; f0 < E; f0 += kCsrCap) {
            const int nE = min(kCsrCap, E - f0);
            int myo[8], myc[8], rk[8];
            double myv[8];
            for (int i = t; i < kCsrOwners * 8 * kCsrOwners; i += kCsrThreads) s_base[i] = 0;
            // row of every staged entry: each row's thread fills its slots
            if (t < nr) {
                const int a = max(off, f0), b = min(off + cnt, f0 + nE);
                for (int f = a; f < b; ++f) s_rowof[f - f0] = (uint8_t)t;
            }
            __syncthreads();
            // eight independent (index, value) loads per thread
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int fl = q * kCsrThreads + t;
                const bool ok = fl < nE;
                const int tr = ok ? s_rowof[fl] : 0;
                const int64_t p = ok ? s_p0[tr] + (f0 + fl - s_off[tr]) : 0;
                myc[q] = ok ? __ldg(indices + p) : 0;
                const double v = ok ? __ldcs(data + p) : 0.0;
                myv[q] = s_sg[tr] < 0 ? -v : v;
                myo[q] = -1;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (q * kCsrThreads + t < nE) {
                    int ow = (int)((float)myc[q] * inv_tw);  // col / tw without a divide
                    ow -= (ow * tw > myc[q]) ? 1 : 0;
                    ow += ((ow + 1) * tw <= myc[q]) ? 1 : 0;
                    myo[q] = ow;
                }
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t peers = __match_any_sync(0xffffffffu, myo[q]);
                rk[q] = __popc(peers & lt);
                if (myo[q] >= 0 && rk[q] == 0)
                    s_base[(myo[q] * 8 + q) * kCsrOwners + w] = __popc(peers);
            }
            __syncthreads();
            {  // exclusive scan over (owner, q, warp): 512 counters, 2 per thread
                const int a0 = s_base[2 * t], a1 = s_base[2 * t + 1];
                int ex, tot;
                BS(scan_tmp).ExclusiveSum(a0 + a1, ex, tot);
                __syncthreads();
                s_base[2 * t] = ex;
                s_base[2 * t + 1] = ex + a0;
            }
            __syncthreads();
            if (t <= kCsrOwners) s_ostart[t] = t < kCsrOwners ? s_base[t * 8 * kCsrOwners] : nE;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (myo[q] >= 0) {
                    const int pos = s_base[(myo[q] * 8 + q) * kCsrOwners + w] + rk[q];
                    s_col[pos] = myc[q];
                    s_val[pos] = myv[q];
                }
            }
            __syncthreads();
            {  // owner warp w adds its tile's entries in row order
                const int a = s_ostart[w], b = s_ostart[w + 1];
                for (int ib = a; ib < b; ib += 32) {
                    const int i = ib + lane;
                    const bool act = i < b;
                    const int c = act ? s_col[i] : -1 - lane;
                    const double v = act ? s_val[i] : 0.0;
                    const uint32_t peers = __match_any_sync(0xffffffffu, c);
                    const int r = __popc(peers & lt);
                    const int maxr = (int)__reduce_max_sync(0xffffffffu, (unsigned)(act ? r : 0));
                    for (int rr = 0; rr <= maxr; ++rr) {
                        if (act && r == rr) acc[c] += v;
                        __syncwarp();
                    }
                }
            }
            __syncthreads();
        }
        q0 = n0;
        q1 = n1;
    }
    __syncthreads();
    for (int64_t c = t; c < cols; c += kCsrThreads) o[c * L + l] = acc[c];
}

// ---- streaming CSR kernel ---------------------------------------------------
// The default path (neither IDS_FLAG_ORDERED nor IDS_FLAG_DETERMINISTIC):
// A is read exactly once, in storage order, with coalesced streaming loads,
// and every nonzero becomes one fp64 reduction (RED.ADD.F64, resolved in L2)
// into Y[col * L + bucket(row)].  Y (L x cols doubles) stays L2-resident; the
// bound is the L2 reduction rate (~1.7e11 fp64 REDs/s measured on B200), not
// HBM.  The summation order inside one Y entry is not fixed, so Y differs
// from scipy's order by rounding only.
//
// Each CTA owns a contiguous range of 2048-entry tiles.  Per tile one warp
// finds the row holding the first entry (32-way split search), the next 256
// rows stamp their (bucket, sign) code over their entries in shared memory,
// and every thread then loads its 8 entries (coalesced across the warp) and
// issues their reductions.  22 registers: 8 CTAs (2048 threads) per SM keep
// enough loads and reductions in flight (4 CTAs/SM measured 1.5x slower).
constexpr int kStrThreads = 256;
constexpr int kStrPer = 8;
constexpr int kStrTile = kStrThreads * kStrPer;

// last r in [0, rows) with indptr[r] <= p (the row holding entry p when
// indptr[0] <= p < indptr[rows]); one warp, 32-way split per step
template <class IP>
__device__ int64_t csr_row_of_entry_warp(const IP* __restrict__ indptr, int64_t rows, int64_t p) {
    const int lane = threadIdx.x & 31;
    int64_t lo = 0, hi = rows - 1;  // answer in [lo, hi]
    while (hi - lo > 32) {
        const int64_t span = hi - lo;
        const int64_t probe = lo + 1 + (span - 1) * lane / 32;  // in (lo, hi]
        const bool le = (int64_t)indptr[probe] <= p;
        const uint32_t m = __ballot_sync(0xffffffffu, le);
        const int k = 31 - __clz((int)m);  // last lane whose probe is <= p (-1 if none)
        const int64_t nlo = k >= 0 ? __shfl_sync(0xffffffffu, probe, k) : lo;
        const int64_t nhi = k < 31 ? __shfl_sync(0xffffffffu, probe, k + 1) - 1 : hi;
        lo = nlo;
        hi = nhi;
    }
    const int64_t probe = lo + lane;
    const bool le = probe <= hi && (int64_t)indptr[probe] <= p;
    const uint32_t m = __ballot_sync(0xffffffffu, le);
    return lo + (31 - __clz((int)m));
}

template <class IP>
__global__ void __launch_bounds__(kStrThreads, 8) cs_csr_stream_kernel(
    const IP* __restrict__ indptr, const int32_t* __restrict__ indices,
    const double* __restrict__ data, int64_t rows, int64_t row0,
    const int32_t* __restrict__ bucket, const int8_t* __restrict__ sign, int64_t L,
    double* __restrict__ Y, int64_t tiles_per_cta) {
    __shared__ int32_t s_code[kStrTile];
    __shared__ int64_t s_r0;
    const int t = threadIdx.x;
    const int64_t pbeg = (int64_t)indptr[0], pend = (int64_t)indptr[rows];
    const int64_t ntiles = (pend - pbeg + kStrTile - 1) / kStrTile;
    const int64_t tb = (int64_t)blockIdx.x * tiles_per_cta;
    const int64_t te = tmin<int64_t>(ntiles, tb + tiles_per_cta);
    for (int64_t tile = tb; tile < te; ++tile) {
        const int64_t p0 = pbeg + tile * kStrTile;
        const int n = (int)tmin<int64_t>(kStrTile, pend - p0);
        const int64_t p1 = p0 + n;
        if (t < 32) {
            const int64_t r = csr_row_of_entry_warp(indptr, rows, p0);
            if (t == 0) s_r0 = r;
        }
        __syncthreads();
        // rows r.. stamp their codes until some row reaches p1 (empty rows
        // cost a pass of 256 each; a row longer than the tile is stamped by
        // its one thread)
        for (int64_t r = s_r0;; r += kStrThreads) {
            const int64_t rr = r + t;
            int64_t b = p1;
            if (rr < rows) {
                const int64_t a = (int64_t)indptr[rr];
                b = (int64_t)indptr[rr + 1];
                if (a < p1 && b > p0) {
                    const int32_t code = enc_row(__ldg(bucket + row0 + rr), __ldg(sign + row0 + rr));
                    const int lo = (int)(tmax(a, p0) - p0), hi = (int)(tmin(b, p1) - p0);
                    for (int x = lo; x < hi; ++x) s_code[x] = code;
                }
            }
            if (__syncthreads_or(rr < rows && b >= p1) || r + kStrThreads >= rows) break;
        }
#pragma unroll
        for (int q = 0; q < kStrPer; ++q) {
            const int f = q * kStrThreads + t;
            if (f < n) {
                const int c = __ldcs(indices + p0 + f);
                const double v = __ldcs(data + p0 + f);
                const int32_t e = s_code[f];
                atomicAdd(Y + (int64_t)c * L + dec_row(e), e >= 0 ? v : -v);
            }
        }
        __syncthreads();  // s_code and s_r0 are rewritten by the next tile
    }
}

template <class IP>
static int launch_csr_stream(const IP* indptr, const int32_t* indices, const double* data,
                             int64_t rows, int64_t nnz, int64_t row0, const int32_t* bucket,
                             const int8_t* sign, int64_t L, double* Y, cudaStream_t st) {
    if (nnz <= 0) return IDS_OK;
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    IDS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cs_csr_stream_kernel<IP>,
                                                               kStrThreads, 0));
    const int64_t ntiles = ceil_div(nnz, kStrTile);
    const int64_t slots = (int64_t)sms * tmax(1, per_sm);
    const int64_t per_cta = ceil_div(ntiles, slots);
    const unsigned grid = (unsigned)ceil_div(ntiles, per_cta);
    cs_csr_stream_kernel<IP><<<grid, kStrThreads, 0, st>>>(indptr, indices, data, rows, row0,
                                                           bucket, sign, L, Y, per_cta);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}

__global__ void csr_seg_reduce_kernel(const double* __restrict__ part, int nseg, int64_t n,
                                      double* __restrict__ Y, int accumulate) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        double a = accumulate ? Y[e] : 0.0;
        for (int s = 0; s < nseg; ++s) a += part[(int64_t)s * n + e];
        Y[e] = a;
    }
}

// Segments per bucket for the unordered mode: the grid is out_dim * nseg
// CTAs over `slots` resident CTAs; pick the nseg in [1, 16] that minimizes the
// (wave-quantized) time waves / nseg -- the fewest segments within 5% of the
// best (less partial traffic) -- keeping the partials under 1 GB.
static int csr_nseg(int64_t out_dim, int64_t cols, int flags) {
    if (flags & IDS_FLAG_ORDERED) return 1;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t per_sm = tmax<int64_t>(1, tmin<int64_t>(2, (227 * 1024) / (cols * 8 + 34 * 1024)));
    const int64_t slots = sms * per_sm;
    double t[17];
    int nmax = 1;
    double best_t = 1e30;
    for (int n = 1; n <= 16; ++n) {
        if (n > 1 && (double)n * cols * out_dim * 8.0 > 1e9) break;
        t[n] = (double)ceil_div(out_dim * n, slots) / n;
        best_t = fmin(best_t, t[n]);
        nmax = n;
    }
    for (int n = 1; n <= nmax; ++n)  // fewest segments within 5% of the best
        if (t[n] <= 1.05 * best_t) return n;
    return 1;
}

extern "C" size_t ids_countsketch_csr_workspace_bytes(int64_t rows, int64_t cols, int64_t nnz,
                                                      int64_t out_dim) {
    (void)rows;
    if (cols <= kCsrMaxCols) {
        WsCount c;
        c.take<double>((size_t)csr_nseg(out_dim, cols, 0) * cols * out_dim);
        return c.off + 256;
    }
    return csr_transpose_ws(cols, nnz, out_dim);
}

extern "C" int ids_countsketch_csr_f64(const void* indptr, int indptr64, const int32_t* indices,
                                       const double* data, int64_t rows, int64_t cols,
                                       int64_t nnz, int64_t row0, int64_t in_dim,
                                       const int32_t* bucket, const int8_t* sign,
                                       const int32_t* order_signed, const int64_t* bstart,
                                       int64_t out_dim, double* Y, int accumulate, int flags,
                                       int32_t* nonfinite, void* workspace, size_t ws_bytes,
                                       void* stream) {
    cudaStream_t st = as_stream(stream);
    if (!(flags & (IDS_FLAG_ORDERED | IDS_FLAG_DETERMINISTIC))) {
        if (rows < 1 || cols < 1 || nnz < 0 || out_dim < 1 || row0 < 0 || row0 + rows > in_dim) {
            ids_set_last_error("csr countsketch: bad arguments");
            return IDS_EINVAL;
        }
        if (!accumulate) IDS_CUDA_TRY(cudaMemsetAsync(Y, 0, sizeof(double) * cols * out_dim, st));
        const int rc =
            indptr64 ? launch_csr_stream(static_cast<const int64_t*>(indptr), indices, data, rows,
                                         nnz, row0, bucket, sign, out_dim, Y, st)
                     : launch_csr_stream(static_cast<const int32_t*>(indptr), indices, data, rows,
                                         nnz, row0, bucket, sign, out_dim, Y, st);
        if (rc != IDS_OK) return rc;
        if (nonfinite) {
            const unsigned g = (unsigned)tmin<int64_t>(ceil_div(cols * out_dim, 256), 148 * 4);
            nonfinite_values_kernel<<<g, 256, 0, st>>>(Y, cols * out_dim, nonfinite);
            IDS_LAUNCH_CHECK();
        }
        return IDS_OK;
    }
    if (cols > kCsrMaxCols || !order_signed || !bstart)
        return csr_transpose_path(indptr, indptr64, indices, data, rows, cols, nnz, row0, in_dim,
                                  bucket, sign, out_dim, Y, accumulate, nonfinite, workspace,
                                  ws_bytes, st);
    if (rows < 1 || cols < 1 || nnz < 0 || out_dim < 1 || row0 < 0 || row0 + rows > in_dim) {
        ids_set_last_error("csr countsketch: bad arguments");
        return IDS_EINVAL;
    }
    const int nseg = csr_nseg(out_dim, cols, flags);
    WsCarve ws(workspace, ws_bytes);
    double* part = nseg > 1 ? ws.take<double>((size_t)nseg * cols * out_dim) : nullptr;
    if (!ws.ok()) {
        ids_set_last_error("csr countsketch: workspace too small");
        return IDS_EWORKSPACE;
    }
    double* out = nseg > 1 ? part : Y;
    const int64_t stride = cols * out_dim;
    const int init = (nseg == 1 && accumulate) ? 1 : 0;
    const int restrict_rows = (row0 != 0 || rows != in_dim) ? 1 : 0;
    const size_t smem = (size_t)cols * sizeof(double);
    const unsigned grid = (unsigned)(out_dim * nseg);
    // rows per batch: about 0.85 of a staging round of nonzeros on average
    const double avg = rows > 0 ? (double)nnz / (double)rows : 1.0;
    const int rpb = (int)tmax<int64_t>(32, tmin<int64_t>(kCsrRows, (int64_t)(0.85 * kCsrCap / tmax(avg, 1.0))));
    if (indptr64) {
        IDS_CUDA_TRY(cudaFuncSetAttribute(cs_csr_bucket_kernel<int64_t>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cs_csr_bucket_kernel<int64_t><<<grid, kCsrThreads, smem, st>>>(
            static_cast<const int64_t*>(indptr), indices, data, cols, row0, rows, restrict_rows,
            order_signed, bstart, out_dim, nseg, out, stride, init, rpb);
    } else {
        IDS_CUDA_TRY(cudaFuncSetAttribute(cs_csr_bucket_kernel<int32_t>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cs_csr_bucket_kernel<int32_t><<<grid, kCsrThreads, smem, st>>>(
            static_cast<const int32_t*>(indptr), indices, data, cols, row0, rows, restrict_rows,
            order_signed, bstart, out_dim, nseg, out, stride, init, rpb);
    }
    IDS_LAUNCH_CHECK();
    if (nseg > 1) {
        const unsigned g = (unsigned)tmin<int64_t>(ceil_div(stride, 256), 148 * 8);
        csr_seg_reduce_kernel<<<g, 256, 0, st>>>(part, nseg, stride, Y, accumulate);
        IDS_LAUNCH_CHECK();
    }
    if (nonfinite) {
        const unsigned g = (unsigned)tmin<int64_t>(ceil_div(stride, 256), 148 * 4);
        nonfinite_values_kernel<<<g, 256, 0, st>>>(Y, stride, nonfinite);
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

// ---- public transpose (CSR of A^T, i.e. CSC of A) ---------------------------
extern "C" size_t ids_csr_transpose_workspace_bytes(int64_t rows, int64_t cols, int64_t nnz) {
    (void)rows;
    WsCount c;
    for (int i = 0; i < 4; ++i) c.take<int32_t>(nnz);
    c.take<char>(sort_bytes(nnz, cols));
    return c.off + 256;
}

extern "C" int ids_csr_transpose_f64(const void* indptr, int indptr64, const int32_t* indices,
                                     const double* data, int64_t rows, int64_t cols, int64_t nnz,
                                     int64_t* t_indptr, int32_t* t_indices, double* t_data,
                                     void* workspace, size_t ws_bytes, void* stream) {
    if (rows < 0 || cols < 1 || nnz < 0 || nnz > 0x7fffffffLL) {
        ids_set_last_error("csr transpose: bad arguments");
        return IDS_EINVAL;
    }
    WsCarve ws(workspace, ws_bytes);
    int32_t* row_of = ws.take<int32_t>(nnz);
    int32_t* iota = ws.take<int32_t>(nnz);
    int32_t* keys = ws.take<int32_t>(nnz);
    int32_t* perm = ws.take<int32_t>(nnz);
    const size_t sb = sort_bytes(nnz, cols);
    void* tmp = ws.take<char>(sb);
    if (!ws.ok()) {
        ids_set_last_error("csr transpose: workspace too small");
        return IDS_EWORKSPACE;
    }
    return build_csc(indptr, indptr64, indices, data, rows, cols, nnz, row_of, iota, keys, perm,
                     tmp, sb, t_indices, t_data, t_indptr, as_stream(stream));
}
