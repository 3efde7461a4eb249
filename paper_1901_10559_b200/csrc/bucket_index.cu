// Bucket index: the CSR structure of the L x I CountSketch operator.
//
// The reference materializes S as a scipy CSR array (sketch.py:108-114) whose
// row l lists the input rows i with h(i) = l in increasing i; scipy's S @ A
// then accumulates each bucket in that order.  Here the same structure is a
// stable device radix sort of (bucket, signed row) pairs plus per-bucket
// start offsets; the sketch kernels gather rows in exactly that order.
#include <cub/cub.cuh>

#include "common.cuh"

namespace {

__global__ void encode_rows_kernel(const int8_t* __restrict__ sign, int64_t n,
                                   int32_t* __restrict__ vals) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        vals[i] = enc_row((int32_t)i, sign[i]);
}

// bstart[l] = first sorted position with key >= l (lower bound), l = 0..L.
__global__ void bucket_starts_kernel(const int32_t* __restrict__ keys, int64_t n, int64_t L,
                                     int64_t* __restrict__ bstart) {
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l <= L;
         l += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)keys[mid] < l) lo = mid + 1;
            else hi = mid;
        }
        bstart[l] = lo;
    }
}

int key_bits(int64_t L) {
    int b = 0;
    while ((1LL << b) < L) ++b;
    return b < 1 ? 1 : b;
}

size_t sort_bytes(int64_t n, int64_t L) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr,
                                    (uint32_t*)nullptr, (const int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)n, 0, key_bits(L));
    return bytes;
}

}  // namespace

extern "C" size_t ids_bucket_index_workspace_bytes(int64_t in_dim, int64_t out_dim) {
    WsCount c;
    c.take<int32_t>(in_dim);
    c.take<int32_t>(in_dim);
    c.take<char>(sort_bytes(in_dim, out_dim));
    return c.off + 256;
}

extern "C" int ids_bucket_index(const int32_t* bucket, const int8_t* sign, int64_t in_dim,
                                int64_t out_dim, int32_t* order_signed, int64_t* bstart,
                                int32_t* sorted_bucket, void* workspace, size_t ws_bytes,
                                void* stream) {
    if (in_dim < 1 || out_dim < 1 || in_dim > 0x7fffffffLL) {
        ids_set_last_error("bucket index: dimensions out of range");
        return IDS_EINVAL;
    }
    cudaStream_t st = as_stream(stream);
    WsCarve ws(workspace, ws_bytes);
    int32_t* vals = ws.take<int32_t>(in_dim);
    int32_t* keys_tmp = ws.take<int32_t>(in_dim);
    int32_t* keys_out = sorted_bucket ? sorted_bucket : keys_tmp;
    const size_t sb = sort_bytes(in_dim, out_dim);
    void* tmp = ws.take<char>(sb);
    if (!ws.ok()) {
        ids_set_last_error("bucket index: workspace too small");
        return IDS_EWORKSPACE;
    }
    const unsigned grid = (unsigned)tmin<int64_t>(ceil_div(in_dim, 256), 148 * 16);
    encode_rows_kernel<<<grid, 256, 0, st>>>(sign, in_dim, vals);
    IDS_LAUNCH_CHECK();
    size_t b = sb;
    IDS_CUDA_TRY(cub::DeviceRadixSort::SortPairs(
        tmp, b, reinterpret_cast<const uint32_t*>(bucket), reinterpret_cast<uint32_t*>(keys_out),
        vals, order_signed, (int)in_dim, 0, key_bits(out_dim), st));
    const unsigned g2 = (unsigned)tmin<int64_t>(ceil_div(out_dim + 1, 256), 148 * 8);
    bucket_starts_kernel<<<g2, 256, 0, st>>>(keys_out, in_dim, out_dim, bstart);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}
