// TensorSketch for transforms longer than one CTA's shared memory holds
// (reference sketch.py:170-186 step by step): per mode, the CountSketch of
// the factor matrix (dense / CSC kernels) is zero-padded to M, transformed by
// a batched Stockham FFT whose passes run through global memory, and
// multiplied into the running spectrum; the inverse transform is folded
// modulo L (a circular convolution of length L is the linear one wrapped
// around; for a power-of-two L, M = L and nothing wraps).
//
// B200 mapping: every pass is one coalesced sweep over the batch -- a
// radix-4 butterfly per thread reads four runs M/4 apart and writes four
// adjacent runs of `s` elements (autosort: no bit reversal pass); the
// transform is HBM-bound at log4(M) read+write sweeps of 16 B per point.
// This is the off-config route (the BASELINE sketch lengths all run in the
// fused shared-memory kernels); it exists so that no length falls back to a
// library FFT.
#include "common.cuh"
#include "fft.cuh"

namespace {

using namespace ids_fft;

constexpr int kSpThreads = 256;

__global__ void __launch_bounds__(kSpThreads)
sp_pad_kernel(const double* __restrict__ y, int64_t nb, int64_t L, int64_t M,
              double2* __restrict__ z) {
    const int64_t tot = nb * M;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / M, t = i - b * M;
        z[i] = make_double2(t < L ? y[b * L + t] : 0.0, 0.0);
    }
}

// Two real rows in one complex transform: z = ya + i yb.
__global__ void __launch_bounds__(kSpThreads)
sp_pad2_kernel(const double* __restrict__ ya, const double* __restrict__ yb, int64_t nb, int64_t L,
               int64_t M, double2* __restrict__ z) {
    const int64_t tot = nb * M;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / M, t = i - b * M;
        z[i] = t < L ? make_double2(ya[b * L + t], yb[b * L + t]) : make_double2(0.0, 0.0);
    }
}

// Z = FFT(ya + i yb): FFT(ya)[k] = (Z[k] + conj Z[M-k]) / 2 and
// FFT(yb)[k] = (Z[k] - conj Z[M-k]) / (2i); their product enters the spectrum.
__global__ void __launch_bounds__(kSpThreads)
sp_mul2_kernel(double2* __restrict__ spec, const double2* __restrict__ z, int64_t nb, int64_t M,
               int first) {
    const int64_t tot = nb * M;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / M, k = i - b * M;
        const double2 zk = z[i], zm = conj2(z[b * M + ((M - k) & (M - 1))]);
        const double2 fa = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y + zm.y));
        const double2 df = csub(zk, zm);
        const double2 fb = make_double2(0.5 * df.y, -0.5 * df.x);  // df / (2i)
        const double2 pr = cmul(fa, fb);
        spec[i] = first ? pr : cmul(spec[i], pr);
    }
}

__device__ __forceinline__ double2 twiddle(int64_t p, int64_t n, int sign) {
    double sn, cs;
    sincospi(2.0 * (double)p / (double)n, &sn, &cs);
    return make_double2(cs, sign < 0 ? -sn : sn);
}

// One radix-4 pass of the Stockham autosort FFT on sub-length n at stride s
// (n * s = M): x -> y for every transform of the batch.
__global__ void __launch_bounds__(kSpThreads)
sp_r4_kernel(const double2* __restrict__ x, double2* __restrict__ y, int64_t nb, int64_t M,
             int64_t n, int64_t s, int sign) {
    const int64_t quarter = M >> 2, n1 = n >> 2, tot = nb * quarter;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / quarter, t = i - b * quarter;
        const int64_t p = t / s, q = t - p * s;
        const double2* xb = x + b * M;
        double2* yb = y + b * M;
        const double2 a = xb[q + s * p], bb = xb[q + s * (p + n1)], c = xb[q + s * (p + 2 * n1)],
                      d = xb[q + s * (p + 3 * n1)];
        const double2 w1 = twiddle(p, n, sign), w2 = cmul(w1, w1), w3 = cmul(w1, w2);
        const double2 apc = cadd(a, c), amc = csub(a, c), bpd = cadd(bb, d), bmd = csub(bb, d);
        // sign * i * (b - d)
        const double2 jb = sign < 0 ? make_double2(bmd.y, -bmd.x) : make_double2(-bmd.y, bmd.x);
        yb[q + s * (4 * p + 0)] = cadd(apc, bpd);
        yb[q + s * (4 * p + 1)] = cmul(w1, cadd(amc, jb));
        yb[q + s * (4 * p + 2)] = cmul(w2, csub(apc, bpd));
        yb[q + s * (4 * p + 3)] = cmul(w3, csub(amc, jb));
    }
}

__global__ void __launch_bounds__(kSpThreads)
sp_r2_kernel(const double2* __restrict__ x, double2* __restrict__ y, int64_t nb, int64_t M,
             int64_t n, int64_t s, int sign) {
    const int64_t half = M >> 1, m = n >> 1, tot = nb * half;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / half, t = i - b * half;
        const int64_t p = t / s, q = t - p * s;
        const double2* xb = x + b * M;
        double2* yb = y + b * M;
        const double2 a = xb[q + s * p], c = xb[q + s * (p + m)];
        yb[q + s * (2 * p + 0)] = cadd(a, c);
        yb[q + s * (2 * p + 1)] = cmul(twiddle(p, n, sign), csub(a, c));
    }
}

__global__ void __launch_bounds__(kSpThreads)
sp_mul_kernel(double2* __restrict__ spec, const double2* __restrict__ z, int64_t tot, int first) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot;
         i += (int64_t)gridDim.x * blockDim.x)
        spec[i] = first ? z[i] : cmul(spec[i], z[i]);
}

// out[b][l] = w[b] / M * sum over t = l, l + L, .. < M of Re z[b][t]
__global__ void __launch_bounds__(kSpThreads)
sp_fold_kernel(const double2* __restrict__ z, int64_t nb, int64_t L, int64_t M,
               const double* __restrict__ w, double* __restrict__ out) {
    const int64_t tot = nb * L;
    const double inv = 1.0 / (double)M;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / L, l = i - b * L;
        double acc = 0.0;
        for (int64_t t = l; t < M; t += L) acc += z[b * M + t].x;
        acc *= inv;
        out[i] = w ? acc * w[b] : acc;
    }
}

unsigned grid_for(int64_t work) {
    const int64_t cap = (int64_t)ids_sm_count() * 16;
    return (unsigned)tmax<int64_t>(1, tmin<int64_t>(ceil_div(work, (int64_t)kSpThreads), cap));
}

// In-place-looking batched FFT: the result of transforming `a` ends in the
// returned buffer (a or b, depending on the number of passes).
int fft_passes(double2* a, double2* b, int64_t nb, int64_t M, int sign, cudaStream_t st,
               const double2** result) {
    double2 *x = a, *y = b;
    int64_t n = M, s = 1;
    while (n >= 4) {
        sp_r4_kernel<<<grid_for(nb * (M >> 2)), kSpThreads, 0, st>>>(x, y, nb, M, n, s, sign);
        IDS_LAUNCH_CHECK();
        n >>= 2;
        s <<= 2;
        double2* t = x;
        x = y;
        y = t;
    }
    if (n == 2) {
        sp_r2_kernel<<<grid_for(nb * (M >> 1)), kSpThreads, 0, st>>>(x, y, nb, M, n, s, sign);
        IDS_LAUNCH_CHECK();
        double2* t = x;
        x = y;
        y = t;
    }
    *result = x;
    return IDS_OK;
}

bool pow2(int64_t v) { return v >= 1 && (v & (v - 1)) == 0; }

}  // namespace

extern "C" int64_t ids_ts_spectral_len(int n_modes, int64_t out_dim) {
    if (n_modes < 1 || out_dim < 1) return 0;
    if (pow2(out_dim)) return out_dim;
    const int64_t need = (int64_t)n_modes * (out_dim - 1) + 1;
    int64_t M = 2;
    while (M < need) M <<= 1;
    return M;
}

extern "C" int ids_ts_spectral_mode_f64(const double* y, int64_t nb, int64_t out_dim, int64_t M,
                                        double* spec, double* work, int first, void* stream) {
    if (!y || !spec || !work || nb < 1 || out_dim < 1 || M < out_dim || !pow2(M)) {
        ids_set_last_error("ts spectral mode: bad arguments");
        return IDS_EINVAL;
    }
    cudaStream_t st = as_stream(stream);
    double2* a = reinterpret_cast<double2*>(work);
    double2* b = a + nb * M;
    sp_pad_kernel<<<grid_for(nb * M), kSpThreads, 0, st>>>(y, nb, out_dim, M, a);
    IDS_LAUNCH_CHECK();
    const double2* z = nullptr;
    if (int rc = fft_passes(a, b, nb, M, -1, st, &z)) return rc;
    sp_mul_kernel<<<grid_for(nb * M), kSpThreads, 0, st>>>(reinterpret_cast<double2*>(spec), z,
                                                          nb * M, first);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}

extern "C" int ids_ts_spectral_pair_f64(const double* ya, const double* yb, int64_t nb,
                                        int64_t out_dim, int64_t M, double* spec, double* work,
                                        int first, void* stream) {
    if (!ya || !yb || !spec || !work || nb < 1 || out_dim < 1 || M < out_dim || !pow2(M)) {
        ids_set_last_error("ts spectral pair: bad arguments");
        return IDS_EINVAL;
    }
    cudaStream_t st = as_stream(stream);
    double2* a = reinterpret_cast<double2*>(work);
    double2* b = a + nb * M;
    sp_pad2_kernel<<<grid_for(nb * M), kSpThreads, 0, st>>>(ya, yb, nb, out_dim, M, a);
    IDS_LAUNCH_CHECK();
    const double2* z = nullptr;
    if (int rc = fft_passes(a, b, nb, M, -1, st, &z)) return rc;
    sp_mul2_kernel<<<grid_for(nb * M), kSpThreads, 0, st>>>(reinterpret_cast<double2*>(spec), z, nb,
                                                           M, first);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}

extern "C" int ids_ts_spectral_finish_f64(double* spec, int64_t nb, int64_t out_dim, int64_t M,
                                          const double* weights, double* work, double* out,
                                          void* stream) {
    if (!spec || !work || !out || nb < 1 || out_dim < 1 || M < out_dim || !pow2(M)) {
        ids_set_last_error("ts spectral finish: bad arguments");
        return IDS_EINVAL;
    }
    cudaStream_t st = as_stream(stream);
    const double2* z = nullptr;
    if (int rc = fft_passes(reinterpret_cast<double2*>(spec), reinterpret_cast<double2*>(work), nb, M,
                            +1, st, &z))
        return rc;
    sp_fold_kernel<<<grid_for(nb * out_dim), kSpThreads, 0, st>>>(z, nb, out_dim, M, weights, out);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}
