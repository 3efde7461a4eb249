// Fused TensorSketch kernel (replaces reference sketch.py:156-186).
//
// The reference evaluates, for the R columns of the N factor matrices,
//   Y = irfft_L( prod_n rfft_L( S_n A_n ) ) * diag(weights)
// with one scipy csr_matvecs per mode, pocketfft transforms and an L x R
// spectrum held in host memory.  Here ONE CTA owns one column r and runs the
// whole chain on chip:
//   for each mode n:
//     c_n[l] = sum over the rows of bucket l (increasing row, the bucket index)
//              of sign * A_n[row, r]         -> written straight into the
//              packed complex FFT buffer (z[m] = c[2m] + i c[2m+1]),
//     Z = FFT_{M/2}(z)   (mixed radix-8/4/2 Stockham passes in shared memory),
//     X = untangle(Z)    (real-input spectrum, bins 0..M/2),
//     S *= X             (running spectrum held in REGISTERS, 2 bins / pair),
//   then the inverse through the same half-length transform, x weight[r],
//   and a contiguous store of column r of Y (col-major L x R).
// The Khatri-Rao column (prod I_n entries) is never formed and the spectrum
// never leaves the SM.
//
// M = L when L is a power of two (cyclic convolution == the reference's
// length-L transforms).  Otherwise the per-mode sketches are zero-padded to
// M = 2^ceil(log2(N(L-1)+1)), the product gives their LINEAR convolution
// exactly, and it is folded mod L -- the same cyclic convolution the
// reference's length-L rfft/irfft computes (sketch.py:176-178).
#include <math.h>

#include "common.cuh"

namespace {

constexpr int kMaxModes = 8;
constexpr int kMaxHalf = 8192;  // largest half-length transform kept in shared memory
constexpr int kStage = 2048;    // sorted CountSketch entries staged per round

struct TsArgs {
    int n_modes;
    const double* factors[kMaxModes];
    int64_t lds[kMaxModes];
    const int32_t* order[kMaxModes];
    const int32_t* keys[kMaxModes];   // bucket of each sorted entry
    int64_t dims[kMaxModes];
    int64_t ncols, L, M, N2;
    int linear;  // 1: zero-pad + fold (L not a power of two)
    const double* weights;
    double* Y;
    double* colnorm2;
    const double2* tw;    // tw[m] = exp(-2 pi i m / M), m < M
    double2* spec_glob;   // per-CTA running spectrum (N2 + 1 bins) when not in smem
    int spec_in_smem;
    int64_t* tlog;        // debug: per-phase ns accumulated by CTA 0 (NULL: off)
};

__device__ __forceinline__ int64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return (int64_t)t;
}

__device__ __forceinline__ int pad(int i) { return i + (i >> 3); }

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 conj2(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }  // * -i

template <int R>
__device__ __forceinline__ void dft(double2* v);

template <>
__device__ __forceinline__ void dft<2>(double2* v) {
    const double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
}

template <>
__device__ __forceinline__ void dft<4>(double2* v) {
    const double2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
    const double2 s13 = cadd(v[1], v[3]), d13 = mul_mi(csub(v[1], v[3]));
    v[0] = cadd(s02, s13);
    v[2] = csub(s02, s13);
    v[1] = cadd(d02, d13);
    v[3] = csub(d02, d13);
}

template <>
__device__ __forceinline__ void dft<8>(double2* x) {
    const double s = 0.70710678118654752440;
    double2 a0 = cadd(x[0], x[4]), a4 = csub(x[0], x[4]);
    double2 a1 = cadd(x[1], x[5]), a5 = csub(x[1], x[5]);
    double2 a2 = cadd(x[2], x[6]), a6 = csub(x[2], x[6]);
    double2 a3 = cadd(x[3], x[7]), a7 = csub(x[3], x[7]);
    a5 = make_double2(s * (a5.x + a5.y), s * (a5.y - a5.x));     // * (s, -s)
    a6 = mul_mi(a6);                                            // * -i
    a7 = make_double2(s * (a7.y - a7.x), -s * (a7.x + a7.y));    // * (-s, -s)
    const double2 b0 = cadd(a0, a2), b2 = csub(a0, a2);
    const double2 b1 = cadd(a1, a3), b3 = mul_mi(csub(a1, a3));
    const double2 b4 = cadd(a4, a6), b6 = csub(a4, a6);
    const double2 b5 = cadd(a5, a7), b7 = mul_mi(csub(a5, a7));
    x[0] = cadd(b0, b1);
    x[4] = csub(b0, b1);
    x[2] = cadd(b2, b3);
    x[6] = csub(b2, b3);
    x[1] = cadd(b4, b5);
    x[5] = csub(b4, b5);
    x[3] = cadd(b6, b7);
    x[7] = csub(b6, b7);
}

// exp(-2 pi i m / M) from two small shared-memory tables:
// coarse[m >> 7] * fine[m & 127]  (M a power of two).
struct Twiddle {
    const double2* coarse;
    const double2* fine;
    __device__ __forceinline__ double2 operator()(int m) const {
        return cmul(coarse[m >> 7], fine[m & 127]);
    }
};

// One in-place Stockham pass of radix R over the N2-point buffer; every
// thread holds EPT >= N2 / blockDim.x points in registers across the barrier.
template <int R, int EPT>
__device__ void stockham_pass(double2* buf, int N2, int Ns, int M, const Twiddle tw) {
    const int B = N2 / R;
    const int T = blockDim.x;
    constexpr int kSlots = EPT / R;  // butterflies per thread
    double2 v[kSlots][R];
#pragma unroll
    for (int s = 0; s < kSlots; ++s) {
        const int j = threadIdx.x + s * T;
        if (j < B) {
#pragma unroll
            for (int r = 0; r < R; ++r) v[s][r] = buf[pad(j + r * B)];
            const int k = j % Ns;
            if (Ns > 1 && k != 0) {
                const double2 w1 = tw(k * (M / (Ns * R)));
                double2 w = w1;
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    v[s][r] = cmul(v[s][r], w);
                    if (r + 1 < R) w = cmul(w, w1);
                }
            }
            dft<R>(v[s]);
        }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < kSlots; ++s) {
        const int j = threadIdx.x + s * T;
        if (j < B) {
            const int k = j % Ns;
            const int base = (j / Ns) * Ns * R + k;
#pragma unroll
            for (int r = 0; r < R; ++r) buf[pad(base + r * Ns)] = v[s][r];
        }
    }
    __syncthreads();
}

// Radix-8 passes while each thread holds 8 points; with 16 points per thread
// (the longest transforms) radix-4 passes keep the live set in registers.
template <int EPT>
__device__ __forceinline__ void fft_forward(double2* buf, int N2, int M, const Twiddle tw) {
    int Ns = 1;
    constexpr int RMAX = EPT >= 16 ? 4 : 8;
    while (Ns * RMAX <= N2) {
        stockham_pass<RMAX, EPT>(buf, N2, Ns, M, tw);
        Ns *= RMAX;
    }
    const int rem = N2 / Ns;
    if (rem == 4) stockham_pass<4, EPT>(buf, N2, Ns, M, tw);
    else if (rem == 2) stockham_pass<2, EPT>(buf, N2, Ns, M, tw);
}

__global__ void twiddle_kernel(double2* tw, int64_t M) {
    for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < M;
         m += (int64_t)gridDim.x * blockDim.x) {
        double s, c;
        sincospi(2.0 * (double)m / (double)M, &s, &c);
        tw[m] = make_double2(c, -s);
    }
}

template <int EPT>
__global__ void __launch_bounds__(512, 1) tensorsketch_kernel(TsArgs g) {
    extern __shared__ double2 buf[];
    __shared__ double2 tw_coarse[kMaxHalf * 2 / 128 + 1];
    __shared__ double2 tw_fine[128];
    __shared__ const double* s_fac[kMaxModes];
    __shared__ const int32_t* s_ord[kMaxModes];
    __shared__ const int32_t* s_key[kMaxModes];
    __shared__ int64_t s_ld[kMaxModes];
    __shared__ int s_dim[kMaxModes];
    double* dbuf = reinterpret_cast<double*>(buf);
    const int T = blockDim.x, t = threadIdx.x;
    const int N2 = (int)g.N2, M = (int)g.M;
    const int L = (int)g.L;
    if (t == 0) {
#pragma unroll
        for (int q = 0; q < kMaxModes; ++q) {  // static indexing: no local copy of g
            s_fac[q] = g.factors[q];
            s_ord[q] = g.order[q];
            s_key[q] = g.keys[q];
            s_ld[q] = g.lds[q];
            s_dim[q] = (int)g.dims[q];
        }
    }
    for (int m = t; m < 128; m += T) {
        double sn, cs;
        sincospi(2.0 * (double)m / (double)M, &sn, &cs);
        tw_fine[m] = make_double2(cs, -sn);
    }
    for (int q = t; q * 128 < M; q += T) {
        double sn, cs;
        sincospi(2.0 * (double)q * 128.0 / (double)M, &sn, &cs);
        tw_coarse[q] = make_double2(cs, -sn);
    }
    __syncthreads();
    const Twiddle tw{tw_coarse, tw_fine};
    const int npairs = N2 / 2 + 1;  // pairs (p, N2 - p), p = 0..N2/2
    // running spectrum S[0..N2]: after the padded FFT buffer in smem, or in
    // this CTA's global (L2-resident) slice
    double2* spec = g.spec_in_smem ? buf + (N2 + N2 / 8 + 1)
                                   : g.spec_glob + (int64_t)blockIdx.x * (N2 + 1);
    double* st_val = reinterpret_cast<double*>(buf + (N2 + N2 / 8 + 1) +
                                               (g.spec_in_smem ? (N2 + 1) : 0));
    int32_t* st_key = reinterpret_cast<int32_t*>(st_val + kStage);
    const bool tl = g.tlog && blockIdx.x == 0 && t == 0;
    int64_t tprev = tl ? gtimer() : 0;
    auto stamp = [&](int phase) {
        if (tl) {
            const int64_t tn = gtimer();
            g.tlog[phase] += tn - tprev;
            tprev = tn;
        }
    };
    for (int64_t r = blockIdx.x; r < g.ncols; r += gridDim.x) {
        // passes 0..N-1: forward transform of mode n's CountSketch, product into S;
        // pass N: inverse transform of S (one inlined FFT for all passes)
        for (int n = 0; n <= g.n_modes; ++n) {
            if (n < g.n_modes) {
                // ---- per-mode CountSketch of column r, into the packed buffer ----
                // zero the M slots, then one thread per bucket run of the sorted
                // index sums its rows in increasing row order (scipy's order)
                const double* col = s_fac[n] + r * s_ld[n];
                const int32_t* ord = s_ord[n];
                const int32_t* key = s_key[n];
                const int In = s_dim[n];
                for (int l = t; l < M; l += T) dbuf[2 * pad(l >> 1) + (l & 1)] = 0.0;
                stamp(0);
                // stage kStage sorted entries at a time: bucket + signed value,
                // all loads independent (coalesced index reads, column gather)
                for (int c0 = 0; c0 < In; c0 += kStage) {
                    const int cn = min(kStage, In - c0);
                    for (int qb = 0; qb < cn; qb += 4 * T) {  // 4 entries per thread in flight
                        int32_t e[4], kq[4];
                        double x[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int q = qb + u * T + t;
                            e[u] = q < cn ? __ldg(ord + c0 + q) : 0;
                            kq[u] = q < cn ? __ldg(key + c0 + q) : 0;
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int q = qb + u * T + t;
                            x[u] = q < cn ? __ldg(col + dec_row(e[u])) : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int q = qb + u * T + t;
                            if (q < cn) {
                                st_key[q] = kq[u];
                                st_val[q] = e[u] >= 0 ? x[u] : -x[u];
                            }
                        }
                    }
                    __syncthreads();
                    stamp(1);
                    // run heads sum their bucket's rows in increasing row order
                    for (int q = t; q < cn; q += T) {
                        const int32_t bkt = st_key[q];
                        const bool head = q > 0 ? st_key[q - 1] != bkt
                                                : (c0 == 0 || __ldg(key + c0 - 1) != bkt);
                        if (!head) continue;
                        double acc = 0.0;
                        int kk = q;
                        while (kk < cn && st_key[kk] == bkt) acc += st_val[kk++];
                        int kg = c0 + kk;  // run continues past the staged block (rare)
                        while (kg < In && __ldg(key + kg) == bkt) {
                            const int32_t e = __ldg(ord + kg);
                            const double x = __ldg(col + dec_row(e));
                            acc = e >= 0 ? acc + x : acc - x;
                            ++kg;
                        }
                        dbuf[2 * pad(bkt >> 1) + (bkt & 1)] = acc;
                    }
                    __syncthreads();
                    stamp(2);
                }
            } else {
                // ---- inverse: pack conj(Z) from S, forward FFT, conj ----
                for (int p = t; p < npairs; p += T) {
                    const double2 xk = spec[p], xm = spec[N2 - p];  // S[p], S[N2 - p]
                    const double2 w = tw(p);
                    const double2 e = make_double2(0.5 * (xk.x + xm.x), 0.5 * (xk.y - xm.y));
                    const double2 d = make_double2(0.5 * (xk.x - xm.x), 0.5 * (xk.y + xm.y));
                    const double2 o = cmul(d, conj2(w));
                    // Z[p] = E + iO ; Z[N2-p] = conj(E) + i conj(O); stored conjugated
                    const double2 zlo = make_double2(e.x - o.y, e.y + o.x);
                    const double2 zhi = make_double2(e.x + o.y, -e.y + o.x);
                    if (p < N2) buf[pad(p)] = conj2(zlo);
                    const int pm = N2 - p;
                    if (pm != p && pm < N2 && pm > 0) buf[pad(pm)] = conj2(zhi);
                }
            }
            __syncthreads();
            stamp(3);
            fft_forward<EPT>(buf, N2, M, tw);
            stamp(4);
            if (n < g.n_modes) {
                // ---- untangle the real spectrum, multiply into S ----
                for (int p = t; p < npairs; p += T) {
                    const double2 zk = buf[pad(p % N2)];
                    const double2 zm = buf[pad((N2 - p) % N2)];
                    const double2 e = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
                    const double2 d = make_double2(zk.x - zm.x, zk.y + zm.y);  // zk - conj(zm)
                    const double2 o = make_double2(0.5 * d.y, -0.5 * d.x);   // d * (-i/2)
                    const double2 wo = cmul(tw(p), o);
                    const double2 xlo = cadd(e, wo);
                    const double2 xhi = conj2(csub(e, wo));
                    if (n == 0) {
                        spec[p] = xlo;
                        if (N2 - p != p) spec[N2 - p] = xhi;
                    } else {
                        spec[p] = cmul(spec[p], xlo);
                        if (N2 - p != p) spec[N2 - p] = cmul(spec[N2 - p], xhi);
                    }
                }
                __syncthreads();
                stamp(5);
            }
        }
        // y[2m] = Re z[m], y[2m+1] = Im z[m], z = conj(FFT(conj Z)) / N2
        const double scale = 1.0 / (double)N2;
        const double wr = g.weights ? g.weights[r] : 1.0;
        double* y = g.Y + r * (int64_t)L;
        double nrm = 0.0;
        if (!g.linear) {
            for (int j = t; j < L; j += T) {
                const double2 z = buf[pad(j >> 1)];
                const double v = ((j & 1) ? -z.y : z.x) * scale * wr;
                y[j] = v;
                nrm = fma(v, v, nrm);
            }
        } else {
            for (int j = t; j < L; j += T) {
                double sacc = 0.0;
                for (int u = j; u < M; u += L) {
                    const double2 z = buf[pad(u >> 1)];
                    sacc += ((u & 1) ? -z.y : z.x) * scale;
                }
                const double v = sacc * wr;
                y[j] = v;
                nrm = fma(v, v, nrm);
            }
        }
        if (g.colnorm2) {
            for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
            if ((t & 31) == 0) atomicAdd(g.colnorm2 + r, nrm);
        }
        __syncthreads();
        stamp(6);
    }
}

int64_t* g_ts_tlog = nullptr;  // debug: per-phase timing of tensorsketch_kernel

struct TsPlan {
    int64_t M, N2;
    int linear;
    int threads;
    int ept;
    int spec_in_smem;
    size_t smem;
};

TsPlan plan_ts(int n_modes, int64_t L) {
    TsPlan p{};
    const bool pow2 = L >= 2 && (L & (L - 1)) == 0;
    if (pow2) {
        p.M = L;
        p.linear = 0;
    } else {
        const int64_t need = (int64_t)n_modes * (L - 1) + 1;
        p.M = 2;
        while (p.M < need) p.M <<= 1;
        p.linear = 1;
    }
    p.N2 = p.M / 2;
    p.ept = p.N2 >= 8192 ? 16 : 8;
    int64_t T = p.N2 / p.ept;
    if (T < 32) T = 32;
    p.threads = (int)T;
    const size_t fft_bytes = (size_t)(p.N2 + p.N2 / 8 + 1) * sizeof(double2);
    const size_t spec_bytes = (size_t)(p.N2 + 1) * sizeof(double2);
    const size_t stage_bytes = (size_t)kStage * (sizeof(double) + sizeof(int32_t));
    p.spec_in_smem = fft_bytes + spec_bytes + stage_bytes <= 200 * 1024;
    p.smem = fft_bytes + (p.spec_in_smem ? spec_bytes : 0) + stage_bytes;
    return p;
}

}  // namespace

// Debug hook: accumulate per-phase ns of tensorsketch_kernel (CTA 0) into
// `buf` (device int64[8]); NULL disables.
extern "C" void ids_debug_ts_timing(int64_t* buf) { g_ts_tlog = buf; }

extern "C" size_t ids_tensorsketch_workspace_bytes(int n_modes, const int64_t* dims,
                                                   int64_t ncols, int64_t out_dim) {
    (void)dims;
    (void)ncols;
    if (n_modes < 1 || out_dim < 1) return 256;
    const TsPlan p = plan_ts(n_modes, out_dim);
    return (size_t)p.M * sizeof(double2) + 148 * 2 * (size_t)(p.N2 + 1) * sizeof(double2) + 1024;
}

extern "C" int ids_tensorsketch_f64(int n_modes, const double* const* factors, const int64_t* dims,
                                    const int64_t* lds, int64_t ncols,
                                    const int32_t* const* order_signed,
                                    const int32_t* const* sorted_bucket, int64_t out_dim,
                                    const double* weights, double* Y, double* colnorm2,
                                    void* workspace, size_t ws_bytes, void* stream) {
    if (n_modes < 1 || n_modes > kMaxModes || ncols < 0 || out_dim < 1) {
        ids_set_last_error("tensorsketch: need 1..8 modes and out_dim >= 1");
        return IDS_EINVAL;
    }
    for (int n = 0; n < n_modes; ++n)
        if (dims[n] < 1 || lds[n] < dims[n]) {
            ids_set_last_error("tensorsketch: bad factor shape");
            return IDS_EINVAL;
        }
    const TsPlan p = plan_ts(n_modes, out_dim);
    if (p.N2 > kMaxHalf) {
        ids_set_last_error("tensorsketch: transform length above 16384 is not supported by this build");
        return IDS_EINVAL;
    }
    if (ncols == 0) return IDS_OK;
    cudaStream_t st = as_stream(stream);
    WsCarve ws(workspace, ws_bytes);
    double2* tw = ws.take<double2>(p.M);
    double2* specg = p.spec_in_smem ? nullptr : ws.take<double2>((size_t)148 * 2 * (p.N2 + 1));
    if (!ws.ok()) {
        ids_set_last_error("tensorsketch: workspace too small");
        return IDS_EWORKSPACE;
    }
    twiddle_kernel<<<(unsigned)tmin<int64_t>(ceil_div(p.M, 256), 256), 256, 0, st>>>(tw, p.M);
    IDS_LAUNCH_CHECK();
    TsArgs a{};
    a.n_modes = n_modes;
    for (int n = 0; n < n_modes; ++n) {
        a.factors[n] = factors[n];
        a.lds[n] = lds[n];
        a.order[n] = order_signed[n];
        a.keys[n] = sorted_bucket[n];
        a.dims[n] = dims[n];
    }
    a.ncols = ncols;
    a.L = out_dim;
    a.M = p.M;
    a.N2 = p.N2;
    a.linear = p.linear;
    a.weights = weights;
    a.Y = Y;
    a.colnorm2 = colnorm2;
    a.tw = tw;
    a.spec_glob = specg;
    a.spec_in_smem = p.spec_in_smem;
    a.tlog = g_ts_tlog;
    if (colnorm2) IDS_CUDA_TRY(cudaMemsetAsync(colnorm2, 0, sizeof(double) * ncols, st));
    auto kern = p.ept == 16 ? tensorsketch_kernel<16> : tensorsketch_kernel<8>;
    if (p.smem > 48 * 1024)
        IDS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)p.smem));
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, p.threads, p.smem);
    if (per_sm < 1) per_sm = 1;
    int64_t cap = (int64_t)sms * per_sm;
    if (!p.spec_in_smem) cap = tmin<int64_t>(cap, 148 * 2);
    const int64_t grid = tmin<int64_t>(ncols, cap);
    kern<<<(unsigned)grid, p.threads, p.smem, st>>>(a);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}
