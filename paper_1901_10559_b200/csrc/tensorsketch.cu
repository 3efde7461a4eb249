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
#include <limits.h>
#include <math.h>

#include "common.cuh"
#include "fft.cuh"

namespace {

using namespace ids_fft;

constexpr int kMaxModes = 8;
constexpr int kMaxHalf = 8192;  // largest half-length transform kept in shared memory
constexpr int kStageExt = 64;   // look-ahead entries staged past a stage's last head

// Per-mode scatter plan (ids_ts_mode_plan).  When a mode's rows spread over
// the buckets with few collisions (I_n < L at the tensor configs), its
// CountSketch is applied by reading the factor column CONTIGUOUSLY: each
// row's first-in-bucket entry (rank 0, in row order) is stored straight into
// the FFT buffer, later entries are parked in shared memory and added in
// rank order, one barrier per rank -- every bucket still sums its rows in
// increasing row order (scipy's), with no gathers from the factor column.
constexpr int kMaxPhase = 32;  // ranks beyond this: the gather path
constexpr int kScatterUnroll = 4;  // factor-column loads in flight per thread (8 measured no faster)
struct TsModePlanHdr {
    int32_t valid, maxr, nstash, pad;
    int32_t hist[64];
    int32_t cursor[64];
    int32_t off[kMaxPhase + 4];  // stash slots of rank r: [off[r], off[r + 1]), r >= 1 (+2 pad)
};
static_assert(sizeof(TsModePlanHdr) % 16 == 0, "plan header keeps the arrays aligned");

__host__ __device__ __forceinline__ int64_t ts_plan_stride(int64_t dim) { return (dim + 3) & ~int64_t(3); }
__host__ __device__ __forceinline__ int32_t* ts_plan_code(const TsModePlanHdr* h) {
    return reinterpret_cast<int32_t*>(const_cast<TsModePlanHdr*>(h) + 1);
}

// Bulk prefetch of [p, p + bytes) into L2 (TMA; 16-byte granules).
__device__ __forceinline__ void l2_prefetch(const void* p, size_t bytes) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
    for (uintptr_t a = a0; a < a1; a += 65536) {
        const uint32_t n = (uint32_t)(a1 - a < 65536 ? a1 - a : 65536);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(n) : "memory");
    }
}

__global__ void ts_plan_rank_kernel(const int32_t* __restrict__ order,
                                    const int32_t* __restrict__ keys,
                                    const int64_t* __restrict__ bstart, int64_t dim,
                                    TsModePlanHdr* hdr, int32_t* __restrict__ code,
                                    int32_t* __restrict__ rank) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < dim;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int32_t e = order[q], b = keys[q];
        const int32_t row = dec_row(e);
        const int32_t r = (int32_t)(q - bstart[b]);
        code[row] = e >= 0 ? b : ~b;
        rank[row] = r;
        if (r >= 1) atomicAdd(&hdr->hist[r < 63 ? r : 63], 1);
    }
}

__global__ void ts_plan_offsets_kernel(TsModePlanHdr* hdr) {
    if (threadIdx.x != 0) return;
    int maxr = 0;
    for (int r = 1; r < 64; ++r)
        if (hdr->hist[r] > 0) maxr = r;
    hdr->maxr = maxr;
    hdr->valid = maxr <= kMaxPhase && hdr->hist[63] == 0;
    int acc = 0;
    hdr->off[0] = 0;
    for (int r = 1; r <= kMaxPhase + 1; ++r) {
        hdr->off[r] = acc;
        if (r <= kMaxPhase) acc += hdr->hist[r];
    }
    hdr->nstash = acc;
}

__global__ void ts_plan_slot_kernel(TsModePlanHdr* hdr, int64_t dim,
                                    const int32_t* __restrict__ code, int32_t* __restrict__ slot,
                                    int32_t* __restrict__ stash_code) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < dim;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = slot[i];  // holds the rank on entry
        if (r == 0) {
            slot[i] = -1;
        } else if (r <= kMaxPhase) {
            // any order inside a rank: its entries hit distinct buckets
            const int32_t sl = hdr->off[r] + atomicAdd(&hdr->cursor[r], 1);
            slot[i] = sl;
            stash_code[sl] = code[i];
        } else {
            slot[i] = -2;  // plan invalid; never read
        }
    }
}

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
    int stage_cap;        // staged CountSketch entries (shared memory) per round
    int y_vec;            // Y 16-byte aligned: paired output stores
    int64_t* tlog;        // debug: per-phase ns accumulated by CTA 0 (NULL: off)
    const TsModePlanHdr* plan[kMaxModes];  // scatter plan of mode n, or NULL
};

__device__ __forceinline__ int64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return (int64_t)t;
}

// Shared-memory index padding against bank conflicts: one extra slot every
// 2^PS complex entries (PS = 3 for radix-8 passes, 4 for radix-16 passes).
template <int PS>
__device__ __forceinline__ int pad(int i) { return i + (i >> PS); }

// Staged entry q lives at sidx(q): within each 256-entry block the [thread][8]
// layout is transposed to [8][thread], so a warp's staging stores (8
// consecutive entries per thread) hit 32 distinct banks.
__device__ __forceinline__ int sidx(int q) { return (q & ~255) | ((q & 7) << 5) | ((q >> 3) & 31); }

__device__ __forceinline__ int fpad(int f) { return f + (f >> 3) + (f >> 6); }
constexpr int kFineSlots = 128 + 16 + 2;

// exp(-2 pi i m / M) from two small shared-memory tables:
// coarse[m >> 7] * fine[m & 127]  (M a power of two).  The fine table is
// padded (fpad) so that the strided index patterns of the passes hit
// distinct shared-memory banks.
struct Twiddle {
    const double2* coarse;
    const double2* fine;
    __device__ __forceinline__ double2 operator()(int m) const {
        return cmul(coarse[m >> 7], fine[fpad(m & 127)]);
    }
};

// One in-place Stockham pass of radix R over the N2-point buffer; every
// thread holds EPT >= N2 / blockDim.x points in registers across the barrier.
template <int R, int EPT, int PS>
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
            for (int r = 0; r < R; ++r) v[s][r] = buf[pad<PS>(j + r * B)];
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
            for (int r = 0; r < R; ++r) buf[pad<PS>(base + r * Ns)] = v[s][r];
        }
    }
    __syncthreads();
}

// The last Stockham pass (Ns * R == N2): butterfly j reads and writes the
// same slots j + r * Ns, so each completes on its own -- no barrier between
// loads and stores and one live butterfly per thread.
template <int R, int PS>
__device__ void stockham_last(double2* buf, int N2, int M, const Twiddle tw) {
    const int B = N2 / R, Ns = B;
    for (int j = threadIdx.x; j < B; j += blockDim.x) {
        double2 u[R];
#pragma unroll
        for (int r = 0; r < R; ++r) u[r] = buf[pad<PS>(j + r * B)];
        if (Ns > 1 && j != 0) {
            const double2 w1 = tw(j * (M / (Ns * R)));
            double2 w = w1;
#pragma unroll
            for (int r = 1; r < R; ++r) {
                u[r] = cmul(u[r], w);
                if (r + 1 < R) w = cmul(w, w1);
            }
        }
        dft<R>(u);
#pragma unroll
        for (int r = 0; r < R; ++r) buf[pad<PS>(j + r * B)] = u[r];
    }
    __syncthreads();
}

// One radix-16 Stockham pass, one butterfly per thread (N2 = 16 * blockDim.x).
// Twiddles w^r: w, w^2, w^4, w^8 from the tables, the rest as products.
__device__ void stockham_pass16(double2* buf, int N2, int Ns, int M, const Twiddle tw) {
    const int B = N2 / 16;
    const int j = threadIdx.x;
    double2 v[16];
    if (j < B) {
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = buf[pad<4>(j + r * B)];
        const int k = j % Ns;
        if (Ns > 1 && k != 0) {
            const int m1 = k * (M / (Ns * 16));
            const double2 w1 = tw(m1);
            const double2 w2 = cmul(w1, w1), w4 = cmul(w2, w2), w8 = cmul(w4, w4);
            v[1] = cmul(v[1], w1);
            v[2] = cmul(v[2], w2);
            v[4] = cmul(v[4], w4);
            v[8] = cmul(v[8], w8);
            const double2 w3 = cmul(w1, w2);
            v[3] = cmul(v[3], w3);
            v[5] = cmul(v[5], cmul(w1, w4));
            const double2 w6 = cmul(w2, w4);
            v[6] = cmul(v[6], w6);
            const double2 w7 = cmul(w3, w4);
            v[7] = cmul(v[7], w7);
            v[9] = cmul(v[9], cmul(w1, w8));
            v[10] = cmul(v[10], cmul(w2, w8));
            v[11] = cmul(v[11], cmul(w3, w8));
            v[12] = cmul(v[12], cmul(w4, w8));
            v[13] = cmul(v[13], cmul(cmul(w1, w4), w8));
            v[14] = cmul(v[14], cmul(w6, w8));
            v[15] = cmul(v[15], cmul(w7, w8));
        }
        dft16(v);
    }
    __syncthreads();
    if (j < B) {
        const int k = j % Ns;
        const int base = (j / Ns) * Ns * 16 + k;
#pragma unroll
        for (int r = 0; r < 16; ++r) buf[pad<4>(base + r * Ns)] = v[r];
    }
    __syncthreads();
}

// 8 points per thread: radix-8 passes (+ one radix-4/2).  16 points per thread
// (N2 = 8192, the longest transform): radix-16 passes in registers + radix-2.
// Every Stockham pass but the last; returns the stride Ns of the last pass
// (its radix is N2 / Ns).
template <int EPT>
__device__ __forceinline__ int fft_head(double2* buf, int N2, int M, const Twiddle tw) {
    constexpr int PS = EPT >= 16 ? 4 : 3;
    int Ns = 1;
    if constexpr (EPT >= 16) {
        while (Ns * 16 < N2) {
            stockham_pass16(buf, N2, Ns, M, tw);
            Ns *= 16;
        }
    } else {
        while (Ns * 8 < N2) {
            stockham_pass<8, EPT, PS>(buf, N2, Ns, M, tw);
            Ns *= 8;
        }
    }
    return Ns;
}

// One butterfly of the last (in-place) pass: outputs X[j + r * Ns].
template <int R, int PS>
__device__ __forceinline__ void last_butterfly(const double2* buf, int N2, int M, const Twiddle tw,
                                               int j, double2* u) {
    const int Ns = N2 / R;
#pragma unroll
    for (int r = 0; r < R; ++r) u[r] = buf[pad<PS>(j + r * Ns)];
    if (Ns > 1 && j != 0) {
        const double2 w1 = tw(j * (M / N2));
        double2 w = w1;
#pragma unroll
        for (int r = 1; r < R; ++r) {
            u[r] = cmul(u[r], w);
            if (r + 1 < R) w = cmul(w, w1);
        }
    }
    dft<R>(u);
}

// The last FFT pass fused with the real-spectrum untangle and the product
// into the running spectrum S.  Untangle pair (p, N2 - p) is complete in the
// butterflies j and Ns - j, so one thread takes both (no shared-memory round
// trip, no barrier); every slot it reads is cleared for the next mode.
template <int R, int PS>
__device__ void last_pass_untangle(double2* buf, int N2, int M, const Twiddle tw,
                                   double2* spec, bool first_mode) {
    const int Ns = N2 / R;
    // item i takes butterflies i and Ns - i (item 0: the self-paired 0 and Ns / 2)
    const int items = Ns > 1 ? Ns / 2 : 1;
    for (int i = threadIdx.x; i < items; i += blockDim.x) {
        const int j = i, j2 = i == 0 ? Ns / 2 : Ns - i;
        const bool two = j2 != j;
        double2 a[R], c[R];
        last_butterfly<R, PS>(buf, N2, M, tw, j, a);
        if (two) last_butterfly<R, PS>(buf, N2, M, tw, j2, c);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            buf[pad<PS>(j + r * Ns)] = make_double2(0.0, 0.0);
            if (two) buf[pad<PS>(j2 + r * Ns)] = make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // outputs of butterfly j (h = 0) and j2 (h = 1)
            if (h == 1 && !two) break;
            const int jj = h == 0 ? j : j2;
            const bool self = jj == 0 || 2 * jj == Ns;  // partner in the same butterfly
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int p = r * Ns + jj;
                if (p > N2 / 2) continue;  // the pair is handled from its lower index
                const double2 zk = h == 0 ? a[r] : c[r];
                double2 zm;
                if (jj == 0) zm = h == 0 ? a[(R - r) % R] : c[(R - r) % R];
                else if (self) zm = h == 0 ? a[R - r - 1] : c[R - r - 1];
                else zm = h == 0 ? c[R - r - 1] : a[R - r - 1];
                const double2 e = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
                const double2 d = make_double2(zk.x - zm.x, zk.y + zm.y);  // zk - conj(zm)
                const double2 o = make_double2(0.5 * d.y, -0.5 * d.x);   // d * (-i/2)
                const double2 wo = cmul(tw(p), o);
                const double2 xlo = cadd(e, wo);
                const double2 xhi = conj2(csub(e, wo));
                if (first_mode) {
                    spec[p] = xlo;
                    if (N2 - p != p) spec[N2 - p] = xhi;
                } else {
                    spec[p] = cmul(spec[p], xlo);
                    if (N2 - p != p) spec[N2 - p] = cmul(spec[N2 - p], xhi);
                }
            }
        }
    }
}

// Inverse transform: the last (radix-2) pass fused with the output.  Butterfly
// j yields z[j] and z[j + N2/2]; y[2m], y[2m+1] = Re z[m], -Im z[m] (scaled)
// leave as 16-byte streaming stores, and the slots are cleared for the next
// column.  Returns this thread's share of the column's squared norm.
template <int PS>
__device__ double last_pass_output(double2* buf, int N2, int M, const Twiddle tw, double2* y2,
                                   double scale, double wr) {
    const int Ns = N2 / 2;
    double nrm = 0.0;
    for (int j = threadIdx.x; j < Ns; j += blockDim.x) {
        double2 u[2];
        last_butterfly<2, PS>(buf, N2, M, tw, j, u);
        buf[pad<PS>(j)] = make_double2(0.0, 0.0);
        buf[pad<PS>(j + Ns)] = make_double2(0.0, 0.0);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const double v0 = u[h].x * scale * wr, v1 = -u[h].y * scale * wr;
            __stcs(y2 + j + h * Ns, make_double2(v0, v1));
            nrm = fma(v0, v0, nrm);
            nrm = fma(v1, v1, nrm);
        }
    }
    return nrm;
}

// Real-spectrum untangle of the finished transform, multiplied into S (each
// slot is read by exactly one pair and cleared for the next mode).
template <int PS>
__device__ void untangle_pairs(double2* buf, int N2, const Twiddle tw, double2* spec,
                               bool first_mode) {
    const int T = blockDim.x, npairs = N2 / 2 + 1;
    for (int p0 = threadIdx.x; p0 < npairs; p0 += 4 * T) {
        double2 sk[4], sm[4];
        if (!first_mode) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {  // independent spectrum loads first
                const int p = min(p0 + u * T, npairs - 1);
                sk[u] = spec[p];
                sm[u] = spec[N2 - p];
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int p = p0 + u * T;
            if (p >= npairs) break;
            const double2 zk = buf[pad<PS>(p % N2)];
            const double2 zm = buf[pad<PS>((N2 - p) % N2)];
            buf[pad<PS>(p % N2)] = make_double2(0.0, 0.0);
            buf[pad<PS>((N2 - p) % N2)] = make_double2(0.0, 0.0);
            const double2 e = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
            const double2 d = make_double2(zk.x - zm.x, zk.y + zm.y);  // zk - conj(zm)
            const double2 o = make_double2(0.5 * d.y, -0.5 * d.x);   // d * (-i/2)
            const double2 wo = cmul(tw(p), o);
            const double2 xlo = cadd(e, wo);
            const double2 xhi = conj2(csub(e, wo));
            if (first_mode) {
                spec[p] = xlo;
                if (N2 - p != p) spec[N2 - p] = xhi;
            } else {
                spec[p] = cmul(sk[u], xlo);
                if (N2 - p != p) spec[N2 - p] = cmul(sm[u], xhi);
            }
        }
    }
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
    constexpr int PS = EPT >= 16 ? 4 : 3;
    extern __shared__ double2 buf[];
    __shared__ double2 tw_coarse[kMaxHalf * 2 / 128 + 1];
    __shared__ double2 tw_fine[kFineSlots];
    __shared__ const double* s_fac[kMaxModes];
    __shared__ const int32_t* s_ord[kMaxModes];
    __shared__ const int32_t* s_key[kMaxModes];
    __shared__ int64_t s_ld[kMaxModes];
    __shared__ int s_dim[kMaxModes];
    __shared__ int32_t s_prevkey;
    __shared__ int s_pvalid[kMaxModes], s_pmaxr[kMaxModes];
    __shared__ int32_t s_poff[kMaxModes][kMaxPhase + 2];
    __shared__ double s_nrm[32];
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
            const TsModePlanHdr* h = q < g.n_modes ? g.plan[q] : nullptr;
            s_pvalid[q] = h && h->valid && h->nstash <= g.stage_cap;
            s_pmaxr[q] = h ? h->maxr : 0;
        }
    }
    for (int i = t; i < kMaxModes * (kMaxPhase + 2); i += T) {
        const int q = i / (kMaxPhase + 2), r = i % (kMaxPhase + 2);
        const TsModePlanHdr* h = q < g.n_modes ? g.plan[q] : nullptr;
        s_poff[q][r] = h ? h->off[r] : 0;
    }
    for (int m = t; m < 128; m += T) {
        double sn, cs;
        sincospi(2.0 * (double)m / (double)M, &sn, &cs);
        tw_fine[fpad(m)] = make_double2(cs, -sn);
    }
    for (int q = t; q * 128 < M; q += T) {
        double sn, cs;
        sincospi(2.0 * (double)q * 128.0 / (double)M, &sn, &cs);
        tw_coarse[q] = make_double2(cs, -sn);
    }
    __syncthreads();
    const Twiddle tw{tw_coarse, tw_fine};
    const int npairs = N2 / 2 + 1;  // pairs (p, N2 - p), p = 0..N2/2
    const int fft_slots = N2 + (N2 >> PS) + 1;
    // running spectrum S[0..N2]: after the padded FFT buffer in smem, or in
    // this CTA's global (L2-resident) slice
    double2* spec = g.spec_in_smem ? buf + fft_slots : g.spec_glob + (int64_t)blockIdx.x * (N2 + 1);
    double* st_val = reinterpret_cast<double*>(buf + fft_slots + (g.spec_in_smem ? (N2 + 1) : 0));
    int32_t* st_key = reinterpret_cast<int32_t*>(st_val + g.stage_cap);
    // heads resolved per stage; the rest of the staged block is look-ahead
    const int stage_heads = g.stage_cap - kStageExt;  // stage_cap == 8 * blockDim.x
    const bool tl = g.tlog && blockIdx.x == 0 && t == 0;
    int64_t tprev = tl ? gtimer() : 0;
    auto stamp = [&](int phase) {
        if (tl) {
            const int64_t tn = gtimer();
            g.tlog[phase] += tn - tprev;
            tprev = tn;
        }
    };
    bool out_done = false;  // the previous column's fused output cleared the buffer
    double out_nrm = 0.0;
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
                if (n == 0 && !out_done)  // else zeroed by the untangle / fused output
                    for (int l = t; l < N2; l += T) buf[pad<PS>(l)] = make_double2(0.0, 0.0);
                stamp(0);
                if (s_pvalid[n]) {
                    // scatter plan: the column is read contiguously; rank-0 rows
                    // store into the (zeroed) buffer, later rows are parked in
                    // the staging area and added rank by rank
                    const TsModePlanHdr* ph = g.plan[n];
                    const int32_t* pcode = ts_plan_code(ph);
                    const int32_t* pslot = pcode + ts_plan_stride(In);
                    if (t == 0) {  // the next (mode, column) factor column into L2
                        int nn = n + 1;
                        int64_t rn = r;
                        if (nn == g.n_modes) {
                            nn = 0;
                            rn = r + gridDim.x;
                        }
                        if (rn < g.ncols) l2_prefetch(s_fac[nn] + rn * s_ld[nn], (size_t)s_dim[nn] * 8);
                    }
                    __syncthreads();  // zeroing (n == 0) before the stores
                    for (int i0 = t; i0 < In; i0 += kScatterUnroll * T) {
                        double v[kScatterUnroll];
                        int32_t c[kScatterUnroll], sl[kScatterUnroll];
#pragma unroll
                        for (int u = 0; u < kScatterUnroll; ++u) {
                            const int i = min(i0 + u * T, In - 1);
                            v[u] = __ldcs(col + i);
                            c[u] = __ldg(pcode + i);
                            sl[u] = __ldg(pslot + i);
                        }
#pragma unroll
                        for (int u = 0; u < kScatterUnroll; ++u) {
                            if (i0 + u * T < In) {
                                const double sv = c[u] >= 0 ? v[u] : -v[u];
                                const int h = dec_row(c[u]);
                                if (sl[u] < 0) {
                                    dbuf[2 * pad<PS>(h >> 1) + (h & 1)] = 0.0 + sv;
                                } else {
                                    st_val[sl[u]] = sv;
                                    st_key[sl[u]] = h;
                                }
                            }
                        }
                    }
                    __syncthreads();
                    stamp(1);
                    for (int rr = 1; rr <= s_pmaxr[n]; ++rr) {
                        for (int q = s_poff[n][rr] + t; q < s_poff[n][rr + 1]; q += T) {
                            const int h = st_key[q];
                            dbuf[2 * pad<PS>(h >> 1) + (h & 1)] += st_val[q];
                        }
                        __syncthreads();
                    }
                    stamp(2);
                }
                for (int c0 = 0; c0 < In && !s_pvalid[n]; c0 += stage_heads) {
                    // stage entries [c0, c0 + ns): the heads below cn and a
                    // look-ahead; thread t owns the 8 consecutive entries
                    // [8t, 8t + 8) (one round: ns <= 8T), loaded with eight
                    // independent gathers in flight and kept in registers
                    const int cn = min(stage_heads, In - c0);
                    const int ns = min(In - c0, cn + kStageExt);
                    const int gb = 8 * t;
                    int32_t kq[8];
                    double x[8];
                    {
                        int32_t e[8];
                        const bool vec = ((reinterpret_cast<uintptr_t>(ord) |
                                           reinterpret_cast<uintptr_t>(key)) & 15) == 0;
                        if (vec && gb + 8 <= ns) {  // 2 x 16-byte loads per array (c0 % 4 == 0)
                            const int4* o4 = reinterpret_cast<const int4*>(ord + c0 + gb);
                            const int4* k4 = reinterpret_cast<const int4*>(key + c0 + gb);
                            const int4 oa = __ldg(o4), ob = __ldg(o4 + 1);
                            const int4 ka = __ldg(k4), kb = __ldg(k4 + 1);
                            e[0] = oa.x; e[1] = oa.y; e[2] = oa.z; e[3] = oa.w;
                            e[4] = ob.x; e[5] = ob.y; e[6] = ob.z; e[7] = ob.w;
                            kq[0] = ka.x; kq[1] = ka.y; kq[2] = ka.z; kq[3] = ka.w;
                            kq[4] = kb.x; kq[5] = kb.y; kq[6] = kb.z; kq[7] = kb.w;
                        } else {
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                const int qc = min(gb + u, ns - 1);
                                e[u] = __ldg(ord + c0 + qc);
                                kq[u] = __ldg(key + c0 + qc);
                            }
                        }
                        if (t == 0) s_prevkey = c0 > 0 ? __ldg(key + c0 - 1) : -1;
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const double v = __ldg(col + dec_row(e[u]));
                            x[u] = e[u] >= 0 ? v : -v;
                        }
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            if (gb + u < ns) {
                                st_key[sidx(gb + u)] = kq[u];
                                st_val[sidx(gb + u)] = x[u];
                            } else {
                                kq[u] = INT_MIN;  // past the staged block
                            }
                        }
                    }
                    __syncthreads();
                    stamp(1);
                    // runs of equal bucket: the thread holding a run's head sums it
                    // in increasing row order (its registers, then the following
                    // threads' entries from shared memory)
                    if (gb < cn) {
                        int32_t cur = gb > 0 ? st_key[sidx(gb - 1)] : s_prevkey;
                        bool own = false;
                        double acc = 0.0;
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            if (kq[u] != cur) {  // a run starts at gb + u
                                if (own) dbuf[2 * pad<PS>(cur >> 1) + (cur & 1)] = acc;
                                own = gb + u < cn && kq[u] != INT_MIN;
                                cur = kq[u];
                                acc = 0.0;
                            }
                            if (own) acc += x[u];
                        }
                        if (own) {  // the last run may continue past this thread
                            int q = gb + 8;
                            while (q < ns && st_key[sidx(q)] == cur) acc += st_val[sidx(q++)];
                            if (q == ns) {  // ... and past the look-ahead (rare)
                                for (int kg = c0 + q; kg < In && __ldg(key + kg) == cur; ++kg) {
                                    const int32_t e = __ldg(ord + kg);
                                    const double v = __ldg(col + dec_row(e));
                                    acc = e >= 0 ? acc + v : acc - v;
                                }
                            }
                            dbuf[2 * pad<PS>(cur >> 1) + (cur & 1)] = acc;
                        }
                    }
                    __syncthreads();
                    stamp(2);
                }
            } else {
                // ---- inverse: pack conj(Z) from S, forward FFT, conj ----
                for (int p0 = t; p0 < npairs; p0 += 4 * T) {
                    double2 xk[4], xm[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {  // independent spectrum loads first
                        const int p = min(p0 + u * T, npairs - 1);
                        xk[u] = spec[p];
                        xm[u] = spec[N2 - p];
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int p = p0 + u * T;
                        if (p >= npairs) break;
                        const double2 w = tw(p);
                        const double2 e = make_double2(0.5 * (xk[u].x + xm[u].x), 0.5 * (xk[u].y - xm[u].y));
                        const double2 d = make_double2(0.5 * (xk[u].x - xm[u].x), 0.5 * (xk[u].y + xm[u].y));
                        const double2 o = cmul(d, conj2(w));
                        // Z[p] = E + iO ; Z[N2-p] = conj(E) + i conj(O); stored conjugated
                        const double2 zlo = make_double2(e.x - o.y, e.y + o.x);
                        const double2 zhi = make_double2(e.x + o.y, -e.y + o.x);
                        if (p < N2) buf[pad<PS>(p)] = conj2(zlo);
                        const int pm = N2 - p;
                        if (pm != p && pm < N2 && pm > 0) buf[pad<PS>(pm)] = conj2(zhi);
                    }
                }
            }
            __syncthreads();
            stamp(3);
            // one call site for the FFT passes (all but the last)
            const int rem = N2 / fft_head<EPT>(buf, N2, M, tw);
            stamp(4);
            if (n < g.n_modes) {
                // ---- last pass + untangle + product into S, fused ----
                if constexpr (EPT >= 16) {  // N2 = 8192 = 16^3 * 2
                    last_pass_untangle<2, PS>(buf, N2, M, tw, spec, n == 0);
                } else {  // shorter transforms: plain last pass, then the untangle
                    if (rem == 2) stockham_last<2, PS>(buf, N2, M, tw);
                    else if (rem == 4) stockham_last<4, PS>(buf, N2, M, tw);
                    else if (rem == 8) stockham_last<8, PS>(buf, N2, M, tw);
                    else stockham_last<1, PS>(buf, N2, M, tw);
                    untangle_pairs<PS>(buf, N2, tw, spec, n == 0);
                }
                __syncthreads();
                stamp(5);
            } else {  // inverse: plain last pass, then the output below
                if constexpr (EPT >= 16) {
                    if (!g.linear && g.y_vec) {  // last pass fused with the output
                        out_nrm = last_pass_output<PS>(buf, N2, M, tw,
                                                       reinterpret_cast<double2*>(g.Y + r * (int64_t)L),
                                                       1.0 / (double)N2, g.weights ? g.weights[r] : 1.0);
                        out_done = true;
                    } else {
                        stockham_last<2, PS>(buf, N2, M, tw);
                    }
                } else {
                    if (rem == 2) stockham_last<2, PS>(buf, N2, M, tw);
                    else if (rem == 4) stockham_last<4, PS>(buf, N2, M, tw);
                    else if (rem == 8) stockham_last<8, PS>(buf, N2, M, tw);
                    else stockham_last<1, PS>(buf, N2, M, tw);
                }
            }
        }
        // y[2m] = Re z[m], y[2m+1] = Im z[m], z = conj(FFT(conj Z)) / N2
        const double scale = 1.0 / (double)N2;
        const double wr = g.weights ? g.weights[r] : 1.0;
        double* y = g.Y + r * (int64_t)L;
        double nrm = out_nrm;
        if (out_done) {
            // written by the fused last pass; the buffer is already clear
        } else if (!g.linear && g.y_vec) {
            // y[2m], y[2m+1] from z[m]: one 16-byte streaming store per pair
            // (L even, Y 16-byte aligned)
            double2* y2 = reinterpret_cast<double2*>(y);
            for (int mm = t; mm < L / 2; mm += T) {
                const double2 z = buf[pad<PS>(mm)];
                const double v0 = z.x * scale * wr, v1 = -z.y * scale * wr;
                __stcs(y2 + mm, make_double2(v0, v1));
                nrm = fma(v0, v0, nrm);
                nrm = fma(v1, v1, nrm);
            }
        } else if (!g.linear) {
            for (int j = t; j < L; j += T) {
                const double2 z = buf[pad<PS>(j >> 1)];
                const double v = ((j & 1) ? -z.y : z.x) * scale * wr;
                y[j] = v;
                nrm = fma(v, v, nrm);
            }
        } else {
            for (int j = t; j < L; j += T) {
                double sacc = 0.0;
                for (int u = j; u < M; u += L) {
                    const double2 z = buf[pad<PS>(u >> 1)];
                    sacc += ((u & 1) ? -z.y : z.x) * scale;
                }
                const double v = sacc * wr;
                y[j] = v;
                nrm = fma(v, v, nrm);
            }
        }
        if (g.colnorm2) {  // fixed-order block reduction: run-to-run identical
            for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
            if ((t & 31) == 0) s_nrm[t >> 5] = nrm;
            __syncthreads();
            if (t == 0) {
                double acc = 0.0;
                for (int w = 0; w < (T >> 5); ++w) acc += s_nrm[w];
                g.colnorm2[r] = acc;
            }
        }
        out_nrm = 0.0;
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
    int stage_cap;
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
    const int ps = p.ept >= 16 ? 4 : 3;  // padding shift of the FFT buffer (pad<PS>)
    const size_t fft_bytes = (size_t)(p.N2 + (p.N2 >> ps) + 1) * sizeof(double2);
    const size_t spec_bytes = (size_t)(p.N2 + 1) * sizeof(double2);
    p.stage_cap = 8 * p.threads;  // one staging round: 8 consecutive entries per thread
    const size_t stage_bytes = (size_t)p.stage_cap * (sizeof(double) + sizeof(int32_t));
    p.spec_in_smem = fft_bytes + spec_bytes + stage_bytes <= 200 * 1024;
    p.smem = fft_bytes + (p.spec_in_smem ? spec_bytes : 0) + stage_bytes;
    return p;
}

}  // namespace

// Debug hook: accumulate per-phase ns of tensorsketch_kernel (CTA 0) into
// `buf` (device int64[8]); NULL disables.
extern "C" void ids_debug_ts_timing(int64_t* buf) { g_ts_tlog = buf; }

extern "C" int ids_tensorsketch_fused_ok(int n_modes, int64_t out_dim) {
    if (n_modes < 1 || n_modes > kMaxModes || out_dim < 1) return 0;
    return plan_ts(n_modes, out_dim).N2 <= kMaxHalf ? 1 : 0;
}

extern "C" size_t ids_tensorsketch_workspace_bytes(int n_modes, const int64_t* dims,
                                                   int64_t ncols, int64_t out_dim) {
    (void)dims;
    (void)ncols;
    if (n_modes < 1 || out_dim < 1) return 256;
    const TsPlan p = plan_ts(n_modes, out_dim);
    return (size_t)p.M * sizeof(double2) +
           (size_t)ids_sm_count() * 2 * (size_t)(p.N2 + 1) * sizeof(double2) + 1024;
}

extern "C" size_t ids_ts_mode_plan_bytes(int64_t dim) {
    if (dim < 1) return 0;
    return sizeof(TsModePlanHdr) + 3 * (size_t)ts_plan_stride(dim) * sizeof(int32_t);
}

extern "C" int ids_ts_mode_plan(const int32_t* order_signed, const int32_t* sorted_bucket,
                                const int64_t* bstart, int64_t dim, int64_t out_dim, void* plan,
                                size_t plan_bytes, void* stream) {
    if (dim < 1 || out_dim < 1 || dim > 0x7fffffffLL || !plan ||
        plan_bytes < ids_ts_mode_plan_bytes(dim) || (reinterpret_cast<uintptr_t>(plan) & 15)) {
        ids_set_last_error("ts mode plan: bad arguments");
        return IDS_EINVAL;
    }
    cudaStream_t st = as_stream(stream);
    TsModePlanHdr* hdr = static_cast<TsModePlanHdr*>(plan);
    int32_t* code = ts_plan_code(hdr);
    int32_t* slot = code + ts_plan_stride(dim);
    int32_t* stash = slot + ts_plan_stride(dim);
    IDS_CUDA_TRY(cudaMemsetAsync(hdr, 0, sizeof(TsModePlanHdr), st));
    const unsigned g = (unsigned)tmin<int64_t>(ceil_div(dim, 256), 148 * 8);
    ts_plan_rank_kernel<<<g, 256, 0, st>>>(order_signed, sorted_bucket, bstart, dim, hdr, code, slot);
    IDS_LAUNCH_CHECK();
    ts_plan_offsets_kernel<<<1, 32, 0, st>>>(hdr);
    IDS_LAUNCH_CHECK();
    ts_plan_slot_kernel<<<g, 256, 0, st>>>(hdr, dim, code, slot, stash);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}

extern "C" int ids_tensorsketch_f64(int n_modes, const double* const* factors, const int64_t* dims,
                                    const int64_t* lds, int64_t ncols,
                                    const int32_t* const* order_signed,
                                    const int32_t* const* sorted_bucket, int64_t out_dim,
                                    const double* weights, double* Y, double* colnorm2,
                                    void* workspace, size_t ws_bytes, void* stream) {
    return ids_tensorsketch_planned_f64(n_modes, factors, dims, lds, ncols, order_signed,
                                        sorted_bucket, nullptr, out_dim, weights, Y, colnorm2,
                                        workspace, ws_bytes, stream);
}

extern "C" int ids_tensorsketch_planned_f64(int n_modes, const double* const* factors,
                                            const int64_t* dims, const int64_t* lds,
                                            int64_t ncols, const int32_t* const* order_signed,
                                            const int32_t* const* sorted_bucket,
                                            const void* const* plans, int64_t out_dim,
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
    // one running-spectrum slice per resident CTA (at most two per SM)
    double2* specg = p.spec_in_smem ? nullptr
                                    : ws.take<double2>((size_t)ids_sm_count() * 2 * (p.N2 + 1));
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
        a.plan[n] = plans ? static_cast<const TsModePlanHdr*>(plans[n]) : nullptr;
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
    a.stage_cap = p.stage_cap;
    a.y_vec = (reinterpret_cast<uintptr_t>(Y) & 15) == 0 && out_dim % 2 == 0;
    a.tlog = g_ts_tlog;
    auto kern = p.ept == 16 ? tensorsketch_kernel<16> : tensorsketch_kernel<8>;
    if (p.smem > 40 * 1024)
        IDS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)p.smem));
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, p.threads, p.smem);
    if (per_sm < 1) per_sm = 1;
    int64_t cap = (int64_t)sms * per_sm;
    if (!p.spec_in_smem) cap = tmin<int64_t>(cap, (int64_t)ids_sm_count() * 2);
    const int64_t grid = tmin<int64_t>(ncols, cap);
    kern<<<(unsigned)grid, p.threads, p.smem, st>>>(a);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}
