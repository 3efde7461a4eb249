// Split-spectrum TensorSketch kernel (sm_100a).  Replaces reference
// sketch.py:156-186 for power-of-two sketch lengths L in {4096, 8192, 16384}
// (C4: L = 4096, C5: L = 16384):
//   Y[:, r] = irfft_L( prod_n rfft_L( S_n A_n[:, r] ) ) * weights[r].
//
// Layout of the work.  The length-L real transform is the packed half-length
// complex transform Z = FFT_{N2}(z), z[m] = c[2m] + i c[2m+1], N2 = L / 2.
// Its first radix-2 decimation-in-frequency stage splits it into two
// independent H-point transforms (H = N2 / 2):
//   Z[2k]   = FFT_H( z[m] + z[m + H] )[k]
//   Z[2k+1] = FFT_H( (z[m] - z[m + H]) W_{N2}^m )[k],
// and z[m] +- z[m + H] is itself a CountSketch: bucket b folds onto slot
// b mod N2 with sign -1 for b >= N2 in the odd half.  So a CLUSTER OF TWO
// CTAs owns one term column r: CTA h (h = cluster rank) CountSketches the
// factor column straight into its folded half (no exchange), runs the
// H-point FFT, untangles the real spectrum at the bins p = 2k + h (the
// untangle pair p, N2 - p has the same parity: it never leaves the CTA) and
// multiplies it into its half of the running spectrum, which lives in TENSOR
// MEMORY (tcgen05.st / tcgen05.ld, 64 KB per CTA at C5) -- not in shared
// memory, registers or L2.  The two halves meet once per column, in the
// inverse: each CTA transforms its half (E or O), and one exchange of H/2
// points per CTA through distributed shared memory combines
//   z[m] = E[m] + W_{N2}^{-m} O[m],   z[m + H] = E[m] - W_{N2}^{-m} O[m].
// Half-size transforms let two CTAs share an SM (106 KB of shared memory and
// 128 KB of TMEM each at C5), so one CTA's scatter overlaps the other's FFT.
//
// CountSketch order.  A per-mode plan (ids_ts_split_plan) cuts the rows into
// one chunk (the whole column) when the later rows of its slots fit the tail
// buffer, else into 16 T-row chunks, and gives every row its slot's buffer
// index, its signs in the two halves and -- unless it is the first row of
// its slot in the chunk -- its position in the chunk's tail buffer; per
// chunk, the tail groups (slots with later rows).  Rows are loaded coalesced
// in rounds of 8 T (two rounds in flight); first rows store (chunk 0) or add
// into their slots -- distinct slots, no conflicts -- later rows park in the
// tail buffer, and after one barrier one thread per group adds them in row
// order.  Run-to-run identical.  (The fold adds the rows of buckets b and
// b + N2 in row order, so the sums differ from the reference's per-bucket
// ones in rounding only: Y agrees to ~1e-15 relative; the FFTs differ from
// pocketfft at that level anyway.)
//
// Twiddles: one table lookup per thread and stage (coarse x fine tables of
// W_L in shared memory); the per-point factors are products of that base
// with compile-time constants W_32^r, because every index a thread touches
// is j + (H/16) r.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "fft.cuh"

namespace {

using namespace ids_fft;

constexpr int kMaxModes = 8;
constexpr int kRows = 8;        // rows per thread per load round (a round = 8 T rows)
constexpr int kChunkRounds = 2; // fixed chunks (long or collision-heavy modes): 16 T rows
constexpr int kTailPerThread = 18;  // tail buffer: 18 T doubles (later rows of a slot)
constexpr int kGroupsReg = 12;  // tail groups per thread whose descriptors are prefetched
constexpr int kSingleMax = 12288;  // modes up to this length are planned by one CTA
// per-row plan code: bits 0-13 the slot's double index in the padded FFT
// buffer, bit 14 / 15 the row's sign in the even / odd half (sign(b), and
// sign(b) * (b >= N2 ? -1 : 1)), bits 16-31 its tail position (kFirst: the
// first row of its slot in the chunk)
constexpr uint32_t kIdxMask = 0x3FFFu;
constexpr int kSignShift = 14;
constexpr int kTailShift = 16;
constexpr uint32_t kFirst = 0xFFFFu;
constexpr uint32_t kPadIdx = 32;  // a padding word of the buffer (never read): rows past the end
constexpr int kFine = 128;
constexpr int kFineSlots = kFine + kFine / 8 + 2;

__host__ __device__ __forceinline__ int64_t split_stride(int64_t dim) { return (dim + 3) & ~int64_t(3); }

// exp(-2 pi i r / 32), r in [0, 16)
__device__ __forceinline__ double2 w32(int r) {
    constexpr double c1 = 0.98078528040323044912618, s1 = 0.19509032201612826784828;
    constexpr double c2 = 0.92387953251128675612818, s2 = 0.38268343236508977172846;
    constexpr double c3 = 0.83146961230254523707879, s3 = 0.55557023301960222474283;
    constexpr double hh = 0.70710678118654752440084;
    constexpr double kc[16] = {1.0, c1, c2, c3, hh, s3, s2, s1, 0.0, -s1, -s2, -s3, -hh, -c3, -c2, -c1};
    constexpr double ks[16] = {0.0, s1, s2, s3, hh, c3, c2, c1, 1.0, c1, c2, c3, hh, s3, s2, s1};
    return make_double2(kc[r], -ks[r]);
}

__device__ __forceinline__ int spad(int i) { return i + (i >> 4); }
__device__ __forceinline__ int fpad(int f) { return f + (f >> 3) + (f >> 6); }

// W_M^m = coarse[m >> 7] * fine[m & 127] (M = L, a power of two)
struct TwM {
    const double2* coarse;
    const double2* fine;
    __device__ __forceinline__ double2 operator()(int m) const {
        return cmul(coarse[m >> 7], fine[fpad(m & (kFine - 1))]);
    }
};

__device__ __forceinline__ double2 shfl16(double2 v) {
    return make_double2(__shfl_xor_sync(0xffffffffu, v.x, 16), __shfl_xor_sync(0xffffffffu, v.y, 16));
}

// v[r] *= w1^r, r = 1..15
__device__ __forceinline__ void twiddle16(double2* v, double2 w1) {
    const double2 w2 = cmul(w1, w1), w4 = cmul(w2, w2), w8 = cmul(w4, w4);
    const double2 w3 = cmul(w1, w2), w5 = cmul(w1, w4), w6 = cmul(w2, w4), w7 = cmul(w3, w4);
    v[1] = cmul(v[1], w1);
    v[2] = cmul(v[2], w2);
    v[3] = cmul(v[3], w3);
    v[4] = cmul(v[4], w4);
    v[5] = cmul(v[5], w5);
    v[6] = cmul(v[6], w6);
    v[7] = cmul(v[7], w7);
    v[8] = cmul(v[8], w8);
    v[9] = cmul(v[9], cmul(w1, w8));
    v[10] = cmul(v[10], cmul(w2, w8));
    v[11] = cmul(v[11], cmul(w3, w8));
    v[12] = cmul(v[12], cmul(w4, w8));
    v[13] = cmul(v[13], cmul(w5, w8));
    v[14] = cmul(v[14], cmul(w6, w8));
    v[15] = cmul(v[15], cmul(w7, w8));
}

// ---- tensor memory --------------------------------------------------------
// one complex per thread (4 columns of its lane): two loads, one wait
__device__ __forceinline__ void tm_ld2(uint32_t ta, uint32_t tb, double2& a, double2& b) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(ta)
                 : "memory");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tb)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    a = make_double2(__hiloint2double((int)r[1], (int)r[0]), __hiloint2double((int)r[3], (int)r[2]));
    b = make_double2(__hiloint2double((int)r[5], (int)r[4]), __hiloint2double((int)r[7], (int)r[6]));
}
__device__ __forceinline__ void tm_st1(uint32_t ta, double2 v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ta),
                 "r"(__double2loint(v.x)), "r"(__double2hiint(v.x)), "r"(__double2loint(v.y)),
                 "r"(__double2hiint(v.y))
                 : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---- cluster ----------------------------------------------------------------
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t peer_addr(const void* local, uint32_t rank) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(local);
    uint32_t out;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(a), "r"(rank));
    return out;
}
__device__ __forceinline__ void st_peer(uint32_t addr, double2 v) {
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void st_peer1(uint32_t addr, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}

__device__ __forceinline__ void l2_prefetch(const void* p, size_t bytes) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
    for (uintptr_t a = a0; a < a1; a += 65536) {
        const uint32_t n = (uint32_t)(a1 - a < 65536 ? a1 - a : 65536);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(n) : "memory");
    }
}

// ---- FFT passes over the H-point half transform -----------------------------
// Stockham pass of radix R at stride Ns (in place, two barriers).  The first
// pass (Ns = 1) optionally applies the odd half's pre-twiddle W_{N2}^m on load.
template <int H, int R, bool FIRST>
__device__ __forceinline__ void split_pass(double2* buf, int Ns, const TwM& tw, bool pretw) {
    constexpr int T = H / 16, B = H / R, S = 16 / R, M = 4 * H;
    const int t = threadIdx.x;
    double2 v[S][R];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int b = t + s * T;
#pragma unroll
        for (int r = 0; r < R; ++r) v[s][r] = buf[spad(b + r * B)];
        if (FIRST) {
            if (pretw) {  // m = b + r B: W_{N2}^m = W_M^{2b} * W_{2R}^r
                const double2 base = tw(2 * b);
                v[s][0] = cmul(v[s][0], base);
#pragma unroll
                for (int r = 1; r < R; ++r) v[s][r] = cmul(v[s][r], cmul(base, w32(r * (16 / R))));
            }
        } else {
            static_assert(FIRST || R == 16, "twiddled passes are radix 16");
            const int k = b & (Ns - 1);
            if (k != 0) twiddle16(v[s], tw(k * (M / (Ns * 16))));
        }
        dft<R>(v[s]);
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int b = t + s * T;
        const int k = b & (Ns - 1);
        const int base = (b - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) buf[spad(base + r * Ns)] = v[s][r];
    }
    __syncthreads();
}

// Last pass (radix 16, Ns = T): butterfly j reads and finishes the slots
// j + T r in place; outputs X[j + T r] in v.
template <int H>
__device__ __forceinline__ void last_pass(double2* buf, int j, const TwM& tw, double2* v, bool zero) {
    constexpr int T = H / 16;
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = buf[spad(j + r * T)];
    if (zero) {
#pragma unroll
        for (int r = 0; r < 16; ++r) buf[spad(j + r * T)] = make_double2(0.0, 0.0);
    }
    if (j != 0) twiddle16(v, tw(4 * j));  // W_H^j = W_M^{4j}
    dft16(v);
}

// Real-spectrum untangle of bin p from Z[p] = zk and Z[N2 - p] = zm.
__device__ __forceinline__ double2 untangle1(double2 zk, double2 zm, double2 w) {
    const double2 e = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
    const double2 d = make_double2(zk.x - zm.x, zk.y + zm.y);
    const double2 o = make_double2(0.5 * d.y, -0.5 * d.x);
    return cadd(e, cmul(w, o));
}
// Inverse packing: conj(Z'[p]) from the spectrum bins S[p] = xk, S[N2 - p] = xm.
__device__ __forceinline__ double2 pack1(double2 xk, double2 xm, double2 w) {
    const double2 e = make_double2(0.5 * (xk.x + xm.x), 0.5 * (xk.y - xm.y));
    const double2 d = make_double2(0.5 * (xk.x - xm.x), 0.5 * (xk.y + xm.y));
    const double2 o = cmul(d, conj2(w));
    return make_double2(e.x - o.y, -(e.y + o.x));
}

struct SplitArgs {
    int n_modes;
    const double* factors[kMaxModes];
    int64_t lds[kMaxModes];
    const int32_t* hdr[kMaxModes];     // per mode: plan header (rows per chunk)
    const uint32_t* code[kMaxModes];   // per mode: per-row code (slot, signs, tail position)
    const uint2* groups[kMaxModes];    // per mode and chunk: tail groups (slot | start << 16, len)
    const int32_t* ngroups[kMaxModes]; // per mode: tail groups per chunk
    int dims[kMaxModes];
    int64_t ncols;
    const double* weights;
    double* Y;
    double* colnorm2;
    int tmem_cols;
    int64_t* tlog;  // debug: per-phase ns accumulated by CTA 0, thread 0 (NULL: off)
};

__device__ __forceinline__ int64_t gtimer() {
    uint64_t v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return (int64_t)v;
}

template <int H>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(H / 16, (H >= 4096 ? 2 : (H == 2048 ? 4 : 8)))
    ts_split_kernel(SplitArgs g) {
    constexpr int T = H / 16, M = 4 * H, R1 = H / 256;
    constexpr int RS = T * kRows;  // rows per load round
    extern __shared__ double2 smem[];
    double2* buf = smem;                                // H + H/16 + 1 padded points
    double2* coarse = buf + (H + H / 16 + 1);           // M / 128
    double2* fine = coarse + M / kFine;                 // kFineSlots
    double* tail = reinterpret_cast<double*>(fine + kFineSlots);  // 18 T values: later rows of a slot
    __shared__ double2 s_stash[32];                     // lane 0 / warp 0 mirrors (bin j = 0)
    __shared__ double s_n2, s_n2f;                      // running / final spectrum at bin N2 (real)
    __shared__ double s_red[T / 32];
    __shared__ double s_peer_nrm;
    __shared__ uint32_t s_taddr;
    // per-mode parameters in shared memory: indexing the kernel parameters
    // with a runtime mode would copy them to local memory
    __shared__ const double* s_fac[kMaxModes];
    __shared__ const uint32_t* s_code[kMaxModes];
    __shared__ const uint2* s_grp[kMaxModes];
    __shared__ const int32_t* s_ngr[kMaxModes];
    __shared__ int64_t s_ld[kMaxModes];
    __shared__ int s_dim[kMaxModes], s_cs[kMaxModes];
    double* dbuf = reinterpret_cast<double*>(buf);
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const uint32_t h = cluster_rank();
    const bool odd = h != 0;
    const int cid = (int)(blockIdx.x >> 1), ncl = (int)(gridDim.x >> 1);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&s_taddr)),
                     "r"(g.tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    for (int i = t; i < H + H / 16 + 1; i += T) buf[i] = make_double2(0.0, 0.0);
    for (int f = t; f < kFine; f += T) {
        double sn, cs;
        sincospi(2.0 * (double)f / (double)M, &sn, &cs);
        fine[fpad(f)] = make_double2(cs, -sn);
    }
    for (int q = t; q < M / kFine; q += T) {
        double sn, cs;
        sincospi(2.0 * (double)(q * kFine) / (double)M, &sn, &cs);
        coarse[q] = make_double2(cs, -sn);
    }
    if (t == 0) {
#pragma unroll
        for (int q = 0; q < kMaxModes; ++q) {  // static indexing of g
            const bool on = q < g.n_modes;
            s_fac[q] = g.factors[q];
            s_code[q] = g.code[q];
            s_grp[q] = g.groups[q];
            s_ngr[q] = g.ngroups[q];
            s_ld[q] = g.lds[q];
            s_dim[q] = g.dims[q];
            s_cs[q] = on ? __ldg(g.hdr[q]) : 1;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = s_taddr + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 64);
    const TwM tw{coarse, fine};

    // last-pass butterfly of this thread: lanes l and l ^ 16 hold the
    // butterflies whose untangle partners they are (j <-> T - j even half,
    // j <-> T - 1 - j odd half); warp 0's lanes 0 / 16 hold the self-paired
    // j = 0 and j = T / 2 of the even half.
    const int u16 = 16 * warp + (lane & 15);
    const int jl = lane < 16 ? u16 : (odd ? T - 1 - u16 : (u16 == 0 ? T / 2 : T - u16));
    const bool self0 = !odd && warp == 0 && lane == 0;   // j = 0: mirror r <-> -r mod 16
    const bool selfh = !odd && warp == 0 && lane == 16;  // j = T/2: mirror r <-> 15 - r, own
    const uint32_t peer = h ^ 1u;
#ifdef IDS_TS_SPLIT_TIMING  // debug: per-phase time of CTA 0, thread 0
    const bool tl = g.tlog && blockIdx.x == 0 && t == 0;
    int64_t tprev = tl ? gtimer() : 0;
    auto stamp = [&](int ph) {
        if (tl) {
            const int64_t tn = gtimer();
            g.tlog[ph] += tn - tprev;
            tprev = tn;
        }
    };
#else
    auto stamp = [](int) {};
#endif

    for (int r = cid; r < (int)g.ncols; r += ncl) {
        const double wr = g.weights ? g.weights[r] : 1.0;
        for (int n = 0; n < g.n_modes; ++n) {
            // ---- folded CountSketch of column r of mode n ----
            // Chunk by chunk (16 T rows): coalesced loads; the first row of
            // each slot in the chunk adds straight into the buffer (distinct
            // slots: no conflicts), later rows park in the tail buffer; then
            // one thread per slot with later rows adds them in row order.
            const int I = s_dim[n];
            const double* col = s_fac[n] + r * s_ld[n];
            const uint32_t* code = s_code[n];
            {
            // Chunk by chunk (the whole column when its later rows fit the
            // tail buffer): coalesced loads in rounds of 8 T rows, two rounds
            // in flight; the first row of each slot in the chunk stores (chunk
            // 0: the slot is still zero) or adds into the buffer -- distinct
            // slots, no conflicts -- later rows park in the tail buffer; then
            // one thread per slot with later rows adds them in row order.
            const int cs = s_cs[n];
            struct RowSet {
                double v[kRows];
                uint32_t k[kRows];
            } A, B;
            // 16-byte loads (rows 2 (t + u T) + {0, 1}) when the column and the
            // plan codes are 8 / 16-byte aligned at even rows
            const bool vec = ((reinterpret_cast<uintptr_t>(col) & 15) | (reinterpret_cast<uintptr_t>(code) & 7)) == 0;
            auto ld = [&](RowSet& S, int r0, int cend) {
                if (vec && (r0 & 1) == 0) {
#pragma unroll
                    for (int u = 0; u < kRows / 2; ++u) {
                        const int i = r0 + 2 * (u * T + t);
                        if (i + 1 < cend) {
                            const double2 v2 = __ldg(reinterpret_cast<const double2*>(col + i));
                            const uint2 k2 = __ldg(reinterpret_cast<const uint2*>(code + i));
                            S.v[2 * u] = v2.x;
                            S.v[2 * u + 1] = v2.y;
                            S.k[2 * u] = k2.x;
                            S.k[2 * u + 1] = k2.y;
                        } else {
                            S.v[2 * u] = i < cend ? __ldg(col + i) : 0.0;
                            S.k[2 * u] = i < cend ? __ldg(code + i) : (kFirst << kTailShift) | kPadIdx;
                            S.v[2 * u + 1] = 0.0;
                            S.k[2 * u + 1] = (kFirst << kTailShift) | kPadIdx;
                        }
                    }
                    return;
                }
#pragma unroll
                for (int u = 0; u < kRows; ++u) {
                    const int i = r0 + u * T + t;
                    S.v[u] = i < cend ? __ldg(col + i) : 0.0;
                    S.k[u] = i < cend ? __ldg(code + i) : (kFirst << kTailShift) | kPadIdx;
                }
            };
            auto proc = [&](RowSet& S, bool add) {
                double old[kRows];
#pragma unroll
                for (int u = 0; u < kRows; ++u) {  // signed values; the first rows' slots
                    const uint64_t sb = (uint64_t)((S.k[u] >> (kSignShift + (int)h)) & 1u) << 63;
                    S.v[u] = __longlong_as_double(__double_as_longlong(S.v[u]) ^ (long long)sb);
                    old[u] = add && (S.k[u] >> kTailShift) == kFirst ? dbuf[S.k[u] & kIdxMask] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < kRows; ++u) {
                    if ((S.k[u] >> kTailShift) == kFirst) dbuf[S.k[u] & kIdxMask] = add ? old[u] + S.v[u] : S.v[u];
                    else tail[S.k[u] >> kTailShift] = S.v[u];
                }
            };
            for (int c = 0; c * cs < I; ++c) {
                const int c0 = c * cs, cend = min(I, c0 + cs);
                const int ng = __ldg(s_ngr[n] + c);
                const uint2* grp = s_grp[n] + (int64_t)c * (cs / 2);
                stamp(0);
                ld(A, c0, cend);
                for (int r0 = c0; r0 < cend; r0 += 2 * RS) {
                    if (r0 + RS < cend) ld(B, r0 + RS, cend);
                    proc(A, c > 0);
                    if (r0 + RS < cend) {
                        if (r0 + 2 * RS < cend) ld(A, r0 + 2 * RS, cend);
                        proc(B, c > 0);
                    }
                }
                uint2 gd[kGroupsReg];
#pragma unroll
                for (int q = 0; q < kGroupsReg; ++q) gd[q] = t + q * T < ng ? __ldg(grp + t + q * T) : make_uint2(kPadIdx, 0u);
                stamp(8);
                __syncthreads();
                stamp(9);
                // later rows, one slot per group, in row order (4 groups at a
                // time; the first four rows of every group loaded up front --
                // longer groups are rare: P(len > 4) ~ 1% at C5)
#pragma unroll
                for (int q0 = 0; q0 < kGroupsReg; q0 += 4) {
                    double gs[4], go[4];
                    double x[4][4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint2 d = gd[q0 + q];
                        const int st0 = (int)(d.x >> 16), len = (int)d.y;
#pragma unroll
                        for (int e = 0; e < 4; ++e) x[q][e] = e < len ? tail[st0 + e] : 0.0;
                        go[q] = dbuf[d.x & kIdxMask];
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint2 d = gd[q0 + q];
                        const int len = (int)d.y;
                        double acc = x[q][0];
                        if (len > 1) acc += x[q][1];
                        if (len > 2) acc += x[q][2];
                        if (len > 3) acc += x[q][3];
                        gs[q] = acc;
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint2 d = gd[q0 + q];
                        const int st0 = (int)(d.x >> 16), len = (int)d.y;
                        if (len > 4)
                            for (int e = 4; e < len; ++e) gs[q] += tail[st0 + e];
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) dbuf[gd[q0 + q].x & kIdxMask] = go[q] + gs[q];
                }
                for (int q = t + kGroupsReg * T; q < ng; q += T) {  // tail-heavy chunks
                    const uint2 d = __ldg(grp + q);
                    const int st0 = (int)(d.x >> 16);
                    double acc = tail[st0];
                    for (int e = 1; e < (int)d.y; ++e) acc += tail[st0 + e];
                    dbuf[d.x & kIdxMask] += acc;
                }
                __syncthreads();  // chunk c's sums before chunk c + 1's first rows; tail free
                stamp(1);
            }
            }
            if (!odd && t == 0) {  // the next factor column this cluster reads, into L2
                int nn = n + 1;
                int64_t rn = r;
                if (nn == g.n_modes) {
                    nn = 0;
                    rn = r + ncl;
                }
                if (rn < g.ncols) l2_prefetch(s_fac[nn] + rn * s_ld[nn], (size_t)s_dim[nn] * 8);
            }
            // ---- H-point FFT of the folded half ----
            split_pass<H, R1, true>(buf, 1, tw, odd);
            split_pass<H, 16, false>(buf, R1, tw, false);
            stamp(2);
            const bool last = n + 1 == g.n_modes;
            double2 v[16];
            last_pass<H>(buf, jl, tw, v, !last);
            // ---- untangle X[p], p = 2 (jl + T r) + h (partner values by shuffle),
            // product into the running spectrum in TMEM, and after the last mode
            // the packing of conj(Z') for the inverse -- one pair (a, 15 - a) at
            // a time: the pair's partners sit at the same pair in lane l ^ 16 ----
            const double2 wb = tw(2 * jl + (int)h);
            if (self0) {
#pragma unroll
                for (int q = 0; q < 16; ++q) s_stash[q] = v[q];
            }
            __syncwarp();
#pragma unroll
            for (int a = 0; a < 8; ++a) {
                const int q = 15 - a;
                double2 ma = shfl16(v[q]), mq = shfl16(v[a]);
                if (selfh) {
                    ma = v[q];
                    mq = v[a];
                }
                if (self0) {
                    ma = s_stash[(16 - a) & 15];
                    mq = s_stash[(16 - q) & 15];
                }
                if (a == 0 && self0) {  // bin N2 = conj(e - o) of the pair (0, N2): real
                    const double x = v[0].x - v[0].y;
                    s_n2f = n == 0 ? x : s_n2 * x;
                    if (!last) s_n2 = s_n2f;
                }
                const double2 wa = cmul(wb, w32(a)), wq = cmul(wb, w32(q));
                double2 xa = untangle1(v[a], ma, wa);
                double2 xq = untangle1(v[q], mq, wq);
                if (n > 0) {
                    double2 sa, sq;
                    tm_ld2(tbase + 4 * a, tbase + 4 * q, sa, sq);
                    xa = cmul(sa, xa);
                    xq = cmul(sq, xq);
                }
                if (!last) {
                    tm_st1(tbase + 4 * a, xa);
                    tm_st1(tbase + 4 * q, xq);
                    continue;
                }
                // final spectrum bins: pack against the partner's mirrored bins
                double2 pa = shfl16(xq), pq = shfl16(xa);
                if (selfh) {
                    pa = xq;
                    pq = xa;
                }
                if (self0) {  // mirrors lie in other pairs: packed after the loop
                    s_stash[16 + a] = xa;
                    s_stash[16 + q] = xq;
                } else {
                    buf[spad(jl + a * T)] = pack1(xa, pa, wa);
                    buf[spad(jl + q * T)] = pack1(xq, pq, wq);
                }
            }
            if (!last) {
                tm_wait_st();
                __syncthreads();  // slots zeroed before the next scatter
                stamp(4);
                continue;
            }
            if (self0) {  // j = 0: bin r pairs with bin 16 - r (bin 0 with bin N2)
#pragma unroll
                for (int a = 0; a < 16; ++a) {
                    const double2 m = a == 0 ? make_double2(s_n2f, 0.0) : s_stash[16 + ((16 - a) & 15)];
                    buf[spad(a * T)] = pack1(s_stash[16 + a], m, cmul(wb, w32(a)));
                }
            }
            __syncthreads();
            stamp(4);
        }
        // ---- inverse: H-point FFT of conj(Z'_h) = conj(E) or conj(O) ----
        split_pass<H, R1, true>(buf, 1, tw, false);
        split_pass<H, 16, false>(buf, R1, tw, false);
        double2 uu[16];
        last_pass<H>(buf, t, tw, uu, false);
        stamp(5);
        cluster_sync_all();  // #1: both CTAs are done reading their buffers
        // CTA 0 outputs m = t + T r for r < 8 and needs O there; CTA 1 the rest
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const int rs = odd ? a : a + 8;  // the half this CTA sends
            st_peer(peer_addr(buf + spad(t + rs * T), peer), odd ? uu[a] : uu[a + 8]);
        }
        cluster_sync_all();  // #2: the peer's half has landed in this buffer
        const double scale = wr / (double)(2 * H);
        double2* y2 = reinterpret_cast<double2*>(g.Y + r * (int64_t)M);
        const double2 wb = tw(2 * t);
        double nrm = 0.0;
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const int ro = odd ? a + 8 : a;
            const double2 other = buf[spad(t + ro * T)];
            const double2 mine = odd ? uu[a + 8] : uu[a];  // constant indices: no local copy
            const double2 uE = odd ? other : mine;
            const double2 uO = odd ? mine : other;
            const double2 wo = cmul(cmul(wb, odd ? w32(a + 8) : w32(a)), uO);
            const double2 zl = cadd(uE, wo), zh = csub(uE, wo);
            const int m = t + ro * T;
            const double2 ol = make_double2(zl.x * scale, -zl.y * scale);
            const double2 oh = make_double2(zh.x * scale, -zh.y * scale);
            __stcs(y2 + m, ol);
            __stcs(y2 + m + H, oh);
            nrm = fma(ol.x, ol.x, nrm);
            nrm = fma(ol.y, ol.y, nrm);
            nrm = fma(oh.x, oh.x, nrm);
            nrm = fma(oh.y, oh.y, nrm);
        }
#pragma unroll
        for (int a = 0; a < 16; ++a) buf[spad(t + a * T)] = make_double2(0.0, 0.0);
        if (g.colnorm2) {  // fixed order: lanes, warps, then the even half + the odd half
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
            if (lane == 0) s_red[warp] = nrm;
            __syncthreads();
            if (t == 0) {
                double acc = 0.0;
#pragma unroll
                for (int w = 0; w < T / 32; ++w) acc += s_red[w];
                if (odd) st_peer1(peer_addr(&s_peer_nrm, peer), acc);
                else s_red[0] = acc;
            }
        }
        cluster_sync_all();  // #3: zeroed buffers, the odd half's norm delivered
        if (g.colnorm2 && !odd && t == 0) g.colnorm2[r] = s_red[0] + s_peer_nrm;
        stamp(6);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_taddr),
                     "r"(g.tmem_cols)
                     : "memory");
}

// Plan of one mode.  The rows are cut into chunks: the whole column when its
// later rows (all but the first row of each slot) fit the kernel's tail
// buffer, else fixed chunks of 16 T rows.  Per row: the slot's buffer index,
// its signs in the two halves, and -- for a row that is not the first of its
// slot in the chunk -- its position in the chunk's tail buffer (ordered by
// slot, then row).  Per chunk: the tail groups (slots with later rows, in
// slot order: buffer index | tail start << 16, count) and their number.
// Header: rows per chunk.

// double index of real slot j (packed complex point j >> 1) in the padded buffer
__device__ __forceinline__ uint32_t split_idx(int j) { return (uint32_t)(2 * spad(j >> 1) + (j & 1)); }

#ifdef IDS_PLAN_TIMING
__device__ long long g_plan_t[8];
#endif

struct PlanOut {
    int32_t* hdr;
    uint32_t* code;
    uint2* groups;
    int32_t* ngroups;
};

// Ranks the rows [i0, i1) among the earlier rows of their slot (warp 0 walks
// them in order, 32 at a time; __match_any_sync resolves equal slots), then
// one block scan of the per-slot (later rows, has-group) counts.  Returns the
// chunk's later-row total; writes codes and groups when it is <= cap.
__device__ int plan_chunk(const int32_t* __restrict__ bucket, const int8_t* __restrict__ sign, int i0,
                          int i1, int N2, int cap, int32_t* cnt, int32_t* rank, uint16_t* wc, int32_t* s_part,
                          uint32_t* __restrict__ code, uint2* __restrict__ gc, int32_t* ngroups) {
    // The rows' (slot, b >= N2, sign) are staged in shared memory first
    // (rank[] holds slot | hi << 13 | neg << 14, the rank joins at << 15).
    // Every warp walks its own eighth of the rows in order (32 at a time,
    // __match_any_sync resolves equal slots) against its own 16-bit slot
    // counters; the per-warp counts are then turned into bases by a prefix
    // over the warps, so rank = base[warp][slot] + rank inside the warp's part.
    const int T = blockDim.x, t = threadIdx.x, w = t >> 5, lane = t & 31, NW = T >> 5;
    const int len = i1 - i0;
#ifdef IDS_PLAN_TIMING
    long long tp0 = clock64();
#define PSTAMP(k) do { if (t == 0) { long long tn = clock64(); g_plan_t[k] += tn - tp0; tp0 = tn; } } while (0)
#else
#define PSTAMP(k) do {} while (0)
#endif
    for (int q0 = 0; q0 < len; q0 += 8 * T) {  // eight loads of each array in flight
        int32_t bb[8];
        int8_t sg[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int q = q0 + u * T + t;
            bb[u] = q < len ? __ldg(bucket + i0 + q) : 0;
            sg[u] = q < len ? __ldg(sign + i0 + q) : (int8_t)1;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int q = q0 + u * T + t;
            if (q < len) rank[q] = (bb[u] & (N2 - 1)) | (bb[u] >= N2 ? 1 << 13 : 0) | (sg[u] < 0 ? 1 << 14 : 0);
        }
    }
    for (int q = t; q < NW * N2 / 8; q += T) reinterpret_cast<uint4*>(wc)[q] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    PSTAMP(0);
    const int sub = (len + NW - 1) / NW;
    const int wa = w * sub, wb = min(len, wa + sub);
    uint16_t* mine = wc + w * N2;
    const unsigned lt = (1u << lane) - 1u;
    for (int base = wa; base < wb; base += 32) {
        const int q = base + lane;
        const bool ok = q < wb;
        const int e = ok ? rank[q] : 0;
        const int slot = e & (N2 - 1);
        const int key = ok ? slot : -1 - lane;
        const unsigned m = __match_any_sync(0xffffffffu, key);
        const int bc = ok ? mine[slot] : 0;
        __syncwarp();
        if (ok && (m >> lane) == 1u) mine[slot] = (uint16_t)(bc + __popc(m));  // highest lane of its group
        __syncwarp();
        if (ok) rank[q] = e | ((bc + __popc(m & lt)) << 15);
    }
    __syncthreads();
    PSTAMP(1);
    for (int g8 = t; g8 < N2 / 8; g8 += T) {  // per-warp counts -> bases; totals (8 slots a thread)
        int run[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int v = 0; v < NW; ++v) {
            uint4* cell = reinterpret_cast<uint4*>(wc + v * N2) + g8;
            const uint4 c = *cell;
            const uint32_t cw[4] = {c.x, c.y, c.z, c.w};
            uint32_t ow[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                ow[h] = (uint32_t)run[2 * h] | ((uint32_t)run[2 * h + 1] << 16);
                run[2 * h] += (int)(cw[h] & 0xFFFFu);
                run[2 * h + 1] += (int)(cw[h] >> 16);
            }
            *cell = make_uint4(ow[0], ow[1], ow[2], ow[3]);
        }
#pragma unroll
        for (int h = 0; h < 8; ++h) cnt[8 * g8 + h] = run[h];
    }
    __syncthreads();
    PSTAMP(2);
    for (int q = t; q < len; q += T) rank[q] += (int)wc[(q / sub) * N2 + (rank[q] & (N2 - 1))] << 15;
    __syncthreads();
    PSTAMP(3);
    // exclusive scan of packed (count - 1, count >= 2): low 16 bits later
    // rows, high 16 bits groups (both < 2^16 for the chunk sizes used).
    // Warp w scans its 1/NW of the slots 32 at a time (lane = slot: no bank
    // conflicts); pass 1 sums, the warp totals are prefixed, pass 2 writes.
    const int span = N2 / NW, s0w = w * span;
    auto packed = [&](int x) { return x >= 2 ? (x - 1) | (1 << 16) : 0; };
    int wsum = 0;
    for (int c0 = 0; c0 < span; c0 += 32) wsum += __reduce_add_sync(0xffffffffu, packed(cnt[s0w + c0 + lane]));
    if (lane == 0) s_part[w] = wsum;
    __syncthreads();
    if (t < 32) {
        int v = t < NW ? s_part[t] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, v, o);
            if (t >= o) v += y;
        }
        if (t < NW) s_part[t] = v;  // inclusive warp totals
    }
    __syncthreads();
    const int total = s_part[NW - 1];
    if ((total & 0xFFFF) > cap) {
        __syncthreads();  // everyone has read s_part before the next use
        return total & 0xFFFF;
    }
    int carry = w ? s_part[w - 1] : 0;
    for (int c0 = 0; c0 < span; c0 += 32) {
        const int sl = s0w + c0 + lane;
        const int x = cnt[sl];
        const int pv = packed(x);
        int inc = pv;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const int run = carry + inc - pv;
        cnt[sl] = run;
        if (x >= 2) gc[run >> 16] = make_uint2(split_idx(sl) | ((uint32_t)(run & 0xFFFF) << 16), (uint32_t)(x - 1));
        carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (t == 0) *ngroups = total >> 16;
    __syncthreads();
    PSTAMP(4);
    for (int q = t; q < len; q += T) {
        const int e = rank[q];
        const int slot = e & (N2 - 1);
        const int rk = e >> 15;
        const uint32_t tp = rk == 0 ? kFirst : (uint32_t)((cnt[slot] & 0xFFFF) + rk - 1);
        const uint32_t neg = (e >> 14) & 1, hi = (e >> 13) & 1;
        code[i0 + q] = split_idx(slot) | (neg << kSignShift) | ((neg ^ hi) << (kSignShift + 1)) | (tp << kTailShift);
    }
    __syncthreads();
    PSTAMP(5);
    return total & 0xFFFF;
#undef PSTAMP
}

// One CTA: the whole column as one chunk if its later rows fit `cap`, else
// fixed chunks of `cs` rows one after another.
__global__ void ts_split_plan_single(const int32_t* __restrict__ bucket, const int8_t* __restrict__ sign,
                                     int dim, int N2, int cs, int cap, PlanOut out) {
    extern __shared__ int32_t sm[];
    __shared__ int32_t s_part[32];
    int32_t* cnt = sm;
    int32_t* rank = sm + N2;
    uint16_t* wc = reinterpret_cast<uint16_t*>(sm + N2 + ((max(dim, cs) + 3) & ~3));
    const int tot = plan_chunk(bucket, sign, 0, dim, N2, cap, cnt, rank, wc, s_part, out.code, out.groups,
                               out.ngroups);
    if (tot <= cap) {
        if (threadIdx.x == 0) out.hdr[0] = dim;
        return;
    }
    for (int c = 0; c * cs < dim; ++c)
        plan_chunk(bucket, sign, c * cs, min(dim, (c + 1) * cs), N2, cs, cnt, rank, wc, s_part, out.code,
                   out.groups + (int64_t)c * (cs / 2), out.ngroups + c);
    if (threadIdx.x == 0) out.hdr[0] = cs;
}

// One CTA per fixed chunk of `cs` rows (long modes).
__global__ void ts_split_plan_chunks(const int32_t* __restrict__ bucket, const int8_t* __restrict__ sign,
                                     int dim, int N2, int cs, PlanOut out) {
    extern __shared__ int32_t sm[];
    __shared__ int32_t s_part[32];
    const int c = blockIdx.x;
    plan_chunk(bucket, sign, c * cs, min(dim, (c + 1) * cs), N2, cs, sm, sm + N2,
               reinterpret_cast<uint16_t*>(sm + N2 + cs), s_part, out.code,
               out.groups + (int64_t)c * (cs / 2), out.ngroups + c);
    if (c == 0 && threadIdx.x == 0) out.hdr[0] = cs;
}

// plan layout: hdr[4] | code[stride(dim)] | groups | ngroups
__host__ __device__ __forceinline__ int split_chunk_rows(int64_t out_dim) {
    return (int)(out_dim / 64 * kRows * kChunkRounds);
}
__host__ __device__ __forceinline__ int split_tail_cap(int64_t out_dim) { return (int)(out_dim / 64 * kTailPerThread); }
static size_t split_code_off() { return 16; }
static size_t split_groups_off(int64_t dim) { return align_up(16 + (size_t)split_stride(dim) * 4, 16); }
static size_t split_groups_count(int64_t dim, int64_t out_dim) {
    const int64_t cs = split_chunk_rows(out_dim);
    return (size_t)tmax<int64_t>(dim / 2 + 8, ceil_div(dim, cs) * (cs / 2));
}
static size_t split_ngroups_off(int64_t dim, int64_t out_dim) {
    return split_groups_off(dim) + split_groups_count(dim, out_dim) * sizeof(uint2);
}

int64_t* g_split_tlog = nullptr;

template <int H>
size_t split_smem_bytes() {
    return (size_t)(H + H / 16 + 1) * 16 + (size_t)(4 * H / kFine) * 16 + (size_t)kFineSlots * 16 +
           (size_t)(H / 16 * kTailPerThread) * 8;
}

template <int H>
int launch_split(const SplitArgs& a0, cudaStream_t st) {
    constexpr int T = H / 16;
    SplitArgs a = a0;
    a.tlog = g_split_tlog;
    // TMEM columns: warps w and w + 4 share lanes, 64 columns (16 complex) each
    const int warps = T / 32;
    a.tmem_cols = warps > 4 ? 128 : 64;
    auto kern = ts_split_kernel<H>;
    size_t smem = split_smem_bytes<H>();
    IDS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    // CTAs per SM from the kernel's registers and shared memory (the
    // occupancy API under-reports cluster kernels); at most 512 / tmem_cols
    // (an SM's TMEM): pad the shared-memory request until that holds
    cudaFuncAttributes fa{};
    IDS_CUDA_TRY(cudaFuncGetAttributes(&fa, kern));
    const int warps_cta = T / 32;
    const int regs_warp = (fa.numRegs * 32 + 255) / 256 * 256;
    const int occ_regs = 65536 / (regs_warp * warps_cta);
    const int cap = 512 / a.tmem_cols;
    auto occ_of = [&](size_t sm) {
        const int occ_smem = (int)((228 * 1024) / (sm + fa.sharedSizeBytes + 1024));
        return tmin(tmin(occ_regs, occ_smem), tmin(2048 / T, 32));
    };
    while (occ_of(smem) > cap && smem < 200 * 1024) smem += 2048;
    const int occ = occ_of(smem);
    if (occ < 1 || occ > cap) {
        ids_set_last_error("tensorsketch split: no occupancy fits TMEM");
        return IDS_EINVAL;
    }
    // persistent grid: every resident CTA pair is one cluster
    int fit = ids_sm_count() * occ / 2;
    const int64_t ncl = tmin<int64_t>(a.ncols, tmax<int64_t>(fit, 1));
    kern<<<(unsigned)(2 * ncl), T, smem, st>>>(a);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}

}  // namespace

// Debug hook: per-phase ns of ts_split_kernel (CTA 0) into device int64[8].
extern "C" void ids_debug_ts_split_timing(int64_t* buf) { g_split_tlog = buf; }

extern "C" int ids_tensorsketch_split_ok(int n_modes, int64_t out_dim) {
    if (n_modes < 1 || n_modes > kMaxModes) return 0;
    return out_dim == 4096 || out_dim == 8192 || out_dim == 16384;
}

extern "C" size_t ids_ts_split_plan_bytes(int64_t dim, int64_t out_dim) {
    if (dim < 1 || out_dim < 4) return 0;
    return split_ngroups_off(dim, out_dim) + (size_t)(ceil_div(dim, split_chunk_rows(out_dim)) + 4) * 4;
}

extern "C" int ids_ts_split_plan(const int32_t* bucket, const int8_t* sign, int64_t dim,
                                 int64_t out_dim, void* plan, size_t plan_bytes, void* stream) {
    if (!ids_tensorsketch_split_ok(1, out_dim) || dim < 1 || dim > 0x7fffffffLL || !plan ||
        plan_bytes < ids_ts_split_plan_bytes(dim, out_dim) ||
        (reinterpret_cast<uintptr_t>(plan) & 15)) {
        ids_set_last_error("ts split plan: bad arguments");
        return IDS_EINVAL;
    }
    cudaStream_t st = as_stream(stream);
    const int N2 = (int)(out_dim / 2), cs = split_chunk_rows(out_dim);
    char* base = static_cast<char*>(plan);
    PlanOut out{reinterpret_cast<int32_t*>(base), reinterpret_cast<uint32_t*>(base + split_code_off()),
                reinterpret_cast<uint2*>(base + split_groups_off(dim)),
                reinterpret_cast<int32_t*>(base + split_ngroups_off(dim, out_dim))};
    if (dim <= kSingleMax) {
        const int64_t rows = (tmax<int64_t>(dim, cs) + 3) & ~int64_t(3);
        const size_t sm = (size_t)(N2 + rows) * sizeof(int32_t) + 8 * (size_t)N2 * sizeof(uint16_t);
        IDS_CUDA_TRY(cudaFuncSetAttribute(ts_split_plan_single, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        ts_split_plan_single<<<1, 256, sm, st>>>(bucket, sign, (int)dim, N2, cs, split_tail_cap(out_dim), out);
    } else {
        const size_t sm = (size_t)(N2 + cs) * sizeof(int32_t) + 8 * (size_t)N2 * sizeof(uint16_t) + 16;
        IDS_CUDA_TRY(cudaFuncSetAttribute(ts_split_plan_chunks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        ts_split_plan_chunks<<<(unsigned)ceil_div(dim, cs), 256, sm, st>>>(bucket, sign, (int)dim, N2, cs, out);
    }
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}

extern "C" int ids_tensorsketch_split_f64(int n_modes, const double* const* factors, const int64_t* dims,
                                          const int64_t* lds, int64_t ncols, const void* const* plans,
                                          int64_t out_dim, const double* weights, double* Y,
                                          double* colnorm2, void* stream) {
    if (!ids_tensorsketch_split_ok(n_modes, out_dim) || ncols < 0) {
        ids_set_last_error("tensorsketch split: need 1..8 modes and out_dim in {4096, 8192, 16384}");
        return IDS_EINVAL;
    }
    SplitArgs a{};
    a.n_modes = n_modes;
    for (int n = 0; n < n_modes; ++n) {
        if (dims[n] < 1 || dims[n] > 0x7fffffffLL || lds[n] < dims[n] || !plans[n] || !factors[n]) {
            ids_set_last_error("tensorsketch split: bad factor shape or missing plan");
            return IDS_EINVAL;
        }
        a.factors[n] = factors[n];
        a.lds[n] = lds[n];
        a.dims[n] = (int)dims[n];
        const char* base = static_cast<const char*>(plans[n]);
        a.hdr[n] = reinterpret_cast<const int32_t*>(base);
        a.code[n] = reinterpret_cast<const uint32_t*>(base + split_code_off());
        a.groups[n] = reinterpret_cast<const uint2*>(base + split_groups_off(dims[n]));
        a.ngroups[n] = reinterpret_cast<const int32_t*>(base + split_ngroups_off(dims[n], out_dim));
    }
    if (ncols == 0) return IDS_OK;
    if ((reinterpret_cast<uintptr_t>(Y) & 15) != 0) {
        ids_set_last_error("tensorsketch split: Y must be 16-byte aligned");
        return IDS_EINVAL;
    }
    a.ncols = ncols;
    a.weights = weights;
    a.Y = Y;
    a.colnorm2 = colnorm2;
    cudaStream_t st = as_stream(stream);
    switch (out_dim) {
        case 4096: return launch_split<1024>(a, st);
        case 8192: return launch_split<2048>(a, st);
        default: return launch_split<4096>(a, st);
    }
}

#ifdef IDS_PLAN_TIMING  // experiments: clock64 per plan phase (thread 0), summed
extern "C" void ids_debug_plan_timing(long long* host8, int reset) {
    if (reset) {
        long long z[8] = {0};
        cudaMemcpyToSymbol(g_plan_t, z, sizeof(z));
    } else {
        cudaMemcpyFromSymbol(host8, g_plan_t, 8 * sizeof(long long));
    }
}
#endif
