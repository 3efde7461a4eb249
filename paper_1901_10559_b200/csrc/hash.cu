// Device CountSketch hash generation, bit-exact with the reference's numpy draws.
//
// Replaces reference sketch.py:77-84 (CountSketchOp.__init__).  The draw
// sequence numpy 2.3.5 performs there is:
//   phase A : I-L (surjective) or I (standard) 32-bit Lemire draws in [0, L),
//   phase B : (surjective) Fisher-Yates over slots = [0..L-1] ++ tail, i = I-1..1,
//             j = masked-rejection draw in [0, i],
//   signs   : I Lemire draws in [0, 2) (never rejected: sign bit of the draw).
// All three phases read ONE stream of 32-bit draws: the low then high halves
// of consecutive PCG64 outputs.
//
// B200 mapping
//   * phases A and signs are embarrassingly parallel: every thread jumps the
//     LCG to its chunk with the 2^k tables (pcg_tables.h) and generates
//     sequentially; Lemire rejections are stream-compacted with a block scan;
//   * phase B's accept/reject chain is inherently sequential in i; it is
//     resolved band by band (i in [2^k, 2^(k+1)): one mask) by a persistent
//     cooperative kernel: every warp summarises a chunk of draws as a function
//     of its unknown starting i (lowest start simulated, near misses folded
//     into "flats"), one warp stitches the summaries in order, the chunks are
//     re-run from their now exact starts to write j[], and one warp walks what
//     is left of the band (and everything below 2^12) exactly;
//   * the Fisher-Yates swaps themselves are applied in parallel: the value
//     that lands at position i is found by chasing "first later swap that
//     targeted this position" links (see fy_final_kernel), O(I) work;
//   * large draws are staged: the chain runs in three band groups and the
//     swaps of a finished group are applied on a side stream beside the rest
//     of the chain (final[i] depends on swaps above i only).  The signs are
//     drawn last, from the stream position the chain ends at, so no row's
//     sign -- and no part of the sketch -- can start before the chain ends.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <mutex>

#include "common.cuh"

namespace cg = cooperative_groups;

#define PCG_TABLE_QUAL __constant__
#include "pcg_tables.h"

typedef unsigned __int128 u128;

namespace {

constexpr int kGenThreads = 256;
constexpr int kChunk = 32;  // 32-bit draws per thread in the parallel phases
constexpr int32_t kNone = 0x7fffffff;

__device__ __forceinline__ u128 ld128(const uint64_t v[2]) {
    return ((u128)v[1] << 64) | (u128)v[0];
}

__device__ __forceinline__ uint64_t xsl_rr(u128 s) {
    const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
    const uint64_t x = hi ^ lo;
    const unsigned r = (unsigned)(hi >> 58);
    return (x >> r) | (x << ((64u - r) & 63u));
}

__device__ __forceinline__ u128 pcg_advance(u128 s, u128 inc, uint64_t n) {
    for (int k = 0; n != 0; ++k, n >>= 1)
        if (n & 1) s = ld128(PCG_MK[k]) * s + inc * ld128(PCG_GK[k]);
    return s;
}

// Sequential reader of the 32-bit draw stream from draw index d onwards.
struct DrawStream {
    u128 s, inc, mult;
    uint64_t cur;
    int half;
    __device__ void init(u128 s0, u128 inc_, uint64_t d) {
        inc = inc_;
        mult = ld128(PCG_MK[0]);
        s = pcg_advance(s0, inc, (d >> 1) + 1);
        cur = xsl_rr(s);
        half = (int)(d & 1);
    }
    __device__ __forceinline__ uint32_t next() {
        if (!half) {
            half = 1;
            return (uint32_t)cur;
        }
        const uint32_t r = (uint32_t)(cur >> 32);
        s = s * mult + inc;
        cur = xsl_rr(s);
        half = 0;
        return r;
    }
};

// PCG64 (state, inc) of a draw: by value, or read from device memory (dev
// non-NULL: {state_hi, state_lo, inc_hi, inc_lo}) so that a captured CUDA
// graph replays the draw for a new seed without re-recording its kernels.
struct Seed {
    uint64_t s_hi, s_lo, i_hi, i_lo;
    const uint64_t* dev;
    __device__ u128 state() const {
        return dev ? ((u128)__ldg(dev) << 64) | __ldg(dev + 1) : ((u128)s_hi << 64) | s_lo;
    }
    __device__ u128 inc() const {
        return dev ? ((u128)__ldg(dev + 2) << 64) | __ldg(dev + 3) : ((u128)i_hi << 64) | i_lo;
    }
};

__device__ __forceinline__ bool lemire_accept(uint32_t x, uint32_t L, uint32_t thresh,
                                              uint32_t* val) {
    const uint64_t m = (uint64_t)x * L;
    *val = (uint32_t)(m >> 32);
    return (uint32_t)m >= thresh;
}

// Fast path of phase A: with the usual sketch sizes a Lemire rejection has
// probability (2^32 mod L) / 2^32 (2e-8 for L = 200), so the first n_acc
// draws are normally all accepted and land at their own index.  This pass
// writes them so (16-byte stores) and raises *rejected if any draw is
// rejected, in which case the two compaction passes below redo phase A.
__global__ void __launch_bounds__(kGenThreads) lemire_fast_kernel(Seed sd, int64_t n_acc, uint32_t L,
                                                                  uint32_t thresh, int32_t* out,
                                                                  int64_t* consumed,
                                                                  int32_t* rejected) {
    const int64_t d0 = ((int64_t)blockIdx.x * kGenThreads + threadIdx.x) * kChunk;
    if (d0 >= n_acc) return;
    DrawStream ds;
    ds.init(sd.state(), sd.inc(), (uint64_t)d0);
    const int cnt = (int)tmin<int64_t>(kChunk, n_acc - d0);
    bool rej = false;
    if (cnt == kChunk && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
        int4* o = reinterpret_cast<int4*>(out + d0);
#pragma unroll
        for (int q = 0; q < kChunk / 4; ++q) {
            uint32_t v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) rej |= !lemire_accept(ds.next(), L, thresh, &v[u]);
            o[q] = make_int4((int)v[0], (int)v[1], (int)v[2], (int)v[3]);
        }
    } else {
        for (int t = 0; t < cnt; ++t) {
            uint32_t v;
            rej |= !lemire_accept(ds.next(), L, thresh, &v);
            out[d0 + t] = (int32_t)v;
        }
    }
    if (rej) atomicExch(rejected, 1);
    if (d0 + cnt == n_acc) *consumed = n_acc;
}

// Pass 1 of the Lemire compaction: accepted draws per block (only when the
// fast path saw a rejection).
__global__ void __launch_bounds__(kGenThreads) lemire_count_kernel(Seed sd, int64_t n_cand,
                                                                   uint32_t L, uint32_t thresh,
                                                                   int64_t* blk_cnt,
                                                                   const int32_t* rejected) {
    if (*rejected == 0) {  // fast path: the scan still reads blk_cnt, keep it defined
        if (threadIdx.x == 0) blk_cnt[blockIdx.x] = 0;
        return;
    }
    typedef cub::BlockReduce<int, kGenThreads> BR;
    __shared__ typename BR::TempStorage tmp;
    const int64_t d0 = ((int64_t)blockIdx.x * kGenThreads + threadIdx.x) * kChunk;
    int cnt = 0;
    if (d0 < n_cand) {
        DrawStream ds;
        ds.init(sd.state(), sd.inc(), (uint64_t)d0);
        const int n = (int)tmin<int64_t>(kChunk, n_cand - d0);
        for (int t = 0; t < n; ++t) {
            uint32_t v;
            cnt += lemire_accept(ds.next(), L, thresh, &v) ? 1 : 0;
        }
    }
    const int tot = BR(tmp).Sum(cnt);
    if (threadIdx.x == 0) blk_cnt[blockIdx.x] = tot;
}

// Pass 2: write the first n_acc accepted values; record draws consumed.  The
// block's accepted values form one contiguous output range: they are staged
// in shared memory (padded by one word per 32 against bank conflicts) and
// written with coalesced stores.
__device__ __forceinline__ int pad32(int x) { return x + (x >> 5); }

__global__ void __launch_bounds__(kGenThreads) lemire_write_kernel(
    Seed sd, int64_t n_cand, uint32_t L, uint32_t thresh, const int64_t* blk_off,
    int64_t n_acc, int32_t* out, int64_t* consumed, const int32_t* rejected) {
    if (*rejected == 0) return;
    typedef cub::BlockScan<int, kGenThreads> BS;
    __shared__ typename BS::TempStorage tmp;
    __shared__ int32_t stage[kGenThreads * kChunk + kGenThreads * kChunk / 32];
    const int64_t d0 = ((int64_t)blockIdx.x * kGenThreads + threadIdx.x) * kChunk;
    const int n = d0 < n_cand ? (int)tmin<int64_t>(kChunk, n_cand - d0) : 0;
    int cnt = 0;
    DrawStream ds;
    if (n > 0) {
        ds.init(sd.state(), sd.inc(), (uint64_t)d0);
        for (int t = 0; t < n; ++t) {
            uint32_t v;
            cnt += lemire_accept(ds.next(), L, thresh, &v) ? 1 : 0;
        }
    }
    int pre, tot;
    BS(tmp).ExclusiveSum(cnt, pre, tot);
    const int64_t ob = blk_off[blockIdx.x];
    if (ob >= n_acc) return;  // whole block past the last needed value
    if (n > 0 && ob + pre < n_acc) {
        ds.init(sd.state(), sd.inc(), (uint64_t)d0);
        int k = pre;
        for (int t = 0; t < n && ob + k < n_acc; ++t) {
            uint32_t v;
            if (lemire_accept(ds.next(), L, thresh, &v)) {
                stage[pad32(k)] = (int32_t)v;
                if (ob + k == n_acc - 1) *consumed = d0 + t + 1;
                ++k;
            }
        }
    }
    __syncthreads();
    const int m = (int)tmin<int64_t>(tot, n_acc - ob);
    for (int k = threadIdx.x; k < m; k += kGenThreads) out[ob + k] = stage[pad32(k)];
}

__global__ void fill_i32_kernel(int32_t* p, int64_t n, int32_t v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

__global__ void set_i64_kernel(int64_t* p, int64_t v) { *p = v; }

// Raw 32-bit draws [start, start + n) with start = sum of the device scalars
// off[0..n_off).
__global__ void __launch_bounds__(kGenThreads) raw_draws_kernel(Seed sd, const int64_t* off,
                                                                int n_off, int64_t n,
                                                                uint32_t* out) {
    int64_t base = 0;
    for (int k = 0; k < n_off; ++k) base += off[k];
    const int64_t d0 = ((int64_t)blockIdx.x * kGenThreads + threadIdx.x) * kChunk;
    if (d0 >= n) return;
    DrawStream ds;
    ds.init(sd.state(), sd.inc(), (uint64_t)(base + d0));
    const int cnt = (int)tmin<int64_t>(kChunk, n - d0);
    if (cnt == kChunk) {  // a thread's 32 draws are 128 aligned bytes: 16-byte stores
        uint4* o = reinterpret_cast<uint4*>(out + d0);
#pragma unroll
        for (int q = 0; q < kChunk / 4; ++q) {
            uint4 v;
            v.x = ds.next();
            v.y = ds.next();
            v.z = ds.next();
            v.w = ds.next();
            o[q] = v;
        }
    } else {
        for (int t = 0; t < cnt; ++t) out[d0 + t] = ds.next();
    }
}

// Signs: integers(0, 2) is Lemire with threshold 0 -> top bit of the draw.
__global__ void __launch_bounds__(kGenThreads) sign_kernel(Seed sd, const int64_t* off,
                                                           int n_off, int64_t n, int8_t* sign,
                                                           int vec) {
    int64_t base = 0;
    for (int k = 0; k < n_off; ++k) base += off[k];
    const int64_t d0 = ((int64_t)blockIdx.x * kGenThreads + threadIdx.x) * kChunk;
    if (d0 >= n) return;
    DrawStream ds;
    ds.init(sd.state(), sd.inc(), (uint64_t)(base + d0));
    const int cnt = (int)tmin<int64_t>(kChunk, n - d0);
    if (vec && cnt == kChunk) {  // 32 signs = 32 aligned bytes: two 16-byte stores
        uint32_t w[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            uint32_t x = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) x |= ((ds.next() >> 31) ? 0x01u : 0xffu) << (8 * b);
            w[q] = x;
        }
        uint4* o = reinterpret_cast<uint4*>(sign + d0);
        o[0] = make_uint4(w[0], w[1], w[2], w[3]);
        o[1] = make_uint4(w[4], w[5], w[6], w[7]);
    } else {
        for (int t = 0; t < cnt; ++t) sign[d0 + t] = (ds.next() >> 31) ? (int8_t)1 : (int8_t)-1;
    }
}

__device__ __forceinline__ uint32_t mask_of(uint32_t i) { return 0xFFFFFFFFu >> __clz(i); }

// ---- phase B: the accept/reject chain of the masked Fisher-Yates draws -----
// i runs n-1 .. 1; each 32-bit draw x gives v = x & mask(i); v <= i is
// accepted (j[i] = v, i -= 1), otherwise it is rejected.  FyState holds the
// exact (draw position, i) between stages.
struct FyState {
    int64_t pos;   // next unconsumed draw (relative to the phase-B stream)
    int64_t i;     // current i
    int64_t done;  // number of chunks resolved by the last stitch
    unsigned bar_count, bar_gen;  // ids_grid_bar state (zeroed before launch)
};


// One warp walks the chain EXACTLY over draws [pos, limit) from a known i,
// until i == i_stop: 256 draws per window, 8 consecutive draws per lane.
// Round: every unfinished lane classifies its draws assuming between 0 and
// 8*(lanes before it) accepts precede it; draws whose fate does not depend on
// that count are definite.  The first lane holding an ambiguous draw ends
// the round: the lanes before it are exact (prefix sum of their accepts) and
// it walks its own 8 draws exactly from the now exact start.  Optionally
// writes j[i] for accepted draws and records "near misses" (rejections with
// gap v - i in [1, w], in draw order) for the speculative chunks.
constexpr int kWalkAhead = 3;

struct WalkOut {
    int64_t i, pos;
    int nev;
};

__device__ WalkOut warp_walk(const uint32_t* __restrict__ g, int64_t pos, int64_t limit,
                             int64_t i64, int64_t i_stop64, int32_t* __restrict__ jout,
                             int64_t w64, int32_t* __restrict__ ev, int evmax) {
    // i < 2^31 (in_dim is limited to 2^31 - 2): the chain state and all the
    // per-draw arithmetic run in 32 bits; only draw positions are 64-bit
    const int ln = threadIdx.x & 31;
    int32_t i = (int32_t)i64;
    const int32_t i_stop = (int32_t)i_stop64;
    const int32_t w = (int32_t)tmin<int64_t>(w64, 0x7fffffff);
    int nev = 0;
    // windows are loaded kWalkAhead windows ahead (the walk of one window is
    // much shorter than a load's latency, even from L2)
    uint32_t xn[kWalkAhead][8];
    {
        const int64_t rem = limit - pos;
#pragma unroll
        for (int d = 0; d < kWalkAhead; ++d)
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int o = 256 * d + 8 * ln + q;
                xn[d][q] = o < rem ? __ldg(g + pos + o) : 0u;
            }
    }
    while (i > i_stop && pos < limit) {
        const int64_t rem = limit - pos;
        const int nval = rem < 256 ? (int)rem : 256;  // valid draws in this window
        uint32_t x[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            x[q] = xn[0][q];
#pragma unroll
            for (int d = 0; d + 1 < kWalkAhead; ++d) xn[d][q] = xn[d + 1][q];
            const int o = 256 * kWalkAhead + 8 * ln + q;
            xn[kWalkAhead - 1][q] = o < rem ? __ldg(g + pos + o) : 0u;
        }
        int b = 0;
        int32_t ib = i;
        bool stop = false;
        int64_t pos_final = 0;
        while (b < 32) {
            // -- speculative classification of this lane's draws
            int a = 0;
            bool amb = false;
            if (ln >= b) {
                const int32_t umax = 8 * (ln - b);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (!amb) {
                        const int32_t hi = ib - a, lo = hi - umax;
                        if (8 * ln + q >= nval || lo <= i_stop || lo < 1 ||
                            mask_of((uint32_t)lo) != mask_of((uint32_t)hi)) {
                            amb = true;
                        } else {
                            const int32_t v = (int32_t)(x[q] & mask_of((uint32_t)hi));
                            if (v <= lo) ++a;
                            else if (v <= hi) amb = true;
                        }
                    }
                }
            }
            const uint32_t ambb = __ballot_sync(0xffffffffu, amb);
            const int ls = ambb ? __ffs(ambb) - 1 : 32;
            const int cnt = (ln >= b && ln < ls) ? a : 0;
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (ln >= o) incl += y;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            // -- exact walk of lanes [b, ls]
            int32_t ii = ib - (incl - cnt);
            int endq = 8;
            int ne = 0;
            int32_t gaps[8];  // gaps[q] (statically indexed): near miss at draw q, or 0
            if (ln >= b && ln <= ls) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    gaps[q] = 0;
                    if (endq == 8) {
                        if (8 * ln + q >= nval || ii <= i_stop) {
                            endq = q;
                        } else {
                            const int32_t v = (int32_t)(x[q] & mask_of((uint32_t)ii));
                            if (v <= ii) {
                                if (jout) jout[ii] = v;
                                --ii;
                            } else if (v - ii <= w) {
                                gaps[q] = v - ii;
                                ++ne;
                            }
                        }
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < 8; ++q) gaps[q] = 0;
            }
            if (w > 0 && __ballot_sync(0xffffffffu, ne > 0)) {
                int einc = ne;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, einc, o);
                    if (ln >= o) einc += y;
                }
                int at = nev + einc - ne;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (gaps[q] != 0) {
                        if (at < evmax) ev[at] = gaps[q];
                        ++at;
                    }
                }
                nev += __shfl_sync(0xffffffffu, einc, 31);
            }
            if (ls == 32) {
                ib -= total;
                break;
            }
            ib = __shfl_sync(0xffffffffu, ii, ls);
            const int eq = __shfl_sync(0xffffffffu, endq, ls);
            b = ls + 1;
            if (eq < 8) {
                stop = true;
                pos_final = pos + 8 * ls + eq;
                break;
            }
        }
        i = ib;
        if (stop) {
            pos = pos_final;
            break;
        }
        pos += 256;
    }
    return WalkOut{i, tmin<int64_t>(pos, limit), nev};
}

// warp_walk for a walk that stays inside one band (cmask = 2 * lo_band - 1,
// lo_band - 1 <= i_stop, i <= cmask): the mask is a constant, and a lane whose
// eight draws are all definite needs no second pass -- its accepts are the
// classification's, so its j[] stores and near-miss gaps follow from the
// exact start by bit counts.  Only the first ambiguous lane walks its draws
// one by one.  The prefix sum of the lanes' accept counts (<= 8 each) is four
// bit-sliced ballots instead of five dependent shuffles.
__device__ WalkOut band_walk(const uint32_t* __restrict__ g, int64_t pos, int64_t limit,
                             int64_t i64, int64_t i_stop64, int32_t* __restrict__ jout,
                             int64_t w64, int32_t* __restrict__ ev, int evmax, uint32_t cmask) {
    const int ln = threadIdx.x & 31;
    const uint32_t ltm = (1u << ln) - 1u;
    int32_t i = (int32_t)i64;
    const int32_t i_stop = (int32_t)i_stop64;
    const int32_t w = (int32_t)tmin<int64_t>(w64, 0x7fffffff);
    int nev = 0;
    uint32_t xn[kWalkAhead][8];
    {
        const int64_t rem = limit - pos;
#pragma unroll
        for (int d = 0; d < kWalkAhead; ++d)
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int o = 256 * d + 8 * ln + q;
                xn[d][q] = o < rem ? __ldg(g + pos + o) : 0u;
            }
    }
    while (i > i_stop && pos < limit) {
        const int64_t rem = limit - pos;
        const int nval = rem < 256 ? (int)rem : 256;  // valid draws in this window
        int32_t v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            v[q] = (int32_t)(xn[0][q] & cmask);
#pragma unroll
            for (int d = 0; d + 1 < kWalkAhead; ++d) xn[d][q] = xn[d + 1][q];
            const int o = 256 * kWalkAhead + 8 * ln + q;
            xn[kWalkAhead - 1][q] = o < rem ? __ldg(g + pos + o) : 0u;
        }
        int b = 0;
        int32_t ib = i;
        bool stop = false;
        int64_t pos_final = 0;
        while (b < 32) {
            // -- speculative classification of this lane's draws
            int a = 0;
            uint32_t accm = 0;
            bool amb = false;
            if (ln >= b) {
                const int32_t umax = 8 * (ln - b);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (!amb) {
                        const int32_t hi = ib - a, lo = hi - umax;
                        if (8 * ln + q >= nval || lo <= i_stop) {
                            amb = true;
                        } else if (v[q] <= lo) {
                            ++a;
                            accm |= 1u << q;
                        } else if (v[q] <= hi) {
                            amb = true;
                        }
                    }
                }
            }
            const uint32_t ambb = __ballot_sync(0xffffffffu, amb);
            const int ls = ambb ? __ffs(ambb) - 1 : 32;
            const int cnt = (ln >= b && ln < ls) ? a : 0;
            const uint32_t c0 = __ballot_sync(0xffffffffu, cnt & 1);
            const uint32_t c1 = __ballot_sync(0xffffffffu, cnt & 2);
            const uint32_t c2 = __ballot_sync(0xffffffffu, cnt & 4);
            const uint32_t c3 = __ballot_sync(0xffffffffu, cnt & 8);
            const int excl = __popc(c0 & ltm) + 2 * __popc(c1 & ltm) + 4 * __popc(c2 & ltm) +
                             8 * __popc(c3 & ltm);
            const int total = __popc(c0) + 2 * __popc(c1) + 4 * __popc(c2) + 8 * __popc(c3);
            int32_t ii = ib - excl;
            int endq = 8;
            int ne = 0;
            int32_t gaps[8];  // gaps[q] (statically indexed): near miss at draw q, or 0
            if (ln >= b && ln < ls) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int32_t iq = ii - __popc(accm & ((1u << q) - 1u));
                    gaps[q] = 0;
                    if ((accm >> q) & 1u) {
                        if (jout) jout[iq] = v[q];
                    } else if (v[q] - iq <= w) {
                        gaps[q] = v[q] - iq;
                        ++ne;
                    }
                }
                ii -= a;
            } else if (ln == ls) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    gaps[q] = 0;
                    if (endq == 8) {
                        if (8 * ln + q >= nval || ii <= i_stop) {
                            endq = q;
                        } else if (v[q] <= ii) {
                            if (jout) jout[ii] = v[q];
                            --ii;
                        } else if (v[q] - ii <= w) {
                            gaps[q] = v[q] - ii;
                            ++ne;
                        }
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < 8; ++q) gaps[q] = 0;
            }
            if (w > 0 && __ballot_sync(0xffffffffu, ne > 0)) {
                int einc = ne;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, einc, o);
                    if (ln >= o) einc += y;
                }
                int at = nev + einc - ne;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (gaps[q] != 0) {
                        if (at < evmax) ev[at] = gaps[q];
                        ++at;
                    }
                }
                nev += __shfl_sync(0xffffffffu, einc, 31);
            }
            if (ls == 32) {
                ib -= total;
                break;
            }
            ib = __shfl_sync(0xffffffffu, ii, ls);
            const int eq = __shfl_sync(0xffffffffu, endq, ls);
            b = ls + 1;
            if (eq < 8) {
                stop = true;
                pos_final = pos + 8 * ls + eq;
                break;
            }
        }
        i = ib;
        if (stop) {
            pos = pos_final;
            break;
        }
        pos += 256;
    }
    return WalkOut{i, tmin<int64_t>(pos, limit), nev};
}

// Small-i variant of warp_walk: one draw per lane (32-draw windows, read 1024
// draws ahead), so the uncertainty of a lane's i is at most 31 -- better when
// i is small and wide windows would be mostly ambiguous.
__device__ WalkOut warp_walk1(const uint32_t* __restrict__ g, int64_t pos, int64_t limit, int64_t i,
                              int64_t i_stop, int32_t* __restrict__ jout) {
    const int ln = threadIdx.x & 31;
    const uint32_t lt = (1u << ln) - 1u;
    while (i > i_stop && pos < limit) {
        uint32_t xs[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const int64_t p = pos + 32 * k + ln;
            xs[k] = p < limit ? __ldg(g + p) : 0u;
        }
        bool stop = false;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            if (stop) break;
            const uint32_t x = xs[k];
            int b = 0;
            while (b < 32) {
                int stt = 0;  // 0 done, 1 accept, 2 reject, 3 ambiguous
                uint32_t v = 0;
                if (ln >= b) {
                    const int64_t hi = i, lo = i - (ln - b);
                    const int64_t p = pos + 32 * k + ln;
                    if (p >= limit || lo <= i_stop || lo < 1 ||
                        mask_of((uint32_t)lo) != mask_of((uint32_t)hi)) {
                        stt = 3;
                    } else {
                        v = x & mask_of((uint32_t)hi);
                        stt = (int64_t)v <= lo ? 1 : ((int64_t)v > hi ? 2 : 3);
                    }
                }
                const uint32_t accb = __ballot_sync(0xffffffffu, stt == 1);
                const uint32_t ambb = __ballot_sync(0xffffffffu, stt == 3);
                const int tamb = ambb ? __ffs(ambb) - 1 : 32;
                const uint32_t before = tamb < 32 ? (accb & ((1u << tamb) - 1u)) : accb;
                if (stt == 1 && ln < tamb && jout) jout[i - __popc(before & lt)] = (int32_t)v;
                const int A = __popc(before);
                if (tamb == 32) {
                    i -= A;
                    break;
                }
                int64_t is = i - A;
                const uint32_t xa = __shfl_sync(0xffffffffu, x, tamb);
                const int64_t pa = pos + 32 * k + tamb;
                if (pa >= limit || is <= i_stop) {
                    pos = pa;
                    i = is;
                    stop = true;
                    break;
                }
                const uint32_t vv = xa & mask_of((uint32_t)is);
                if ((int64_t)vv <= is) {
                    if (ln == 0 && jout) jout[is] = (int32_t)vv;
                    --is;
                }
                i = is;
                b = tamb + 1;
                if (i == i_stop) {
                    pos = pa + 1;
                    stop = true;
                    break;
                }
            }
        }
        if (stop) break;
        pos += 1024;
    }
    return WalkOut{i, tmin<int64_t>(pos, limit), 0};
}

// Speculative chunks of band [lo_band, hi_band] (mask = 2*lo_band - 1):
// chunk c covers draws st->pos + [c*T, (c+1)*T).  Its true starting i is
// unknown; the expected trajectory gives a window [s, s + W] that contains it
// with overwhelming probability.  The LOWEST start s is simulated; any start
// s + d stays exactly d above it except at "near misses", draws the base
// rejects with gap g = v - i_base in [1, W]: a trajectory whose current
// offset is >= g accepts there and its offset drops by one.  The gaps are
// folded into sorted "flats" of the end-state function
// D(d) = d - #{flats <= d}, evaluated by the stitch.
constexpr int kEvMax = 26;
struct __align__(16) FyChunk {
    int64_t s;    // lowest start in the window
    int32_t w;    // window width (-1: chunk not usable)
    int32_t a;    // accepts of the base trajectory
    int32_t ne;   // flats (-1: overflow)
    int32_t ev[kEvMax];
    int32_t pad_;
};
static_assert(sizeof(FyChunk) % 16 == 0, "FyChunk is staged with 16-byte copies");

// One warp: the summary of chunk c of the current epoch (state = epoch start).
__device__ void chunk_work(const uint32_t* __restrict__ g, int64_t nbuf, int64_t i0, int64_t pos,
                           int64_t lo_band, int64_t T, int64_t c, FyChunk* __restrict__ ch,
                           int32_t* ev) {
    const int ln = threadIdx.x & 31;
    const double tau = (double)(c * T);
    const double m2 = (double)(2 * lo_band);  // mask + 1
    const double gi = (double)(i0 + 1) * exp(-tau / m2) - 1.0;
    const int64_t half = c == 0 ? 0 : (int64_t)(3.0 * sqrt(tau) + 16.0);
    int64_t s = (int64_t)floor(gi) - half;
    int64_t hi = tmin<int64_t>((int64_t)floor(gi) + half, i0);
    if (c == 0) s = hi = i0;
    const int64_t pos0 = pos + c * T;
    int64_t o_s = 0;
    int32_t o_w = -1, o_a = 0, o_ne = 0;
    int32_t myf = 0x7fffffff;  // lane f holds flat f of the sorted list (never <= d when unused)
    if (s - T > lo_band && hi >= s && pos0 + T <= nbuf) {
        const int64_t w = hi - s;
        const WalkOut r = band_walk(g, pos0, pos0 + T, s, s - T - 1, nullptr, w, ev, kEvMax,
                                    (uint32_t)(2 * lo_band - 1));
        __syncwarp();
        o_s = s;
        o_w = (int32_t)w;
        o_a = (int32_t)(s - r.i);
        // gap g is taken by every trajectory whose current offset is >= g: the
        // smallest such start d* solves d* = g + #{flats <= d*}; the count is
        // one ballot over the lanes' flats
        int nf = 0;
        const bool over = r.nev > kEvMax;
        if (!over) {
            for (int e = 0; e < r.nev; ++e) {
                const int gap = ev[e];
                int d = gap, cnt;
                for (;;) {
                    cnt = __popc(__ballot_sync(0xffffffffu, myf <= d));
                    if (gap + cnt == d) break;
                    d = gap + cnt;
                }
                if (d > w) continue;  // no trajectory of the window reaches it
                // sorted insert at position cnt: later flats move up one lane
                const int32_t up = __shfl_up_sync(0xffffffffu, myf, 1);
                if (ln > cnt) myf = up;
                else if (ln == cnt) myf = d;
                ++nf;
            }
        }
        o_ne = over ? -1 : nf;
        if (over) myf = 0x7fffffff;
        __syncwarp();
    }
    if (ln == 0) {
        ch[c].s = o_s;
        ch[c].w = o_w;
        ch[c].a = o_a;
        ch[c].ne = o_ne;
    }
    if (ln < kEvMax) ch[c].ev[ln] = myf;
}

// One block (warp 0 walks, the block stages summaries in shared memory):
// resolves the chunks in order from the exact epoch start; stops at the first
// chunk whose start leaves its window (the exact walk continues from there).
// Summaries arrive in batches of kStitchBatch through two shared buffers: the
// next batch is copied (cp.async) while warp 0 resolves the current one.
constexpr int kStitchBatch = 64;

__device__ __forceinline__ void stage_batch(FyChunk* dst, const FyChunk* __restrict__ src, int cnt) {
    const int words = (int)(cnt * sizeof(FyChunk) / 16);
    const char* s = reinterpret_cast<const char*>(src);
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    for (int w = threadIdx.x; w < words; w += blockDim.x)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d + 16 * w), "l"(s + 16 * w)
                     : "memory");
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}

__device__ void stitch_block(FyState* st, const FyChunk* __restrict__ ch, int64_t nchunks,
                             int64_t T, int64_t* __restrict__ starts, FyChunk* sm2) {
    __shared__ int64_t s_S, s_done;
    __shared__ int s_ok;
    __shared__ int32_t s_cs[kStitchBatch], s_k[kStitchBatch], s_cw[kStitchBatch];
    const int64_t pos0 = st->pos;
    if (threadIdx.x == 0) {
        s_S = st->i;
        s_ok = 1;
        s_done = 0;
        starts[-1] = pos0;
    }
    const int64_t nb = (nchunks + kStitchBatch - 1) / kStitchBatch;
    if (nb > 0) stage_batch(sm2, ch, (int)tmin<int64_t>(kStitchBatch, nchunks));
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t c0 = b * kStitchBatch;
        const int cnt = (int)tmin<int64_t>(kStitchBatch, nchunks - c0);
        FyChunk* sm = sm2 + (b & 1) * kStitchBatch;
        if (b + 1 < nb) {
            stage_batch(sm2 + ((b + 1) & 1) * kStitchBatch, ch + c0 + kStitchBatch,
                        (int)tmin<int64_t>(kStitchBatch, nchunks - c0 - kStitchBatch));
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        if (!s_ok) break;
        if (threadIdx.x < 32) {  // warp 0: lane e holds flat e; one ballot per chunk
            // The serial chain per chunk is start -> offset -> ballot -> popc ->
            // next start.  Everything else is taken off it: starts are kept
            // relative to the batch's first window (32-bit), the per-chunk
            // constants are prepared by the lanes in parallel, a chunk that
            // cannot be resolved is recorded (not branched on) and the walk
            // of the batch simply runs on, and the exact starts are written
            // 32 at a time.
            const int ln = threadIdx.x;
            const int64_t base = sm[0].s;
            for (int l = ln; l < cnt; l += 32) {
                const int32_t c32 = (int32_t)(sm[l].s - base);
                s_cs[l] = c32;
                s_k[l] = c32 - sm[l].a;
                s_cw[l] = (sm[l].w < 0 || sm[l].ne < 0) ? -1 : sm[l].w;
            }
            __syncwarp();
            const int64_t S0 = s_S;
            // a start outside +-2^30 of the first window fails chunk 0 anyway
            const int64_t rel = S0 - base;
            int32_t S = rel > (1 << 30) ? (1 << 30) : rel < -(1 << 30) ? -(1 << 30) : (int32_t)rel;
            int bad = cnt;
            int32_t Sbad = 0, keep = 0;
            int32_t cs = s_cs[0], ck = s_k[0], cw = s_cw[0];
            int32_t cf = ln < kEvMax ? sm[0].ev[ln] : 0x7fffffff;
#pragma unroll 4
            for (int l = 0; l < cnt; ++l) {
                const int nl = l + 1 < cnt ? l + 1 : l;
                const int32_t ncs = s_cs[nl], nk = s_k[nl], nw = s_cw[nl];
                const int32_t nf = ln < kEvMax ? sm[nl].ev[ln] : 0x7fffffff;
                const int32_t d = S - cs;
                if ((d < 0 || d > cw) && l < bad) {
                    bad = l;
                    Sbad = S;
                }
                const int nflat = __popc(__ballot_sync(0xffffffffu, cf <= d));
                if (ln == (l & 31)) keep = S;
                S = ck + d - nflat;
                if ((l & 31) == 31 || l == cnt - 1) {
                    const int l0 = l & ~31;
                    if (l0 + ln <= l && l0 + ln < bad) starts[c0 + l0 + ln] = base + keep;
                }
                cs = ncs;
                ck = nk;
                cw = nw;
                cf = nf;
            }
            if (ln == 0) {
                if (bad < cnt) s_ok = 0;
                s_S = bad < cnt ? (bad == 0 ? S0 : base + Sbad) : base + S;
                s_done += bad;
            }
        }
        __syncthreads();  // this buffer is refilled two batches on
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        st->i = s_S;
        st->pos = pos0 + s_done * T;
        st->done = s_done;
    }
}

__device__ __forceinline__ int64_t band_chunk_dev(int k, double mul, int64_t tmax) {
    const double want = mul * exp2(0.5 * k);
    int64_t T = 256;
    while (T < want && T < tmax) T <<= 1;
    return T;
}

// The whole phase-B chain in ONE persistent cooperative kernel: per band two
// speculative epochs (chunks -> stitch -> exact re-runs) and an exact warp
// walk of the band's tail, then a walk of the small bands; grid barriers
// separate the stages.
constexpr int kPbThreads = 128;
__global__ void __launch_bounds__(kPbThreads) fy_phaseb_kernel(
    const uint32_t* __restrict__ g, int64_t nbuf, int64_t n, int32_t* __restrict__ jout,
    FyState* st, FyChunk* __restrict__ ch, int64_t* __restrict__ starts, int64_t max_chunks,
    int kmin, int64_t* consumed, int64_t* status, int64_t* tlog, double tmul, int64_t t1max,
    int custom_bar, double e2_min_draws, int k_first, int k_last, int is_first, int is_last,
    int64_t walk1_below) {
    cg::grid_group grid = cg::this_grid();
    auto gsync = [&]() {
        if (custom_bar) ids_grid_bar(&st->bar_count, gridDim.x);
        else grid.sync();
    };
    int tl = 0;  // optional stage timestamps (globaltimer, ns) written by block 0
    auto stamp = [&](int tag) {
        if (tlog && blockIdx.x == 0 && threadIdx.x == 0 && tl < 254) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            tlog[2 * tl] = tag;
            tlog[2 * tl + 1] = (int64_t)t;
            ++tl;
        }
    };
    __shared__ int32_t evs[kPbThreads / 32][kEvMax];
    __shared__ FyChunk sm[2 * kStitchBatch];
    const int wib = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * (kPbThreads / 32) + wib;
    const int64_t nw = (int64_t)gridDim.x * (kPbThreads / 32);
    const bool lead_warp = blockIdx.x == 0 && wib == 0;
    if (n <= 1) {
        if (blockIdx.x == 0 && threadIdx.x == 0) *consumed = 0;
        return;
    }
    // A launch covers bands k_first .. k_last of the chain (the staged draw
    // splits it so that finished bands' swaps are applied beside the rest of
    // the chain); st carries the exact (pos, i) from one launch to the next.
    if (is_first) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            st->pos = 0;
            st->i = n - 1;
            st->done = 0;
        }
        gsync();
    }
    stamp(0);
    int top = 0;
    while ((2LL << top) <= n - 1) ++top;
    if (k_first < top) top = k_first;
    if (k_last > kmin) kmin = k_last;
    for (int k = top; k >= kmin; --k) {
        const int64_t lo_band = 1LL << k;
        const int64_t i0 = tmin<int64_t>(2 * lo_band - 1, n - 1);
        if (i0 < lo_band) continue;
        const int64_t T1 = band_chunk_dev(k, tmul, t1max);
        const double draws1 = (double)(2 * lo_band) * log((double)(i0 + 1) / (double)lo_band);
        const int64_t rem_i = (int64_t)(3.0 * sqrt(draws1) + 16.0) + T1 + 64;
        const int64_t T2 = tmax<int64_t>(256, T1 / 8);
        // Both epochs are stitched first; their exact re-runs (which only
        // write j) then run on every other warp while the lead warp walks
        // the band's tail.
        int64_t done_e[2] = {0, 0};
        for (int e = 0; e < 2; ++e) {
            const int64_t T = e == 0 ? T1 : T2;
            const int64_t nch = tmin<int64_t>(e == 0 ? (int64_t)(draws1 / (double)T1) + 2
                                                      : (2 * rem_i) / T2 + 2,
                                              max_chunks);
            if (nch < 2) continue;
            // the second (short-chunk) epoch only pays on long bands: on short
            // ones the exact tail walk is cheaper than its barriers and stitch
            if (e == 1 && draws1 < e2_min_draws) continue;
            const int64_t ei = st->i, ep = st->pos;
            for (int64_t c = gw; c < nch; c += nw) chunk_work(g, nbuf, ei, ep, lo_band, T, c, ch, evs[wib]);
            stamp(100 * k + 10 * e + 1);
            gsync();
            stamp(100 * k + 10 * e + 2);
            if (blockIdx.x == 0) stitch_block(st, ch, nch, T, starts + e * (max_chunks + 1), sm);
            stamp(100 * k + 10 * e + 3);
            gsync();
            stamp(100 * k + 10 * e + 4);
            done_e[e] = st->done;  // the next stitch (behind a grid barrier) rewrites it
        }
        stamp(100 * k + 6);
        if (lead_warp) {
            const WalkOut r = lo_band < walk1_below
                                  ? warp_walk1(g, st->pos, nbuf, st->i, lo_band - 1, jout)
                                  : band_walk(g, st->pos, nbuf, st->i, lo_band - 1, jout, 0, nullptr, 0,
                                              (uint32_t)(2 * lo_band - 1));
            // every lane holds r: st is read by all of them above
            __syncwarp();
            if (threadIdx.x == 0) {
                if (r.i > lo_band - 1) *status = IDS_ERETRY;
                st->i = r.i;
                st->pos = r.pos;
            }
        } else {
            const int64_t wk = nw > 1 ? nw - 1 : 1;
            for (int e = 0; e < 2; ++e) {
                const int64_t T = e == 0 ? T1 : T2;
                const int64_t* se = starts + e * (max_chunks + 1);
                for (int64_t c = gw - 1; c < done_e[e]; c += wk) {
                    const int64_t p0 = se[-1] + c * T;
                    band_walk(g, p0, p0 + T, se[c], lo_band, jout, 0, nullptr, 0,
                              (uint32_t)(2 * lo_band - 1));
                }
            }
        }
        stamp(100 * k + 7);
        gsync();
    }
    stamp(9000);
    if (!is_last) return;
    if (lead_warp) {
        const WalkOut r = st->i < 16384 ? warp_walk1(g, st->pos, nbuf, st->i, 0, jout)
                                        : warp_walk(g, st->pos, nbuf, st->i, 0, jout, 0, nullptr, 0);
        if (threadIdx.x == 0) {
            if (r.i > 0) *status = IDS_ERETRY;
            st->i = r.i;
            st->pos = r.pos;
            *consumed = r.pos;
        }
    }
    stamp(9999);
    if (tlog && blockIdx.x == 0 && threadIdx.x == 0) tlog[2 * tl] = -1;
}

// ---- parallel application of the Fisher-Yates swaps --------------------------
// Swap s (s = n-1 .. 1, in that order) exchanges positions s and j[s] <= s.
// S_p = {s > p : j[s] = p} are the swaps that target position p from above.
//   first[p]   = min S_p  (the last of them to execute),
//   incoming(s) = value at position s just before swap s
//              = incoming(first[s]) if S_s is non-empty, else slots[s],
//   final[i]   = incoming(i) if j[i] == i;
//              = incoming(min{s in S_{j[i]} : s > i}) if that exists,
//              = slots[j[i]] otherwise;     final[0] = incoming(0).
//
// Staged form: the swaps of [s_lo, s_hi) can be applied as soon as the chain
// has passed s_lo, while it is still resolving the lower swaps: final[i] for
// i >= s_lo depends on swaps > i only.  A later stage [s_lo', s_lo) groups
// only its own swaps; the earlier stages' swaps into p are all above it, so
// the smallest of them, the value first[p] held before this stage's count
// (`first_prev`), stands in for their whole list.
__global__ void fy_count_kernel(const int32_t* __restrict__ j, int64_t s_lo, int64_t n,
                                int32_t* first, int32_t* gcount) {
    if (s_lo < 1) s_lo = 1;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + s_lo; s < n;
         s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = j[s];
        if (p < s) {
            atomicMin(&first[p], (int32_t)s);
            atomicAdd(&gcount[p], 1);
        }
    }
}

__global__ void fy_scatter_kernel(const int32_t* __restrict__ j, int64_t s_lo, int64_t n,
                                  const int32_t* __restrict__ goff, int32_t* cursor,
                                  int32_t* members) {
    if (s_lo < 1) s_lo = 1;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + s_lo; s < n;
         s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = j[s];
        if (p < s) members[goff[p] + atomicAdd(&cursor[p], 1)] = (int32_t)s;
    }
}

__device__ __forceinline__ int32_t slot_value(int64_t p, int64_t L, const int32_t* tail) {
    return p < L ? (int32_t)p : tail[p - L];
}

__device__ __forceinline__ int32_t incoming(int32_t s, const int32_t* __restrict__ first,
                                            int64_t L, const int32_t* __restrict__ tail) {
    int32_t f = first[s];
    while (f != kNone) {
        s = f;
        f = first[s];
    }
    return slot_value(s, L, tail);
}

__global__ void fy_final_kernel(const int32_t* __restrict__ j, int64_t i_lo, int64_t n, int64_t L,
                                const int32_t* __restrict__ tail,
                                const int32_t* __restrict__ first,
                                const int32_t* __restrict__ first_prev,
                                const int32_t* __restrict__ goff,
                                const int32_t* __restrict__ members, int32_t* bucket) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + i_lo; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t out;
        if (i == 0) {
            out = incoming(0, first, L, tail);
        } else {
            const int32_t p = j[i];
            if (p == i) {
                out = incoming((int32_t)i, first, L, tail);
            } else {
                int32_t best = kNone;
                for (int32_t k = goff[p], e = goff[p + 1]; k < e; ++k) {
                    const int32_t m = members[k];
                    if (m > i && m < best) best = m;
                }
                if (best == kNone && first_prev) best = first_prev[p];
                out = best == kNone ? slot_value(p, L, tail) : incoming(best, first, L, tail);
            }
        }
        bucket[i] = out;
    }
}

int64_t* g_fy_tlog = nullptr;  // debug: stage timestamps of the phase-B kernel (single stage)
int g_fy_stages = 3;           // band groups of the staged draw (1 = chain, then every swap)
int64_t g_fy_stage_min = 1 << 21;  // shorter draws are not staged (no gain measured at 1e6)
int g_fy_kmin = 12;            // bands below 2^kmin are walked exactly by one warp
int64_t g_fy_walk1_below = 16384;  // band tails below this use the one-draw-per-lane walk
int g_fy_per_sm = 2;           // chain CTAs per SM (x 4 warps)
int g_fy_side_per_sm = 4;      // CTAs per SM of the applications that run beside the chain
int g_fy_split[2] = {3, 3};    // bands per stage (stage 1, stage 2)

// Side streams for the staged swap application: a small per-device pool
// handed out round robin, so concurrent draws (trial batches) do not queue
// their applications behind one another.
struct SidePipe {
    std::mutex mu;  // held while one draw enqueues on the pipe (its events are re-recorded per draw)
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t done = nullptr;
};
constexpr int kPipes = 8, kPipeDevs = 16;
SidePipe g_pipes[kPipeDevs][kPipes];
unsigned g_pipe_next[kPipeDevs];
std::mutex g_pipe_mu;

SidePipe* side_pipe() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kPipeDevs) return nullptr;
    std::lock_guard<std::mutex> lk(g_pipe_mu);
    // all of a device's pipes are made by its first staged draw (a stream
    // costs ~0.3 ms to create: not something to meet again on later calls)
    if (!g_pipes[dev][kPipes - 1].stream) {
        for (int k = 0; k < kPipes; ++k) {
            SidePipe* sp = &g_pipes[dev][k];
            if (sp->stream) continue;
            cudaStream_t s;
            if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
                cudaGetLastError();
                return nullptr;
            }
            bool ok = cudaEventCreateWithFlags(&sp->done, cudaEventDisableTiming) == cudaSuccess;
            for (int t = 0; t < 3; ++t)
                ok = ok &&
                     cudaEventCreateWithFlags(&sp->ev[t], cudaEventDisableTiming) == cudaSuccess;
            if (!ok) {
                cudaGetLastError();
                cudaStreamDestroy(s);
                return nullptr;
            }
            sp->stream = s;
        }
    }
    return &g_pipes[dev][g_pipe_next[dev]++ % kPipes];
}

int g_fy_grid_cap = 0;         // >0: cap on the phase-B grid (CTAs)
double g_fy_e2_min = 65536.0;  // bands with fewer draws skip the second epoch (swept 0..1e30)
int g_fy_custom_bar = 1;       // 1: nanosleep grid barrier (measured ~10% faster than cg grid.sync)
double g_fy_tmul = 1.6;        // chunk length of band k: pow2 >= tmul * 2^(k/2) (swept: 0.575..4.6)
int64_t g_fy_tmax = 4096;      // ... capped here

struct HashPlan {
    int64_t I, L;
    int surj;
    int64_t n_acc, n_cand, nblk, nbuf;
    int64_t max_chunks;
    size_t scan_bytes, scan2_bytes;
};

constexpr int kMinBand = 12;  // bands below 2^12 are walked exactly by one warp


HashPlan make_plan(int64_t I, int64_t L, int surj) {
    HashPlan p;
    p.I = I;
    p.L = L;
    p.surj = surj;
    p.n_acc = surj ? I - L : I;
    if (L <= 1) {
        p.n_cand = 0;
    } else {
        const double pr = (double)((uint32_t)(0u - (uint32_t)L) % (uint32_t)L) / 4294967296.0;
        const double mean = (double)p.n_acc * pr;
        p.n_cand = p.n_acc + (int64_t)(1.25 * mean + 16.0 * sqrt(mean + 1.0)) + 1024;
    }
    p.nblk = ceil_div(p.n_cand, (int64_t)kGenThreads * kChunk);
    if (p.nblk < 1) p.nblk = 1;
    p.nbuf = surj ? 2 * I + 16 * (int64_t)sqrt((double)I + 1.0) + 4096 : 0;
    p.nbuf = (p.nbuf + 1023) / 1024 * 1024;
    p.max_chunks = surj ? (2 * I) / 256 + 64 : 0;
    p.scan_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, p.scan_bytes, (int64_t*)nullptr, (int64_t*)nullptr,
                                  (int)p.nblk);
    p.scan2_bytes = 0;
    if (surj)
        cub::DeviceScan::ExclusiveSum(nullptr, p.scan2_bytes, (int32_t*)nullptr,
                                      (int32_t*)nullptr, (int)(I + 1));
    return p;
}

template <class W>
void carve(W& ws, const HashPlan& p, int64_t** blk_cnt, int64_t** blk_off, int64_t** scal,
           void** scan_tmp, int32_t** tail, uint32_t** draws, int32_t** jarr, int32_t** first,
           int32_t** first_prev, int32_t** gcount, int32_t** goff, int32_t** members, FyState** fst, FyChunk** chunks,
           int64_t** starts) {
    *blk_cnt = ws.template take<int64_t>(p.nblk);
    *blk_off = ws.template take<int64_t>(p.nblk);
    *scal = ws.template take<int64_t>(6);  // [4], [5]: phase-A rejection flag (int32)
    *scan_tmp = ws.template take<char>(p.scan_bytes > p.scan2_bytes ? p.scan_bytes
                                                                      : p.scan2_bytes);
    if (p.surj) {
        *tail = ws.template take<int32_t>(p.I - p.L + 1);
        *draws = ws.template take<uint32_t>(p.nbuf);
        *jarr = ws.template take<int32_t>(p.I + 1);
        *first = ws.template take<int32_t>(p.I + 1);
        *first_prev = ws.template take<int32_t>(p.I + 1);
        *gcount = ws.template take<int32_t>(p.I + 1);
        *goff = ws.template take<int32_t>(p.I + 1);
        *members = ws.template take<int32_t>(p.I + 1);
        *fst = ws.template take<FyState>(1);
        *chunks = ws.template take<FyChunk>(p.max_chunks);
        *starts = ws.template take<int64_t>(2 * (p.max_chunks + 1));  // one list per epoch
    }
}

struct NullCarve {
    size_t off = 0;
    template <class T>
    T* take(size_t n) {
        off = align_up(off, 256) + n * sizeof(T);
        return nullptr;
    }
};

}  // namespace

extern "C" size_t ids_hash_workspace_bytes(int64_t in_dim, int64_t out_dim, int surjective) {
    if (in_dim < 1 || out_dim < 1) return 0;
    HashPlan p = make_plan(in_dim, out_dim, surjective);
    NullCarve nc;
    int64_t *a, *b, *c;
    void* d;
    int32_t *e, *g, *h, *hp, *i2, *j2, *k2;
    uint32_t* f;
    FyState* fs;
    FyChunk* fc;
    int64_t* sts;
    carve(nc, p, &a, &b, &c, &d, &e, &f, &g, &h, &hp, &i2, &j2, &k2, &fs, &fc, &sts);
    return nc.off + 256;
}

static int countsketch_hash(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                            uint64_t inc_lo, const uint64_t* seed_dev, int64_t in_dim,
                            int64_t out_dim, int surjective, int32_t* bucket, int8_t* sign,
                            int64_t* draws_out, void* workspace, size_t ws_bytes, void* stream);

extern "C" int ids_countsketch_hash(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                                    uint64_t inc_lo, int64_t in_dim, int64_t out_dim,
                                    int surjective, int32_t* bucket, int8_t* sign,
                                    int64_t* draws_out, void* workspace, size_t ws_bytes,
                                    void* stream) {
    return countsketch_hash(state_hi, state_lo, inc_hi, inc_lo, nullptr, in_dim, out_dim,
                            surjective, bucket, sign, draws_out, workspace, ws_bytes, stream);
}

extern "C" int ids_countsketch_hash_dev(const uint64_t* seed_dev, int64_t in_dim, int64_t out_dim,
                                        int surjective, int32_t* bucket, int8_t* sign,
                                        int64_t* draws_out, void* workspace, size_t ws_bytes,
                                        void* stream) {
    if (!seed_dev) {
        ids_set_last_error("hash: seed_dev is NULL");
        return IDS_EINVAL;
    }
    return countsketch_hash(0, 0, 0, 0, seed_dev, in_dim, out_dim, surjective, bucket, sign,
                            draws_out, workspace, ws_bytes, stream);
}

static int countsketch_hash(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                            uint64_t inc_lo, const uint64_t* seed_dev, int64_t in_dim,
                            int64_t out_dim, int surjective, int32_t* bucket, int8_t* sign,
                            int64_t* draws_out, void* workspace, size_t ws_bytes, void* stream) {
    if (in_dim < 1 || out_dim < 1 || out_dim > 0x7fffffffLL || in_dim > 0x7ffffffeLL) {
        ids_set_last_error("hash: dimensions out of range");
        return IDS_EINVAL;
    }
    if (surjective && out_dim > in_dim) {
        ids_set_last_error("surjective mode requires out_dim <= in_dim");
        return IDS_EINVAL;
    }
    cudaStream_t st = as_stream(stream);
    HashPlan p = make_plan(in_dim, out_dim, surjective);
    WsCarve ws(workspace, ws_bytes);
    int64_t *blk_cnt, *blk_off, *scal;
    void* scan_tmp;
    int32_t *tail = nullptr, *jarr = nullptr, *first = nullptr, *first_prev = nullptr,
            *gcount = nullptr,
            *goff = nullptr, *members = nullptr;
    uint32_t* draws = nullptr;
    FyState* fst = nullptr;
    FyChunk* chunks = nullptr;
    int64_t* starts = nullptr;
    carve(ws, p, &blk_cnt, &blk_off, &scal, &scan_tmp, &tail, &draws, &jarr, &first, &first_prev,
          &gcount,
          &goff, &members, &fst, &chunks, &starts);
    if (!ws.ok()) {
        ids_set_last_error("hash: workspace too small");
        return IDS_EWORKSPACE;
    }
    int64_t* d = draws_out ? draws_out : scal;
    cudaEvent_t join = nullptr;  // set when swaps were applied on a side stream
    std::unique_lock<std::mutex> pipe_lock;  // that stream's pipe, held until the join is enqueued
    IDS_CUDA_TRY(cudaMemsetAsync(d, 0, 4 * sizeof(int64_t), st));
    Seed sd{state_hi, state_lo, inc_hi, inc_lo, seed_dev};
    const uint32_t L = (uint32_t)out_dim;
    const uint32_t thresh = L > 1 ? (uint32_t)(0u - L) % L : 0u;
    int32_t* phaseA_out = surjective ? tail : bucket;

    // ---- phase A / A': Lemire draws in [0, L) ----
    if (p.n_acc > 0) {
        if (L == 1) {  // numpy draws nothing for a single-value range
            fill_i32_kernel<<<1024, 256, 0, st>>>(phaseA_out, p.n_acc, 0);
            IDS_LAUNCH_CHECK();
        } else {
            int32_t* rejected = reinterpret_cast<int32_t*>(scal + 4);
            IDS_CUDA_TRY(cudaMemsetAsync(rejected, 0, sizeof(int32_t), st));
            const unsigned gf = (unsigned)ceil_div(p.n_acc, (int64_t)kGenThreads * kChunk);
            lemire_fast_kernel<<<gf, kGenThreads, 0, st>>>(sd, p.n_acc, L, thresh, phaseA_out,
                                                          d + 0, rejected);
            IDS_LAUNCH_CHECK();
            lemire_count_kernel<<<(unsigned)p.nblk, kGenThreads, 0, st>>>(sd, p.n_cand, L,
                                                                         thresh, blk_cnt, rejected);
            IDS_LAUNCH_CHECK();
            size_t sb = p.scan_bytes;
            IDS_CUDA_TRY(cub::DeviceScan::ExclusiveSum(scan_tmp, sb, blk_cnt, blk_off,
                                                       (int)p.nblk, st));
            lemire_write_kernel<<<(unsigned)p.nblk, kGenThreads, 0, st>>>(
                sd, p.n_cand, L, thresh, blk_off, p.n_acc, phaseA_out, d + 0, rejected);
            IDS_LAUNCH_CHECK();
        }
    }

    // ---- phase B: Fisher-Yates over slots ----
    if (surjective) {
        const int64_t I = in_dim;
        const unsigned gb = (unsigned)ceil_div(p.nbuf, (int64_t)kGenThreads * kChunk);
        raw_draws_kernel<<<gb, kGenThreads, 0, st>>>(sd, d, 1, p.nbuf, draws);
        IDS_LAUNCH_CHECK();
        // Stage plan: the chain is launched band group by band group; the
        // swaps of a finished group are applied on a side stream beside the
        // rest of the chain (only the last group's application stays on the
        // critical path).  Captured streams, short draws and draws with a
        // capped grid (the caller runs other draws or a sketch beside this
        // one, which already fill the chain's idle SMs: staging measured
        // 2.33-2.48 vs 2.12 ms per C3 trial) take one stage.
        int top = 0;
        while ((2LL << top) <= I - 1) ++top;
        int nst = 1;
        SidePipe* pipe = nullptr;
        if (I > 1 && g_fy_stages > 1 && g_fy_grid_cap == 0 && I >= g_fy_stage_min && top - 6 > kMinBand && !g_fy_tlog) {
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            IDS_CUDA_TRY(cudaStreamIsCapturing(st, &cs));
            if (cs == cudaStreamCaptureStatusNone) pipe = side_pipe();
            if (pipe) {
                nst = g_fy_stages > 3 ? 3 : g_fy_stages;
                pipe_lock = std::unique_lock<std::mutex>(pipe->mu);
            }
        }
        // stage t covers bands k_first[t] .. k_last[t]; its swaps are [s_lo[t], s_hi[t])
        int k_first[3] = {top, 0, 0}, k_last[3] = {0, 0, 0};
        int64_t s_lo[3] = {0, 0, 0}, s_hi[3] = {I, 0, 0};
        if (nst >= 2) {
            k_last[0] = top - g_fy_split[0] + 1;
            k_first[1] = k_last[0] - 1;
        }
        if (nst == 3) {
            k_last[1] = k_first[1] - g_fy_split[1] + 1;
            k_first[2] = k_last[1] - 1;
        }
        for (int t = 0; t + 1 < nst; ++t) {
            s_lo[t] = 1LL << k_last[t];
            s_hi[t + 1] = s_lo[t];
        }
        cudaStream_t ap = pipe ? pipe->stream : st;  // where the swaps are applied
        if (I > 1) {
            fill_i32_kernel<<<1024, 256, 0, st>>>(first, I, kNone);
            IDS_LAUNCH_CHECK();
        }
        int dev = 0, sms = 148, per_sm = 1;
        cudaGetDevice(&dev);
        {  // launch geometry, queried once per device
            static int c_sms[kPipeDevs], c_per_sm[kPipeDevs];
            static std::mutex mu;
            std::lock_guard<std::mutex> lk(mu);
            if (dev >= 0 && dev < kPipeDevs && c_sms[dev] > 0) {
                sms = c_sms[dev];
                per_sm = c_per_sm[dev];
            } else {
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fy_phaseb_kernel,
                                                              kPbThreads, 0);
                if (dev >= 0 && dev < kPipeDevs) {
                    c_sms[dev] = sms;
                    c_per_sm[dev] = per_sm;
                }
            }
        }
        int G = tmax(1, sms * tmin(per_sm, g_fy_per_sm));
        if (g_fy_grid_cap > 0) G = tmin(G, g_fy_grid_cap);
        if (g_fy_custom_bar) IDS_CUDA_TRY(cudaMemsetAsync(fst, 0, sizeof(FyState), st));
        for (int t = 0; t < nst; ++t) {
            {
                const uint32_t* dr = draws;
                int64_t nbuf = p.nbuf, nI = I, mc = p.max_chunks;
                int kmin = g_fy_kmin;
                int64_t wb = g_fy_walk1_below;
                int64_t* sts = starts + 1;
                int64_t* cons = d + 1;
                int64_t* stat = d + 3;
                int64_t* tlog = g_fy_tlog;
                int cbar = g_fy_custom_bar;
                double tmul = g_fy_tmul;
                double e2min = g_fy_e2_min;
                int64_t tmax = g_fy_tmax;
                int kf = k_first[t], kl = k_last[t], isf = t == 0, isl = t == nst - 1;
                void* args[] = {&dr,   &nbuf, &nI,   &jarr, &fst,  &chunks, &sts, &mc,  &kmin, &cons,
                                &stat, &tlog, &tmul, &tmax, &cbar, &e2min,  &kf,  &kl,  &isf,  &isl, &wb};
                IDS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)fy_phaseb_kernel, dim3(G),
                                                         dim3(kPbThreads), args, 0, st));
                ids_count_launch();
            }
            if (I <= 1) break;
            if (pipe) {
                IDS_CUDA_TRY(cudaEventRecord(pipe->ev[t], st));
                IDS_CUDA_TRY(cudaStreamWaitEvent(ap, pipe->ev[t], 0));
            }
            const int64_t lo = s_lo[t], hi = s_hi[t];  // targets of these swaps lie in [0, hi)
            const unsigned agrid = (unsigned)tmin<int64_t>(
                ceil_div(hi - lo, 256), (int64_t)sms * (t + 1 < nst ? g_fy_side_per_sm : 16));
            const int32_t* prev = nullptr;
            if (t > 0) {  // what the earlier stages left in first[0, hi)
                IDS_CUDA_TRY(cudaMemcpyAsync(first_prev, first, sizeof(int32_t) * hi,
                                             cudaMemcpyDeviceToDevice, ap));
                prev = first_prev;
            }
            IDS_CUDA_TRY(cudaMemsetAsync(gcount, 0, sizeof(int32_t) * (hi + 1), ap));
            fy_count_kernel<<<agrid, 256, 0, ap>>>(jarr, lo, hi, first, gcount);
            IDS_LAUNCH_CHECK();
            size_t sb = p.scan2_bytes;
            IDS_CUDA_TRY(
                cub::DeviceScan::ExclusiveSum(scan_tmp, sb, gcount, goff, (int)(hi + 1), ap));
            IDS_CUDA_TRY(cudaMemsetAsync(gcount, 0, sizeof(int32_t) * (hi + 1), ap));
            fy_scatter_kernel<<<agrid, 256, 0, ap>>>(jarr, lo, hi, goff, gcount, members);
            IDS_LAUNCH_CHECK();
            fy_final_kernel<<<agrid, 256, 0, ap>>>(jarr, lo, hi, out_dim, tail, first, prev, goff,
                                                   members, bucket);
            IDS_LAUNCH_CHECK();
        }
        if (pipe && I > 1) {  // the caller's stream continues after the last application
            IDS_CUDA_TRY(cudaEventRecord(pipe->done, ap));
            join = pipe->done;
        }
        if (I <= 1) {
            fill_i32_kernel<<<1, 32, 0, st>>>(bucket, 1, 0);
            IDS_LAUNCH_CHECK();
        }
    }

    // ---- signs ----
    {
        const unsigned gb = (unsigned)ceil_div(in_dim, (int64_t)kGenThreads * kChunk);
        const int vec = (reinterpret_cast<uintptr_t>(sign) & 15) == 0;
        sign_kernel<<<gb, kGenThreads, 0, st>>>(sd, d, 2, in_dim, sign, vec);
        IDS_LAUNCH_CHECK();
        set_i64_kernel<<<1, 1, 0, st>>>(d + 2, in_dim);
        IDS_LAUNCH_CHECK();
    }
    if (join) IDS_CUDA_TRY(cudaStreamWaitEvent(st, join, 0));
    return IDS_OK;
}

// Tuning hook (experiments): chunk-length rule of the speculative epochs.
extern "C" void ids_debug_fy_custom_bar(int v) { g_fy_custom_bar = v; }

extern "C" void ids_debug_fy_e2_min(double d) { g_fy_e2_min = d; }

extern "C" void ids_debug_phaseb_chunks(double mul, int64_t tmax) {
    g_fy_tmul = mul > 0 ? mul : 1.6;
    g_fy_tmax = tmax >= 256 ? tmax : 4096;
}

// Debug hook: record phase-B stage timestamps into `buf` (device int64[512])
// for the next hash draws; NULL disables.
extern "C" void ids_debug_phaseb_timing(int64_t* buf) { g_fy_tlog = buf; }

// Cap the phase-B grid at `ctas` CTAs (0 = whole GPU); lets several hash
// streams share the GPU.
extern "C" void ids_set_hash_grid_cap(int ctas) { g_fy_grid_cap = ctas > 0 ? ctas : 0; }

extern "C" void ids_debug_fy_per_sm(int v) { g_fy_per_sm = v > 0 ? v : 2; }

extern "C" void ids_debug_fy_small(int kmin, int64_t walk1_below) {
    g_fy_kmin = kmin >= 9 && kmin <= kMinBand ? kmin : kMinBand;
    g_fy_walk1_below = walk1_below > 0 ? walk1_below : 16384;
}

extern "C" void ids_debug_fy_side(int per_sm, int b0, int b1) {
    g_fy_side_per_sm = per_sm > 0 ? per_sm : 4;
    g_fy_split[0] = b0 > 0 ? b0 : 3;
    g_fy_split[1] = b1 > 0 ? b1 : 3;
}

// Band groups of the staged surjective draw (1..3; 1 = unstaged) and the
// smallest in_dim that is staged (0 keeps the default).
extern "C" void ids_set_hash_stages(int stages, int64_t min_in_dim) {
    g_fy_stages = stages < 1 ? 1 : stages > 3 ? 3 : stages;
    if (min_in_dim > 0) g_fy_stage_min = min_in_dim;
}
