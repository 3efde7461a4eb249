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
//     resolved by one CTA that classifies 1024 draws per round (definite
//     accept / reject / ambiguous) and only settles ambiguous lanes one at a
//     time, then by one warp once i < 65536;
//   * the Fisher-Yates swaps themselves are applied in parallel: the value
//     that lands at position i is found by chasing "first later swap that
//     targeted this position" links (see fy_final_kernel), O(I) work.
#include <cub/cub.cuh>

#include "common.cuh"

#define PCG_TABLE_QUAL __constant__
#include "pcg_tables.h"

typedef unsigned __int128 u128;

namespace {

constexpr int kGenThreads = 256;
constexpr int kChunk = 32;  // 32-bit draws per thread in the parallel phases
constexpr uint32_t kBlockMin = 65536;
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

struct Seed {
    uint64_t s_hi, s_lo, i_hi, i_lo;
    __device__ u128 state() const { return ((u128)s_hi << 64) | s_lo; }
    __device__ u128 inc() const { return ((u128)i_hi << 64) | i_lo; }
};

__device__ __forceinline__ bool lemire_accept(uint32_t x, uint32_t L, uint32_t thresh,
                                              uint32_t* val) {
    const uint64_t m = (uint64_t)x * L;
    *val = (uint32_t)(m >> 32);
    return (uint32_t)m >= thresh;
}

// Pass 1 of the Lemire compaction: accepted draws per block.
__global__ void __launch_bounds__(kGenThreads) lemire_count_kernel(Seed sd, int64_t n_cand,
                                                                   uint32_t L, uint32_t thresh,
                                                                   int64_t* blk_cnt) {
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

// Pass 2: write the first n_acc accepted values; record draws consumed.
__global__ void __launch_bounds__(kGenThreads) lemire_write_kernel(
    Seed sd, int64_t n_cand, uint32_t L, uint32_t thresh, const int64_t* blk_off,
    int64_t n_acc, int32_t* out, int64_t* consumed) {
    typedef cub::BlockScan<int, kGenThreads> BS;
    __shared__ typename BS::TempStorage tmp;
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
    int pre;
    BS(tmp).ExclusiveSum(cnt, pre);
    int64_t o = blk_off[blockIdx.x] + pre;
    if (n == 0 || o >= n_acc) return;
    ds.init(sd.state(), sd.inc(), (uint64_t)d0);
    for (int t = 0; t < n && o < n_acc; ++t) {
        uint32_t v;
        if (lemire_accept(ds.next(), L, thresh, &v)) {
            out[o] = (int32_t)v;
            if (o == n_acc - 1) *consumed = d0 + t + 1;
            ++o;
        }
    }
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
    for (int t = 0; t < cnt; ++t) out[d0 + t] = ds.next();
}

// Signs: integers(0, 2) is Lemire with threshold 0 -> top bit of the draw.
__global__ void __launch_bounds__(kGenThreads) sign_kernel(Seed sd, const int64_t* off,
                                                           int n_off, int64_t n, int8_t* sign) {
    int64_t base = 0;
    for (int k = 0; k < n_off; ++k) base += off[k];
    const int64_t d0 = ((int64_t)blockIdx.x * kGenThreads + threadIdx.x) * kChunk;
    if (d0 >= n) return;
    DrawStream ds;
    ds.init(sd.state(), sd.inc(), (uint64_t)(base + d0));
    const int cnt = (int)tmin<int64_t>(kChunk, n - d0);
    for (int t = 0; t < cnt; ++t) sign[d0 + t] = (ds.next() >> 31) ? (int8_t)1 : (int8_t)-1;
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
};

enum { ST_DONE = 0, ST_ACC = 1, ST_REJ = 2, ST_AMB = 3 };

// Lane of a 32-draw window: the true i before it lies in [i - u, i].  Definite
// when the mask is the same over that range, the range stays above i_stop and
// v is outside (lo, i].
__device__ __forceinline__ int classify(uint32_t x, int64_t i, int64_t u, int64_t i_stop,
                                        uint32_t* v) {
    const int64_t lo = i - u;
    const uint32_t m = mask_of((uint32_t)i);
    if (lo <= i_stop || lo < 1 || mask_of((uint32_t)lo) != m) return ST_AMB;
    *v = x & m;
    if ((int64_t)*v <= lo) return ST_ACC;
    if ((int64_t)*v > i) return ST_REJ;
    return ST_AMB;
}

// One warp walks the chain exactly from st->(pos, i) until i == i_stop,
// 32 draws per round (ambiguous lanes are settled one at a time).  When
// i_stop == 0 the walk ends the phase and *consumed gets the draw count.
__device__ void fy_walk_warp(const uint32_t* __restrict__ g, int64_t nbuf, int64_t i_stop,
                             int32_t* __restrict__ jout, FyState* st, int64_t* status) {
    const int ln = threadIdx.x & 31;
    const uint32_t lt_mask = (1u << ln) - 1u;
    int64_t i = st->i, pos = st->pos;
    while (i > i_stop) {
        if (pos + 1024 > nbuf) {
            if (ln == 0) *status = IDS_ERETRY;
            break;
        }
        uint32_t xs[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) xs[k] = __ldg(g + pos + 32 * k + ln);
        bool stop = false;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            if (stop) break;
            const uint32_t x = xs[k];
            int b = 0;
            while (b < 32) {
                uint32_t v = 0;
                const int stt = (ln >= b) ? classify(x, i, ln - b, i_stop, &v) : ST_DONE;
                const uint32_t accb = __ballot_sync(0xffffffffu, stt == ST_ACC);
                const uint32_t ambb = __ballot_sync(0xffffffffu, stt == ST_AMB);
                const int tamb = ambb ? __ffs(ambb) - 1 : 32;
                const uint32_t before = tamb < 32 ? (accb & ((1u << tamb) - 1u)) : accb;
                if (stt == ST_ACC && ln < tamb) jout[i - __popc(before & lt_mask)] = (int32_t)v;
                const int A = __popc(before);
                if (tamb == 32) {
                    i -= A;
                    break;
                }
                int64_t is = i - A;
                const uint32_t xa = __shfl_sync(0xffffffffu, x, tamb);
                if (is <= i_stop) {  // stage ends before this draw
                    pos += 32 * k + tamb;
                    i = is;
                    stop = true;
                    break;
                }
                const uint32_t vv = xa & mask_of((uint32_t)is);
                if ((int64_t)vv <= is) {
                    if (ln == 0) jout[is] = (int32_t)vv;
                    --is;
                }
                i = is;
                b = tamb + 1;
                if (i == i_stop) {
                    pos += 32 * k + tamb + 1;
                    stop = true;
                    break;
                }
            }
        }
        if (!stop) pos += 1024;
    }
    __syncwarp();
    if (ln == 0) {
        st->i = i;
        st->pos = pos;
    }
}

__global__ void fy_walk_kernel(const uint32_t* __restrict__ g, int64_t nbuf, int64_t i_stop,
                               int32_t* __restrict__ jout, FyState* st, int64_t* consumed,
                               int64_t* status) {
    fy_walk_warp(g, nbuf, i_stop, jout, st, status);
    if (i_stop == 0 && threadIdx.x == 0) *consumed = st->pos;
}

__global__ void fy_init_kernel(FyState* st, int64_t n) {
    st->pos = 0;
    st->i = n - 1;
    st->done = 0;
}

// Speculative chunks of band [lo_band, hi_band] (mask = 2*lo_band - 1):
// chunk c covers draws st->pos + [c*T, (c+1)*T).  Its true starting i is
// unknown; the expected trajectory gives a window [s, s + W] that contains it
// with overwhelming probability.  The LOWEST start s is simulated; any start
// s + d stays exactly d above it except at "near misses", draws the base
// rejects with gap g = v - i_base in [1, W]: a trajectory whose current
// offset is >= g accepts there and its offset drops by one.  Recording those
// gaps (in order) makes the chunk's end state a cheap function of the true
// start, evaluated by the stitch below.
constexpr int kEvMax = 24;
struct FyChunk {
    int64_t s;    // lowest start in the window
    int32_t w;    // window width (-1: chunk not usable)
    int32_t a;    // accepts of the base trajectory
    int32_t ne;   // near-miss events recorded (-1: overflow)
    int32_t ev[kEvMax];
};

__global__ void fy_chunk_kernel(const uint32_t* __restrict__ g, int64_t nbuf, const FyState* st,
                                int64_t i0, int64_t lo_band, int64_t T, int64_t nchunks,
                                FyChunk* __restrict__ ch) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nchunks) return;
    FyChunk out;
    out.w = -1;
    out.a = 0;
    out.ne = 0;
    out.s = 0;
    const double tau = (double)(c * T);
    const double m2 = (double)(2 * lo_band);  // mask + 1
    const double gi = (double)(i0 + 1) * exp(-tau / m2) - 1.0;
    const int64_t half = c == 0 ? 0 : (int64_t)(3.0 * sqrt(tau) + 16.0);
    int64_t s = (int64_t)floor(gi) - half;
    int64_t hi = tmin<int64_t>((int64_t)floor(gi) + half, i0);
    if (c == 0) s = hi = i0;
    const int64_t pos0 = st->pos + c * T;
    if (s - T > lo_band && hi >= s && pos0 + T <= nbuf) {
        const uint32_t m = (uint32_t)(2 * lo_band - 1);
        const int64_t w = hi - s;
        int64_t i = s;
        int a = 0, ne = 0;
        const uint32_t* x = g + pos0;
        for (int64_t t = 0; t < T; ++t) {
            const int64_t v = (int64_t)(__ldg(x + t) & m);
            if (v <= i) {
                --i;
                ++a;
            } else if (v - i <= w) {
                if (ne < kEvMax) out.ev[ne] = (int32_t)(v - i);
                ++ne;
            }
        }
        out.s = s;
        out.w = (int32_t)w;
        out.a = a;
        out.ne = ne <= kEvMax ? ne : -1;
    }
    ch[c] = out;
}

// Exact re-run of chunk c from its resolved start, writing j (one thread each).
__global__ void fy_chunk_exact_kernel(const uint32_t* __restrict__ g, const FyState* st0,
                                      const int64_t* __restrict__ starts, int64_t lo_band,
                                      int64_t T, int32_t* __restrict__ jout, int64_t pos_base) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= st0->done) return;
    const uint32_t m = (uint32_t)(2 * lo_band - 1);
    int64_t i = starts[c];
    const uint32_t* x = g + starts[-1] + c * T;  // starts[-1] holds the band's first draw
    for (int64_t t = 0; t < T; ++t) {
        const uint32_t v = __ldg(x + t) & m;
        if ((int64_t)v <= i) {
            jout[i] = (int32_t)v;
            --i;
        }
    }
    (void)pos_base;
}

// One warp resolves the chunks in order: the true start of chunk c gives its
// offset d in the window; replaying the near-miss gaps gives the end state.
// A chunk whose start falls outside its window (or overflowed) stops the
// stitch; the exact walk then continues from there.
__global__ void fy_stitch_kernel(FyState* st, const FyChunk* __restrict__ ch, int64_t nchunks,
                                 int64_t T, int64_t* __restrict__ starts) {
    const int ln = threadIdx.x & 31;
    int64_t S = st->i;
    const int64_t pos0 = st->pos;
    if (ln == 0) starts[-1] = pos0;
    int64_t done = 0;
    bool ok = true;
    for (int64_t c0 = 0; c0 < nchunks && ok; c0 += 32) {
        const int64_t c = c0 + ln;
        FyChunk mine;
        mine.w = -1;
        if (c < nchunks) mine = ch[c];
        const int cnt = (int)tmin<int64_t>(32, nchunks - c0);
        for (int l = 0; l < cnt; ++l) {
            const int64_t s = __shfl_sync(0xffffffffu, mine.s, l);
            const int w = __shfl_sync(0xffffffffu, mine.w, l);
            const int ne = __shfl_sync(0xffffffffu, mine.ne, l);
            const int64_t d = S - s;
            if (w < 0 || ne < 0 || d < 0 || d > w) {
                ok = false;
                break;
            }
            int64_t dd = d;
            if (ln == l) {
                for (int e = 0; e < ne; ++e)
                    if (dd >= mine.ev[e]) --dd;
            }
            dd = __shfl_sync(0xffffffffu, dd, l);
            const int a = __shfl_sync(0xffffffffu, mine.a, l);
            if (ln == 0) starts[c0 + l] = S;
            S = s - a + dd;
            ++done;
        }
    }
    __syncwarp();
    if (ln == 0) {
        st->i = S;
        st->pos = pos0 + done * T;
        st->done = done;
    }
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
__global__ void fy_count_kernel(const int32_t* __restrict__ j, int64_t n, int32_t* first,
                                int32_t* gcount) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; s < n;
         s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = j[s];
        if (p < s) {
            atomicMin(&first[p], (int32_t)s);
            atomicAdd(&gcount[p], 1);
        }
    }
}

__global__ void fy_scatter_kernel(const int32_t* __restrict__ j, int64_t n,
                                  const int32_t* __restrict__ goff, int32_t* cursor,
                                  int32_t* members) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; s < n;
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

__global__ void fy_final_kernel(const int32_t* __restrict__ j, int64_t n, int64_t L,
                                const int32_t* __restrict__ tail,
                                const int32_t* __restrict__ first,
                                const int32_t* __restrict__ goff,
                                const int32_t* __restrict__ members, int32_t* bucket) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
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
                out = best == kNone ? slot_value(p, L, tail) : incoming(best, first, L, tail);
            }
        }
        bucket[i] = out;
    }
}

struct HashPlan {
    int64_t I, L;
    int surj;
    int64_t n_acc, n_cand, nblk, nbuf;
    int64_t max_chunks;
    size_t scan_bytes, scan2_bytes;
};

constexpr int kMinBand = 15;  // bands below 2^15 are walked exactly by one warp

// Chunk length for band k: ~8 expected near-miss events per chunk.
int64_t band_chunk(int k) {
    const double want = 2.3 * pow(2.0, 0.5 * k);
    int64_t T = 256;
    while (T < want && T < 4096) T <<= 1;
    return T;
}

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
           int32_t** gcount, int32_t** goff, int32_t** members, FyState** fst, FyChunk** chunks,
           int64_t** starts) {
    *blk_cnt = ws.template take<int64_t>(p.nblk);
    *blk_off = ws.template take<int64_t>(p.nblk);
    *scal = ws.template take<int64_t>(4);
    *scan_tmp = ws.template take<char>(p.scan_bytes > p.scan2_bytes ? p.scan_bytes
                                                                      : p.scan2_bytes);
    if (p.surj) {
        *tail = ws.template take<int32_t>(p.I - p.L + 1);
        *draws = ws.template take<uint32_t>(p.nbuf);
        *jarr = ws.template take<int32_t>(p.I + 1);
        *first = ws.template take<int32_t>(p.I + 1);
        *gcount = ws.template take<int32_t>(p.I + 1);
        *goff = ws.template take<int32_t>(p.I + 1);
        *members = ws.template take<int32_t>(p.I + 1);
        *fst = ws.template take<FyState>(1);
        *chunks = ws.template take<FyChunk>(p.max_chunks);
        *starts = ws.template take<int64_t>(p.max_chunks + 1);
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
    int32_t *e, *g, *h, *i2, *j2, *k2;
    uint32_t* f;
    FyState* fs;
    FyChunk* fc;
    int64_t* sts;
    carve(nc, p, &a, &b, &c, &d, &e, &f, &g, &h, &i2, &j2, &k2, &fs, &fc, &sts);
    return nc.off + 256;
}

extern "C" int ids_countsketch_hash(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                                    uint64_t inc_lo, int64_t in_dim, int64_t out_dim,
                                    int surjective, int32_t* bucket, int8_t* sign,
                                    int64_t* draws_out, void* workspace, size_t ws_bytes,
                                    void* stream) {
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
    int32_t *tail = nullptr, *jarr = nullptr, *first = nullptr, *gcount = nullptr,
            *goff = nullptr, *members = nullptr;
    uint32_t* draws = nullptr;
    FyState* fst = nullptr;
    FyChunk* chunks = nullptr;
    int64_t* starts = nullptr;
    carve(ws, p, &blk_cnt, &blk_off, &scal, &scan_tmp, &tail, &draws, &jarr, &first, &gcount,
          &goff, &members, &fst, &chunks, &starts);
    if (!ws.ok()) {
        ids_set_last_error("hash: workspace too small");
        return IDS_EWORKSPACE;
    }
    int64_t* d = draws_out ? draws_out : scal;
    IDS_CUDA_TRY(cudaMemsetAsync(d, 0, 4 * sizeof(int64_t), st));
    Seed sd{state_hi, state_lo, inc_hi, inc_lo};
    const uint32_t L = (uint32_t)out_dim;
    const uint32_t thresh = L > 1 ? (uint32_t)(0u - L) % L : 0u;
    int32_t* phaseA_out = surjective ? tail : bucket;

    // ---- phase A / A': Lemire draws in [0, L) ----
    if (p.n_acc > 0) {
        if (L == 1) {  // numpy draws nothing for a single-value range
            fill_i32_kernel<<<1024, 256, 0, st>>>(phaseA_out, p.n_acc, 0);
            IDS_LAUNCH_CHECK();
        } else {
            lemire_count_kernel<<<(unsigned)p.nblk, kGenThreads, 0, st>>>(sd, p.n_cand, L,
                                                                         thresh, blk_cnt);
            IDS_LAUNCH_CHECK();
            size_t sb = p.scan_bytes;
            IDS_CUDA_TRY(cub::DeviceScan::ExclusiveSum(scan_tmp, sb, blk_cnt, blk_off,
                                                       (int)p.nblk, st));
            lemire_write_kernel<<<(unsigned)p.nblk, kGenThreads, 0, st>>>(
                sd, p.n_cand, L, thresh, blk_off, p.n_acc, phaseA_out, d + 0);
            IDS_LAUNCH_CHECK();
        }
    }

    // ---- phase B: Fisher-Yates over slots ----
    if (surjective) {
        const int64_t I = in_dim;
        const unsigned gb = (unsigned)ceil_div(p.nbuf, (int64_t)kGenThreads * kChunk);
        raw_draws_kernel<<<gb, kGenThreads, 0, st>>>(sd, d, 1, p.nbuf, draws);
        IDS_LAUNCH_CHECK();
        fy_init_kernel<<<1, 1, 0, st>>>(fst, I);
        IDS_LAUNCH_CHECK();
        int top = 0;
        while ((2LL << top) <= I - 1) ++top;  // band of i = I - 1
        for (int k = top; k >= kMinBand && I > 1; --k) {
            const int64_t lo_band = 1LL << k;
            const int64_t i0 = tmin<int64_t>(2 * lo_band - 1, I - 1);
            if (i0 < lo_band) continue;
            const int64_t T = band_chunk(k);
            const double draws_est = (double)(2 * lo_band) * log((double)(i0 + 1) / (double)lo_band);
            const int64_t nch = tmin<int64_t>((int64_t)(draws_est / (double)T) + 2, p.max_chunks);
            if (nch >= 2) {
                const unsigned gb = (unsigned)ceil_div(nch, 128);
                fy_chunk_kernel<<<gb, 128, 0, st>>>(draws, p.nbuf, fst, i0, lo_band, T, nch, chunks);
                IDS_LAUNCH_CHECK();
                fy_stitch_kernel<<<1, 32, 0, st>>>(fst, chunks, nch, T, starts + 1);
                IDS_LAUNCH_CHECK();
                fy_chunk_exact_kernel<<<gb, 128, 0, st>>>(draws, fst, starts + 1, lo_band, T, jarr, 0);
                IDS_LAUNCH_CHECK();
            }
            fy_walk_kernel<<<1, 32, 0, st>>>(draws, p.nbuf, lo_band - 1, jarr, fst, d + 1, d + 3);
            IDS_LAUNCH_CHECK();
        }
        fy_walk_kernel<<<1, 32, 0, st>>>(draws, p.nbuf, 0, jarr, fst, d + 1, d + 3);
        IDS_LAUNCH_CHECK();
        if (I > 1) {
            fill_i32_kernel<<<1024, 256, 0, st>>>(first, I, kNone);
            IDS_LAUNCH_CHECK();
            IDS_CUDA_TRY(cudaMemsetAsync(gcount, 0, sizeof(int32_t) * (I + 1), st));
            const unsigned grid = (unsigned)tmin<int64_t>(ceil_div(I, 256), 148 * 16);
            fy_count_kernel<<<grid, 256, 0, st>>>(jarr, I, first, gcount);
            IDS_LAUNCH_CHECK();
            size_t sb = p.scan2_bytes;
            IDS_CUDA_TRY(
                cub::DeviceScan::ExclusiveSum(scan_tmp, sb, gcount, goff, (int)(I + 1), st));
            IDS_CUDA_TRY(cudaMemsetAsync(gcount, 0, sizeof(int32_t) * (I + 1), st));
            fy_scatter_kernel<<<grid, 256, 0, st>>>(jarr, I, goff, gcount, members);
            IDS_LAUNCH_CHECK();
            fy_final_kernel<<<grid, 256, 0, st>>>(jarr, I, out_dim, tail, first, goff,
                                                   members, bucket);
            IDS_LAUNCH_CHECK();
        } else {
            fill_i32_kernel<<<1, 32, 0, st>>>(bucket, 1, 0);
            IDS_LAUNCH_CHECK();
        }
    }

    // ---- signs ----
    {
        const unsigned gb = (unsigned)ceil_div(in_dim, (int64_t)kGenThreads * kChunk);
        sign_kernel<<<gb, kGenThreads, 0, st>>>(sd, d, 2, in_dim, sign);
        IDS_LAUNCH_CHECK();
        set_i64_kernel<<<1, 1, 0, st>>>(d + 2, in_dim);
        IDS_LAUNCH_CHECK();
    }
    return IDS_OK;
}
