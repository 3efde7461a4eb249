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

enum { ST_DONE = 0, ST_ACC = 1, ST_REJ = 2, ST_AMB = 3 };

__device__ __forceinline__ int classify(uint32_t x, int64_t i, int64_t u, uint32_t* v) {
    const int64_t lo = i - u;
    const uint32_t m = mask_of((uint32_t)i);
    if (lo < 1 || mask_of((uint32_t)lo) != m) return ST_AMB;
    *v = x & m;
    if ((int64_t)*v <= lo) return ST_ACC;
    if ((int64_t)*v > i) return ST_REJ;
    return ST_AMB;
}

// Phase B accept/reject chain.  g: the phase-B draw stream (nbuf draws).
// Writes jout[i] for i = n-1..1 and the number of draws consumed.
__global__ void __launch_bounds__(1024, 1) fy_scan_kernel(const uint32_t* __restrict__ g,
                                                          int64_t nbuf, int64_t n,
                                                          int32_t* __restrict__ jout,
                                                          int64_t* consumed, int64_t* status) {
    __shared__ uint32_t s_acc[32], s_amb[32];
    __shared__ int s_pref[32];
    __shared__ int s_tamb, s_A, s_done;
    __shared__ int64_t s_i, s_cons;
    const int t = threadIdx.x, w = t >> 5, ln = t & 31;
    const uint32_t lt_mask = (1u << ln) - 1u;
    if (n <= 1) {
        if (t == 0) *consumed = 0;
        return;
    }
    int64_t i = n - 1;
    int64_t pos = 0;
    if (t == 0) s_done = 0;
    __syncthreads();
    // ---------------- block regime: 1024 draws per window -----------------
    uint32_t x_next = (pos + t < nbuf) ? g[pos + t] : 0u;
    while (i >= (int64_t)kBlockMin) {
        if (pos + 1024 > nbuf) {
            if (t == 0) *status = IDS_ERETRY;
            return;
        }
        const uint32_t x = x_next;
        x_next = (pos + 1024 + t < nbuf) ? g[pos + 1024 + t] : 0u;
        int b = 0;
        while (b < 1024) {
            uint32_t v = 0;
            const int st = (t >= b) ? classify(x, i, t - b, &v) : ST_DONE;
            const uint32_t accb = __ballot_sync(0xffffffffu, st == ST_ACC);
            const uint32_t ambb = __ballot_sync(0xffffffffu, st == ST_AMB);
            if (ln == 0) {
                s_acc[w] = accb;
                s_amb[w] = ambb;
            }
            __syncthreads();
            if (w == 0) {
                const uint32_t a = s_acc[ln], am = s_amb[ln];
                const uint32_t anyamb = __ballot_sync(0xffffffffu, am != 0u);
                const int fw = anyamb ? __ffs(anyamb) - 1 : 32;
                const int tamb = fw < 32 ? fw * 32 + __ffs(__shfl_sync(0xffffffffu, am, fw)) - 1
                                         : 1024;
                int cnt;
                if (ln < fw) cnt = __popc(a);
                else if (ln == fw) cnt = __popc(a & ((1u << (tamb & 31)) - 1u));
                else cnt = 0;
                int inc = cnt;
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, inc, o);
                    if (ln >= o) inc += y;
                }
                s_pref[ln] = inc - cnt;
                if (ln == 31) {
                    s_A = inc;
                    s_tamb = tamb;
                }
            }
            __syncthreads();
            const int tamb = s_tamb, A = s_A;
            if (st == ST_ACC && t < tamb) {
                const int a_t = s_pref[w] + __popc(accb & lt_mask);
                jout[i - a_t] = (int32_t)v;
            }
            if (tamb == 1024) {
                i -= A;
                break;
            }
            if (t == tamb) {
                int64_t is = i - A;
                if (is < 1) {
                    s_done = 1;
                    s_cons = pos + tamb;
                } else {
                    const uint32_t vv = x & mask_of((uint32_t)is);
                    if ((int64_t)vv <= is) {
                        jout[is] = (int32_t)vv;
                        --is;
                    }
                    s_i = is;
                    if (is == 0) {
                        s_done = 1;
                        s_cons = pos + tamb + 1;
                    }
                }
            }
            __syncthreads();
            if (s_done) {
                if (t == 0) *consumed = s_cons;
                return;
            }
            i = s_i;
            b = tamb + 1;
        }
        pos += 1024;
    }
    // ---------------- warp regime: 32 draws per window ---------------------
    if (w != 0) return;
    for (;;) {
        if (pos >= nbuf) {
            if (ln == 0) *status = IDS_ERETRY;
            return;
        }
        uint32_t xs[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const int64_t p = pos + 32 * k + ln;
            xs[k] = p < nbuf ? g[p] : 0u;
        }
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const uint32_t x = xs[k];
            int b = 0;
            while (b < 32) {
                uint32_t v = 0;
                const int st = (ln >= b) ? classify(x, i, ln - b, &v) : ST_DONE;
                const uint32_t accb = __ballot_sync(0xffffffffu, st == ST_ACC);
                const uint32_t ambb = __ballot_sync(0xffffffffu, st == ST_AMB);
                const int tamb = ambb ? __ffs(ambb) - 1 : 32;
                const uint32_t before = tamb < 32 ? (accb & ((1u << tamb) - 1u)) : accb;
                if (st == ST_ACC && ln < tamb) jout[i - __popc(before & lt_mask)] = (int32_t)v;
                const int A = __popc(before);
                if (tamb == 32) {
                    i -= A;
                    break;
                }
                int64_t is = i - A;
                const uint32_t xa = __shfl_sync(0xffffffffu, x, tamb);
                if (is < 1) {
                    if (ln == 0) *consumed = pos + 32 * k + tamb;
                    return;
                }
                const uint32_t vv = xa & mask_of((uint32_t)is);
                if ((int64_t)vv <= is) {
                    if (ln == 0) jout[is] = (int32_t)vv;
                    --is;
                }
                if (is == 0) {
                    if (ln == 0) *consumed = pos + 32 * k + tamb + 1;
                    return;
                }
                i = is;
                b = tamb + 1;
            }
        }
        pos += 1024;
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
    size_t scan_bytes, scan2_bytes;
};

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
           int32_t** gcount, int32_t** goff, int32_t** members) {
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
    carve(nc, p, &a, &b, &c, &d, &e, &f, &g, &h, &i2, &j2, &k2);
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
    carve(ws, p, &blk_cnt, &blk_off, &scal, &scan_tmp, &tail, &draws, &jarr, &first, &gcount,
          &goff, &members);
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
        fy_scan_kernel<<<1, 1024, 0, st>>>(draws, p.nbuf, I, jarr, d + 1, d + 3);
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
