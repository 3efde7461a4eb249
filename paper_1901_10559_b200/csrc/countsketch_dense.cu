// Dense CountSketch Y = S @ A on B200 (replaces reference sketch.py:119 for
// dense A: scipy csr_matvecs over the CSR operator built at sketch.py:108-114).
//
// Row-major A (the numpy default):  bucket-gather kernel.  One warp owns one
// (bucket l, 64-column chunk) unit and walks the rows of bucket l in
// increasing row order (the bucket index), streaming each row segment with
// 16-byte loads and accumulating in registers.  A is read exactly once, with
// no atomics and no shared memory; the per-entry summation order is scipy's,
// so Y is bit-identical to the reference when each bucket is one segment.
//
// Col-major A (Fortran order, what the reference's as_dense produces):
// tiled kernels over 512-row tiles whose rows a pre-pass sorts by bucket
// (cs_coltile_ra_kernel: producer warp + bulk copies, register running sums;
// cs_coltile_kernel: 32 slots with shared-memory sums for L > 512), and a
// column-stream fallback (one warp per NC columns and a row segment, lanes
// ordered per bucket with __match_any_sync ranks).  Every path adds each Y
// entry's terms in increasing row order.
//
// Both paths are HBM-streaming kernels (algorithmic traffic = bytes of A);
// tensor cores have nothing to do here.
#include <limits.h>
#include <stdlib.h>

#include "common.cuh"

namespace {

constexpr int kWarpsPerBlock = 8;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ int64_t lower_bound_rows(const int32_t* __restrict__ order,
                                                    int64_t lo, int64_t hi, int64_t row) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)dec_row(order[mid]) < row) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <int VEC>
struct VecT;
template <>
struct VecT<1> {
    typedef double T;
    static __device__ __forceinline__ void load(const double* p, double* v) { v[0] = __ldcs(p); }
};
template <>
struct VecT<2> {
    typedef double2 T;
    static __device__ __forceinline__ void load(const double* p, double* v) {
        const double2 x = __ldcs(reinterpret_cast<const double2*>(p));
        v[0] = x.x;
        v[1] = x.y;
    }
};

// unit = ((l * nseg + seg) * nchunks + chunk); one warp per unit.
template <int VEC, int UNR>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    cs_rowmajor_kernel(const double* __restrict__ A, int64_t ld, int64_t cols, int64_t row0,
                       int64_t rows, int restrict_rows, const int32_t* __restrict__ order,
                       const int64_t* __restrict__ bstart, int64_t L, int nchunks, int nseg,
                       double* __restrict__ out, int64_t seg_stride, int init_from_out) {
    const int64_t gw = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (gw >= L * nchunks * nseg) return;
    const int chunk = (int)(gw % nchunks);
    const int64_t t = gw / nchunks;
    const int seg = (int)(t % nseg);
    const int64_t l = t / nseg;

    int64_t k0 = bstart[l], k1 = bstart[l + 1];
    if (restrict_rows) {
        const int64_t a = lower_bound_rows(order, k0, k1, row0);
        k1 = lower_bound_rows(order, a, k1, row0 + rows);
        k0 = a;
    }
    const int64_t len = k1 - k0;
    const int64_t s0 = k0 + len * seg / nseg, s1 = k0 + len * (seg + 1) / nseg;

    const int64_t c = (int64_t)chunk * 32 * VEC + (int64_t)lane * VEC;
    const bool valid = c < cols;
    double acc[VEC];
    double* o = out + (int64_t)seg * seg_stride;
#pragma unroll
    for (int v = 0; v < VEC; ++v)
        acc[v] = (init_from_out && valid && c + v < cols) ? o[(c + v) * L + l] : 0.0;

    // lanes past the last column read a valid column (results discarded) so
    // that the hot loop is branch-free and all loads of a batch are in flight
    const int64_t cl = valid ? c : (cols - VEC);
    const double* Abase = A + cl - row0 * ld;
    int64_t kb = s0;
    for (; kb + 32 <= s1; kb += 32) {  // full batches: 32 rows, two rounds of 16 loads
        const int32_t e = __ldg(order + kb + lane);
#pragma unroll
        for (int h = 0; h < 32; h += UNR) {
            double x[UNR][VEC];
            int32_t ev[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                ev[u] = __shfl_sync(kFull, e, h + u);
                VecT<VEC>::load(Abase + (int64_t)dec_row(ev[u]) * ld, x[u]);
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
#pragma unroll
                for (int v = 0; v < VEC; ++v)
                    acc[v] = ev[u] >= 0 ? acc[v] + x[u][v] : acc[v] - x[u][v];
            }
        }
    }
    if (kb < s1) {  // tail batch (< 32 rows), in order
        const int n = (int)(s1 - kb);
        const int32_t e = lane < n ? __ldg(order + kb + lane) : 0;
        for (int u = 0; u < n; ++u) {
            const int32_t ev = __shfl_sync(kFull, e, u);
            double x[VEC];
            VecT<VEC>::load(Abase + (int64_t)dec_row(ev) * ld, x);
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[v] = ev >= 0 ? acc[v] + x[v] : acc[v] - x[v];
        }
    }
    if (valid) {
#pragma unroll
        for (int v = 0; v < VEC; ++v)
            if (c + v < cols) o[(c + v) * L + l] = acc[v];
    }
}

// unit = seg * ngroups + group; one warp per unit; per-warp acc NC x L.
template <int NC, int UNR>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    cs_colmajor_kernel(const double* __restrict__ A, int64_t ld, int64_t rows, int64_t cols,
                       int64_t row0, const int32_t* __restrict__ bucket,
                       const int8_t* __restrict__ sign, int64_t L, int ngroups, int nseg,
                       int warps_per_block, double* __restrict__ out, int64_t seg_stride,
                       int init_from_out, double* __restrict__ gacc) {
    extern __shared__ double smem_acc[];
    const int wib = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (wib >= warps_per_block) return;
    const int64_t gw = (int64_t)blockIdx.x * warps_per_block + wib;
    if (gw >= (int64_t)ngroups * nseg) return;
    const int group = (int)(gw % ngroups);
    const int seg = (int)(gw / ngroups);
    double* acc = gacc ? gacc + gw * (int64_t)NC * L : smem_acc + (int64_t)wib * NC * L;
    const int64_t c0 = (int64_t)group * NC;
    const int nc = (int)tmin<int64_t>(NC, cols - c0);
    double* o = out + (int64_t)seg * seg_stride;
    for (int64_t q = lane; q < (int64_t)NC * L; q += 32) {
        const int64_t qc = q / L, ql = q % L;
        acc[q] = (init_from_out && qc < nc) ? o[(c0 + qc) * L + ql] : 0.0;
    }
    __syncwarp();
    const int64_t r0 = rows * seg / nseg, r1 = rows * (seg + 1) / nseg;
    const uint32_t lt = (1u << lane) - 1u;
    for (int64_t rb = r0; rb < r1; rb += 32 * UNR) {
        int32_t h[UNR];
        int8_t s[UNR];
        double x[UNR][NC];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int64_t i = rb + u * 32 + lane;
            const bool act = i < r1;
            h[u] = act ? __ldg(bucket + row0 + i) : -1;
            s[u] = act ? __ldg(sign + row0 + i) : (int8_t)1;
#pragma unroll
            for (int q = 0; q < NC; ++q)
                x[u][q] = (act && q < nc) ? __ldcs(A + (c0 + q) * ld + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint32_t peers = __match_any_sync(kFull, h[u]);
            const int rank = __popc(peers & lt);
            const int maxr = (int)__reduce_max_sync(kFull, (unsigned)(h[u] >= 0 ? rank : 0));
            for (int rr = 0; rr <= maxr; ++rr) {
                if (h[u] >= 0 && rank == rr) {
#pragma unroll
                    for (int q = 0; q < NC; ++q) {
                        double* p = acc + (int64_t)q * L + h[u];
                        *p = s[u] > 0 ? *p + x[u][q] : *p - x[u][q];
                    }
                }
                __syncwarp();
            }
        }
    }
    __syncwarp();
    for (int64_t q = lane; q < (int64_t)nc * L; q += 32) {
        const int64_t qc = q / L, ql = q % L;
        o[(c0 + qc) * L + ql] = acc[q];
    }
}

// ---- column-major tiled kernel (F-order A, the reference's as_dense layout) ----
// Rows are cut into tiles of kTT.  A pre-pass (tile_slot_lists_kernel) sorts
// each tile's rows ONCE by owner slot (bucket mod kSlots; stable, so every
// slot's list is in increasing row order), packing (bucket, sign, tile row)
// into one int32 per row.  The sketch kernel gives each CTA at most kCt
// columns and a row segment (all rows when ordered); its 256 threads form
// kSlots slots of kCt lanes, slot x owning the buckets l = x (mod kSlots).
// Tile after tile -- A's column runs, the lists and the slot starts arriving
// through a kCtStages-deep cp.async pipeline -- each slot walks its list and
// every lane adds its column into acc[l][c], an accumulator no other slot
// touches.  Each Y entry is therefore summed in increasing row order from
// +0.0 (scipy's order, bit for bit) while A streams once at full width.
constexpr int kCtThreads = 256;
constexpr int kCt = 8;                       // columns per CTA (lanes per slot)
constexpr int kSlots = kCtThreads / kCt;     // 32
constexpr int kTT = 512;                     // rows per tile
constexpr int kTTp = kTT + 2;                // padded column stride in shared memory
constexpr int kStartsStride = 36;            // int32 slot starts per tile (kSlots + 1, 16-byte padded)
constexpr int kCtStages = 3;

__global__ void row_codes_kernel(const int32_t* __restrict__ bucket, const int8_t* __restrict__ sign,
                                 int64_t row0, int64_t rows, int32_t* __restrict__ codes) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
         r += (int64_t)gridDim.x * blockDim.x)
        codes[r] = enc_row(bucket[row0 + r], sign[row0 + r]);
}

// One CTA per tile: lists[tile][q] = (bucket << 10 | negative << 9 | row in
// tile), grouped by slot in increasing row order; starts[tile][x] = first q
// of slot x (x = 0..kSlots).
__global__ void __launch_bounds__(kCtThreads) tile_slot_lists_kernel(
    const int32_t* __restrict__ codes, int64_t rows, int32_t* __restrict__ lists,
    int32_t* __restrict__ starts) {
    constexpr int kRpt = kTT / kCtThreads, kGroups = kTT / 32, kWarps = kCtThreads / 32;
    __shared__ int s_cnt[kGroups][kSlots + 1];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t rb = (int64_t)blockIdx.x * kTT;
    const int n = (int)tmin<int64_t>(kTT, rows - rb);
    const uint32_t lt = (1u << lane) - 1u;
    int sl2[kRpt], rank2[kRpt], ent2[kRpt];
#pragma unroll
    for (int h = 0; h < kRpt; ++h) {
        const int g = warp + kWarps * h, r = 32 * g + lane;
        const int32_t e = r < n ? codes[rb + r] : INT_MIN;
        const int sl = e == INT_MIN ? kSlots : (dec_row(e) % kSlots);
        ent2[h] = (dec_row(e) << 10) | (e < 0 ? 512 : 0) | r;
        const uint32_t peers = __match_any_sync(0xffffffffu, sl);
        const int rank = __popc(peers & lt);
        for (int x = lane; x <= kSlots; x += 32) s_cnt[g][x] = 0;
        __syncwarp();
        if (rank == 0) s_cnt[g][sl] = __popc(peers);
        sl2[h] = sl;
        rank2[h] = rank;
    }
    __syncthreads();
    if (warp == 0) {  // lane = slot (kSlots == 32): bases per (group, slot), slot starts
        int tot = 0;
        for (int g = 0; g < kGroups; ++g) tot += s_cnt[g][lane];
        int incl = tot;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += y;
        }
        int run = incl - tot;
        starts[blockIdx.x * (int64_t)kStartsStride + lane] = run;
        if (lane == 31) {
            starts[blockIdx.x * (int64_t)kStartsStride + kSlots] = incl;
            for (int x = kSlots + 1; x < kStartsStride; ++x)
                starts[blockIdx.x * (int64_t)kStartsStride + x] = incl;
        }
        for (int g = 0; g < kGroups; ++g) {
            const int cg = s_cnt[g][lane];
            s_cnt[g][lane] = run;
            run += cg;
        }
    }
    __syncthreads();
#pragma unroll
    for (int h = 0; h < kRpt; ++h) {
        const int g = warp + kWarps * h;
        if (sl2[h] < kSlots) lists[rb + s_cnt[g][sl2[h]] + rank2[h]] = ent2[h];
    }
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

constexpr size_t kCtStageBytes =
    (size_t)kCt * kTTp * sizeof(double) + kTT * sizeof(int32_t) + kStartsStride * sizeof(int32_t);

size_t coltile_smem(int64_t L) { return (size_t)L * kCt * sizeof(double) + kCtStages * kCtStageBytes; }

__global__ void __launch_bounds__(kCtThreads) cs_coltile_kernel(
    const double* __restrict__ A, int64_t ld, int64_t rows, int64_t cols,
    const int32_t* __restrict__ lists, const int32_t* __restrict__ starts, int64_t L,
    int ngroups, int nseg, int vec16, double* __restrict__ out, int64_t seg_stride,
    int init_from_out) {
    extern __shared__ double sm[];
    double* acc = sm;  // [L][kCt]
    char* stages = reinterpret_cast<char*>(acc + L * kCt);
    const int t = threadIdx.x;
    const int group = blockIdx.x % ngroups, seg = blockIdx.x / ngroups;
    // column groups of at most kCt columns, balanced (ngroups >= cols / kCt)
    const int64_t c0 = cols * group / ngroups;
    const int nc = (int)(cols * (group + 1) / ngroups - c0);
    // segment rows: boundaries on tile multiples (tile bases stay aligned)
    const int64_t ntl = (rows + kTT - 1) / kTT;
    const int64_t tb = ntl * seg / nseg, te = ntl * (seg + 1) / nseg;
    double* o = out + (int64_t)seg * seg_stride;
    for (int64_t q = t; q < L * kCt; q += kCtThreads) {
        const int64_t l = q / kCt, c = q % kCt;
        acc[q] = (init_from_out && c < nc) ? o[(c0 + c) * L + l] : 0.0;
    }
    auto stage_tile = [&](int s) { return reinterpret_cast<double*>(stages + s * kCtStageBytes); };
    auto stage_list = [&](int s) {
        return reinterpret_cast<int32_t*>(stages + s * kCtStageBytes + (size_t)kCt * kTTp * sizeof(double));
    };
    auto stage_starts = [&](int s) { return stage_list(s) + kTT; };
    // copy tile k (k = 0 .. te - tb - 1) into stage k % kCtStages
    auto issue = [&](int64_t k) {
        const int64_t tile = tb + k;
        if (tile < te) {
            const int64_t rb = tile * kTT;
            const int n = (int)tmin<int64_t>(kTT, rows - rb);
            const int s = (int)(k % kCtStages);
            double* dst = stage_tile(s);
            if (vec16 && n == kTT) {
                static_assert(kTT / 2 == kCtThreads, "one 16-byte copy per thread and column");
                const double* src = A + c0 * ld + rb + 2 * t;
#pragma unroll
                for (int c = 0; c < kCt; ++c, src += ld)
                    if (c < nc) cp_async16(dst + c * kTTp + 2 * t, src);
            } else {
                for (int q = t; q < kCt * kTT; q += kCtThreads) {
                    const int c = q / kTT, j = q % kTT;
                    if (c < nc && j < n) cp_async8(dst + c * kTTp + j, A + (c0 + c) * ld + rb + j);
                }
            }
            int32_t* ldst = stage_list(s);
            for (int q = t; q < kTT / 4 + kStartsStride / 4; q += kCtThreads) {
                if (q < kTT / 4) cp_async16(ldst + 4 * q, lists + rb + 4 * q);
                else cp_async16(stage_starts(s) + 4 * (q - kTT / 4),
                                starts + tile * kStartsStride + 4 * (q - kTT / 4));
            }
        }
        cp_commit();
    };
    for (int64_t k = 0; k < kCtStages - 1; ++k) issue(k);
    const int slot = t / kCt, c = t % kCt;
    for (int64_t k = 0; k < te - tb; ++k) {
        issue(k + kCtStages - 1);
        cp_wait<kCtStages - 1>();
        __syncthreads();
        const int s = (int)(k % kCtStages);
        const double* tl = stage_tile(s);
        const int32_t* lst = stage_list(s);
        const int32_t* sts = stage_starts(s);
        // every slot walks its own rows; its lanes own one column each.  Two
        // rows per step: independent unless they share a bucket.
        if (c < nc) {
            const int q1 = sts[slot + 1];
            int q = sts[slot];
            for (; q + 1 < q1; q += 2) {
                const int32_t e0 = lst[q], e1 = lst[q + 1];
                const double v0 = tl[c * kTTp + (e0 & 511)], v1 = tl[c * kTTp + (e1 & 511)];
                const int b0 = e0 >> 10, b1 = e1 >> 10;
                double* p0 = acc + (int64_t)b0 * kCt + c;
                double a0 = *p0;
                a0 = (e0 & 512) ? a0 - v0 : a0 + v0;
                if (b0 == b1) {
                    a0 = (e1 & 512) ? a0 - v1 : a0 + v1;
                    *p0 = a0;
                } else {
                    double* p1 = acc + (int64_t)b1 * kCt + c;
                    const double a1 = *p1;
                    *p0 = a0;
                    *p1 = (e1 & 512) ? a1 - v1 : a1 + v1;
                }
            }
            if (q < q1) {
                const int32_t e0 = lst[q];
                const double v0 = tl[c * kTTp + (e0 & 511)];
                double* p0 = acc + (int64_t)(e0 >> 10) * kCt + c;
                *p0 = (e0 & 512) ? *p0 - v0 : *p0 + v0;
            }
        }
        __syncthreads();  // the stage is refilled by a later issue()
    }
    cp_wait<0>();
    __syncthreads();
    for (int64_t q = t; q < L * kCt; q += kCtThreads) {
        const int64_t l = q % L, cc = q / L;  // consecutive threads: consecutive l (coalesced Y)
        if (cc < nc) o[(c0 + cc) * L + l] = acc[l * kCt + cc];
    }
}

// ---- column-major tiled kernel, register accumulators ----
// The same tile pipeline, but every tile's rows are sorted by BUCKET (stable,
// so each bucket's run is in increasing row order) and each (slot, column)
// lane owns BPL buckets -- slot x owns x, x + nslots, ... with nslots =
// ceil(L / BPL) -- whose running sums stay in registers: per tile the lane
// walks its buckets' runs one after the other.  Per element that is one list
// load, one tile load, a sign flip on the high word and one DADD; the
// per-tile time is the longest slot (~kTT * BPL / L rows) instead of the
// 32-slot layout's (whose L = 100 slots 0..3 own 4 buckets and the rest 3).
// Order per Y entry: increasing row from +0.0 (or from Y when accumulating),
// so Y is bit-identical to the 32-slot kernel's and to scipy's.
constexpr int kRaMaxBuckets = 512;

// One CTA per TT-row tile: lists[tile][q] = 8 * row in tile | sign << 31, grouped
// by bucket in increasing row order; starts[tile * ss + b] = first q of
// bucket b (b = 0..L), padded with the tile's total up to ss.
template <int TT>
__global__ void __launch_bounds__(kCtThreads) tile_bucket_lists_kernel(
    const int32_t* __restrict__ codes, int64_t rows, int nb, int ss,
    int32_t* __restrict__ lists, int32_t* __restrict__ starts) {
    constexpr int kRpt = TT / kCtThreads, kGroups = TT / 32, kWarps = kCtThreads / 32;
    constexpr int kPerLane = kRaMaxBuckets / 32;
    static_assert(TT % kCtThreads == 0 && TT <= 512, "rows per tile");
    __shared__ int s_cnt[kGroups][kRaMaxBuckets + 1];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t rb = (int64_t)blockIdx.x * TT;
    const int n = (int)tmin<int64_t>(TT, rows - rb);
    const uint32_t lt = (1u << lane) - 1u;
    int b2[kRpt], rank2[kRpt], ent2[kRpt];
#pragma unroll
    for (int h = 0; h < kRpt; ++h) {
        const int g = warp + kWarps * h, r = 32 * g + lane;
        const int32_t e = r < n ? codes[rb + r] : INT_MIN;
        const int b = e == INT_MIN ? nb : (int)dec_row(e);
        ent2[h] = (e < 0 ? (int)0x80000000u : 0) | (r << 3);  // byte offset of the row
        const uint32_t peers = __match_any_sync(0xffffffffu, b);
        const int rank = __popc(peers & lt);
        for (int x = lane; x <= nb; x += 32) s_cnt[g][x] = 0;
        __syncwarp();
        if (rank == 0) s_cnt[g][b] = __popc(peers);
        b2[h] = b;
        rank2[h] = rank;
    }
    __syncthreads();
    if (warp == 0) {  // lane owns buckets kPerLane lane .. kPerLane (lane + 1) - 1
        int sum = 0;
        for (int j = 0; j < kPerLane; ++j) {
            const int x = kPerLane * lane + j;
            if (x < nb)
                for (int g = 0; g < kGroups; ++g) sum += s_cnt[g][x];
        }
        int incl = sum;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += y;
        }
        int run = incl - sum;
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        int32_t* st = starts + blockIdx.x * (int64_t)ss;
        for (int j = 0; j < kPerLane; ++j) {
            const int x = kPerLane * lane + j;
            if (x < nb) {
                st[x] = run;
                for (int g = 0; g < kGroups; ++g) {
                    const int cg = s_cnt[g][x];
                    s_cnt[g][x] = run;
                    run += cg;
                }
            }
        }
        for (int x = nb + lane; x < ss; x += 32) st[x] = total;
    }
    __syncthreads();
#pragma unroll
    for (int h = 0; h < kRpt; ++h) {
        const int g = warp + kWarps * h;
        if (b2[h] < nb) lists[rb + s_cnt[g][b2[h]] + rank2[h]] = ent2[h];
    }
}

// stage = CT columns of a 512-row tile (padded stride) + its list + its starts
template <int CT>
__host__ __device__ __forceinline__ size_t coltile_ra_stage_bytes(int ss) {
    return (size_t)CT * kTTp * sizeof(double) + kTT * sizeof(int32_t) + (size_t)ss * sizeof(int32_t);
}

__device__ __forceinline__ uint32_t cs_smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// Needs 16-byte aligned columns (A and ld even).  Warp-specialised: the last
// warp is the producer -- per tile, one bulk copy per column (one lane each)
// plus the list and the bucket starts, against the stage's `full` mbarrier --
// and every consumer warp walks its buckets and releases the stage on its
// `empty` mbarrier, so warps drift up to kCtStages tiles apart instead of
// meeting at a CTA barrier per tile, and no consumer issues copies.  The CTA
// owns up to CT = 8 * CPL columns; lane (slot, c) adds into columns c, c + 8,
// .. (CPL of them), so one list entry's decode serves CPL columns.
template <int BPL, int CPL>
__global__ void __launch_bounds__(512 + 32, CPL == 1 ? 2 : 1) cs_coltile_ra_kernel(
    const double* __restrict__ A, int64_t ld, int64_t rows, int64_t cols,
    const int32_t* __restrict__ lists, const int32_t* __restrict__ starts, int64_t L, int nslots,
    int ss, int ngroups, double* __restrict__ out, int init_from_out) {
    constexpr int S = kCtStages, CT = kCt * CPL;
    extern __shared__ __align__(16) char ra_stages[];
    __shared__ __align__(8) uint64_t s_full[S], s_empty[S];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int ncw = (int)(blockDim.x >> 5) - 1;  // consumer warps; warp ncw produces
    const int group = blockIdx.x;
    const int64_t c0 = cols * group / ngroups;
    const int nc = (int)(cols * (group + 1) / ngroups - c0);
    const int64_t ntl = (rows + kTT - 1) / kTT;
    const size_t stage_bytes = coltile_ra_stage_bytes<CT>(ss);
    auto stage_tile = [&](int s) { return reinterpret_cast<double*>(ra_stages + s * stage_bytes); };
    auto stage_list = [&](int s) {
        return reinterpret_cast<int32_t*>(ra_stages + s * stage_bytes + (size_t)CT * kTTp * sizeof(double));
    };
    auto stage_starts = [&](int s) { return stage_list(s) + kTT; };
    auto wait = [&](uint64_t* mb, uint32_t parity) {
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "RA_WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra RA_WAIT_%=;\n}" ::"r"(cs_smem_addr(mb)),
            "r"(parity)
            : "memory");
    };
    if (t == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cs_smem_addr(&s_full[s])) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(cs_smem_addr(&s_empty[s])), "r"(ncw)
                         : "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    if (warp == ncw) {  // ---- producer ----
        for (int64_t k = 0; k < ntl; ++k) {
            const int s = (int)(k % S);
            if (k >= S) wait(&s_empty[s], (uint32_t)((k / S - 1) & 1));
            const int64_t rb = k * kTT;
            const int n = (int)tmin<int64_t>(kTT, rows - rb);
            double* dst = stage_tile(s);
            const uint32_t col_bytes = (uint32_t)(n & ~1) * 8u;
            if ((n & 1) && lane < nc)  // odd last tile: its last row by plain loads
                dst[lane * kTTp + n - 1] = A[(c0 + lane) * ld + rb + n - 1];
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                                 cs_smem_addr(&s_full[s])),
                             "r"(nc * col_bytes + kTT * 4u + (uint32_t)ss * 4u)
                             : "memory");
            __syncwarp();
            const void* src = nullptr;
            void* d = nullptr;
            uint32_t bytes = 0;
            if (lane < nc) {
                src = A + (c0 + lane) * ld + rb;
                d = dst + lane * kTTp;
                bytes = col_bytes;
            } else if (lane == CT) {
                src = lists + rb;
                d = stage_list(s);
                bytes = kTT * 4u;
            } else if (lane == CT + 1) {
                src = starts + k * ss;
                d = stage_starts(s);
                bytes = (uint32_t)ss * 4u;
            }
            if (bytes)
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        cs_smem_addr(d)),
                    "l"(src), "r"(bytes), "r"(cs_smem_addr(&s_full[s]))
                    : "memory");
        }
        return;
    }

    // ---- consumers ----
    const int slot = t / kCt, c = t % kCt;
    const bool active = c < nc && slot < nslots;
    // columns c + 8 p past nc read stale shared memory into sums never written
    double acc[BPL][CPL];
#pragma unroll
    for (int j = 0; j < BPL; ++j)
#pragma unroll
        for (int p = 0; p < CPL; ++p) {
            const int64_t b = slot + (int64_t)j * nslots;
            const int cc = c + kCt * p;
            acc[j][p] = (init_from_out && active && cc < nc && b < L) ? out[(c0 + cc) * L + b] : 0.0;
        }
    auto sgn = [](int32_t e, double v) {  // v with the entry's sign applied
        return __hiloint2double(__double2hiint(v) ^ (e & (int)0x80000000u), __double2loint(v));
    };
    for (int64_t k = 0; k < ntl; ++k) {
        const int s = (int)(k % S);
        wait(&s_full[s], (uint32_t)((k / S) & 1));
        const char* tb = reinterpret_cast<const char*>(stage_tile(s) + c * kTTp);
        const int32_t* lst = stage_list(s);
        const int32_t* sts = stage_starts(s);
        // value of column c + 8 p at the entry's row
        auto at = [&](int32_t e, int p) {
            return *reinterpret_cast<const double*>(tb + (e & 0xFF8) + p * (kCt * kTTp * 8));
        };
        if (active) {
            if constexpr (BPL <= 2) {
                // the runs walked side by side: BPL x CPL independent add
                // chains per lane, as many steps as the longest run
                int q[BPL], q1[BPL];
#pragma unroll
                for (int j = 0; j < BPL; ++j) {
                    const int b = slot + j * nslots;
                    q[j] = b < L ? sts[b] : 0;
                    q1[j] = b < L ? sts[b + 1] : 0;
                }
                int steps = 0;
#pragma unroll
                for (int j = 0; j < BPL; ++j) steps = max(steps, q1[j] - q[j]);
                for (int i = 0; i < steps; ++i) {
                    int32_t e[BPL];
                    double v[BPL][CPL];
#pragma unroll
                    for (int j = 0; j < BPL; ++j) {
                        e[j] = lst[min(q[j] + i, max(q1[j] - 1, 0))];
#pragma unroll
                        for (int p = 0; p < CPL; ++p) v[j][p] = at(e[j], p);
                    }
#pragma unroll
                    for (int j = 0; j < BPL; ++j)
                        if (q[j] + i < q1[j])
#pragma unroll
                            for (int p = 0; p < CPL; ++p) acc[j][p] += sgn(e[j], v[j][p]);
                }
            } else {  // one run after the other
#pragma unroll
                for (int j = 0; j < BPL; ++j) {
                    const int b = slot + j * nslots;
                    if (b < L) {
                        int q = sts[b];
                        const int q1 = sts[b + 1];
                        for (; q + 1 < q1; q += 2) {
                            const int32_t e0 = lst[q], e1 = lst[q + 1];
                            double v0[CPL], v1[CPL];
#pragma unroll
                            for (int p = 0; p < CPL; ++p) {
                                v0[p] = at(e0, p);
                                v1[p] = at(e1, p);
                            }
#pragma unroll
                            for (int p = 0; p < CPL; ++p) {
                                acc[j][p] += sgn(e0, v0[p]);
                                acc[j][p] += sgn(e1, v1[p]);
                            }
                        }
                        if (q < q1) {
                            const int32_t e0 = lst[q];
#pragma unroll
                            for (int p = 0; p < CPL; ++p) acc[j][p] += sgn(e0, at(e0, p));
                        }
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0)  // this warp is done with the stage
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(cs_smem_addr(&s_empty[s])) : "memory");
    }
    if (active) {
#pragma unroll
        for (int j = 0; j < BPL; ++j)
#pragma unroll
            for (int p = 0; p < CPL; ++p) {
                const int64_t b = slot + (int64_t)j * nslots;
                const int cc = c + kCt * p;
                if (b < L && cc < nc) out[(c0 + cc) * L + b] = acc[j][p];
            }
    }
}

// Y[e] = (accumulate ? Y[e] : 0) + sum_s part[s][e], s in order.
__global__ void seg_reduce_kernel(const double* __restrict__ part, int nseg, int64_t n,
                                  int64_t seg_stride, double* __restrict__ Y, int accumulate) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        double acc = accumulate ? Y[e] : 0.0;
        for (int s = 0; s < nseg; ++s) acc += part[(int64_t)s * seg_stride + e];
        Y[e] = acc;
    }
}

__global__ void nonfinite_scan_kernel(const double* __restrict__ Y, int64_t n, int32_t* flag) {
    bool bad = false;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(Y[e]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
}

__global__ void dense_nonfinite_kernel(const double* __restrict__ A, int64_t outer,
                                       int64_t inner, int64_t ld, int32_t* flag) {
    bool bad = false;
    const int64_t n = outer * inner;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = e / inner, in = e % inner;
        bad |= !isfinite(A[o * ld + in]);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
}

struct DensePlan {
    int layout;
    int vec, nchunks;   // row-major
    int nc, ngroups;    // col-major
    int wpb;            // col-major warps per block
    bool global_acc;
    int nseg;
    int64_t units;
    size_t smem;
};

// warps wanted for a whole-GPU row-major launch (16 per SM) and the floor
// below which rows are split into segments (8 per SM)
static inline int64_t target_warps() { return (int64_t)ids_sm_count() * 16; }
static inline int64_t min_warps() { return (int64_t)ids_sm_count() * 8; }

DensePlan plan_dense(int64_t rows, int64_t cols, int64_t L, int layout, int flags,
                     bool aligned2, int64_t bucket_rows) {
    DensePlan p{};
    p.layout = layout;
    p.nseg = 1;
    if (layout == IDS_ROW_MAJOR) {
        p.vec = aligned2 ? 2 : 1;
        p.nchunks = (int)ceil_div(cols, 32 * p.vec);
        p.units = L * p.nchunks;
        if (!(flags & IDS_FLAG_ORDERED) && p.units < min_warps()) {
            int64_t ns = ceil_div(target_warps(), p.units);
            const int64_t cap = tmax<int64_t>(1, bucket_rows / 256);
            p.nseg = (int)tmax<int64_t>(1, tmin<int64_t>(ns, cap));
        }
        p.units *= p.nseg;
    } else {
        p.nc = cols >= 2 * target_warps() ? 2 : 1;
        p.ngroups = (int)ceil_div(cols, p.nc);
        p.units = p.ngroups;
        if (!(flags & IDS_FLAG_ORDERED) && p.units < min_warps()) {
            int64_t ns = ceil_div(target_warps(), p.units);
            const int64_t cap = tmax<int64_t>(1, rows / 1024);
            p.nseg = (int)tmax<int64_t>(1, tmin<int64_t>(ns, cap));
        }
        p.units *= p.nseg;
        const size_t per_warp = (size_t)p.nc * L * sizeof(double);
        const size_t budget = 160 * 1024;
        p.wpb = (int)tmin<size_t>(kWarpsPerBlock, budget / per_warp);
        if (p.wpb < 1) {
            p.wpb = kWarpsPerBlock;
            p.global_acc = true;
            p.smem = 0;
        } else {
            p.global_acc = false;
            p.smem = per_warp * p.wpb;
        }
    }
    return p;
}

struct ColTilePlan {
    bool use;
    int ngroups, nseg;
    int64_t ntiles;
    size_t smem;
    // register-accumulator variant (cs_coltile_ra_kernel): BPL buckets per slot
    int bpl, cpl, nslots, ss, threads, ngroups_ra;
    size_t smem_ra;
    int64_t starts_stride;  // int32 per tile in the starts array
};

// columns per lane of the register variant: 1 (8-column CTAs, two per SM) or
// 2 (16-column CTAs, one per SM); IDS_COLTILE_CPL overrides the default
int coltile_ra_cpl() {
    static const int cpl = [] {
        const char* e = getenv("IDS_COLTILE_CPL");
        return (e && atoi(e) == 1) ? 1 : (e && atoi(e) == 2 ? 2 : 2);
    }();
    return cpl;
}

template <int BPL, int CPL>
int coltile_ra_occupancy(int threads, size_t smem) {
    static int cached[1024 / 32 + 1] = {};
    int& c = cached[threads / 32];
    if (!c) {
        // every ss this kernel takes (<= kRaMaxBuckets + 4) fits the attribute
        const size_t smax = kCtStages * coltile_ra_stage_bytes<kCt * CPL>(kRaMaxBuckets + 4);
        IDS_CUDA_TRY(cudaFuncSetAttribute(cs_coltile_ra_kernel<BPL, CPL>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax));
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cs_coltile_ra_kernel<BPL, CPL>,
                                                          threads + 32, smem) != cudaSuccess || occ < 1)
            occ = 1;
        c = occ;
    }
    return c;
}

int coltile_ra_occ(int bpl, int cpl, int threads, size_t smem) {
    if (cpl == 2) switch (bpl) {
            case 2: return coltile_ra_occupancy<2, 2>(threads, smem);
            case 4: return coltile_ra_occupancy<4, 2>(threads, smem);
            default: return coltile_ra_occupancy<8, 2>(threads, smem);
        }
    switch (bpl) {
        case 2: return coltile_ra_occupancy<2, 1>(threads, smem);
        case 4: return coltile_ra_occupancy<4, 1>(threads, smem);
        default: return coltile_ra_occupancy<8, 1>(threads, smem);
    }
}

// The tiled kernels need kCt columns of a tile per stage; the 32-slot one
// also L x kCt accumulators, and both pack buckets into 21 bits of a list
// entry.  The register variant takes over when L <= 512 (at most 64 slots of
// up to 8 buckets, <= 512 threads) and no row segments are needed; set
// IDS_COLTILE_RA=0 to keep the 32-slot kernel.
ColTilePlan plan_coltile(int64_t rows, int64_t cols, int64_t L, int flags) {
    ColTilePlan p{};
    p.smem = coltile_smem(L);
    p.use = p.smem <= 200 * 1024 && L < (1 << 21);
    p.ntiles = ceil_div(rows, kTT);
    // whole waves of two CTAs per SM when the columns allow it
    const int64_t wave = 2 * (int64_t)ids_sm_count();  // two CTAs per SM
    p.ngroups = (int)tmax<int64_t>(ceil_div(cols, kCt), tmin<int64_t>(cols, wave));
    p.nseg = 1;
    if (!(flags & IDS_FLAG_ORDERED) && p.ngroups < wave)
        p.nseg = (int)tmax<int64_t>(1, tmin<int64_t>(ceil_div(wave, p.ngroups), p.ntiles / 4));
    p.starts_stride = kStartsStride;
    static const int ra_env = [] {
        const char* e = getenv("IDS_COLTILE_RA");
        return e ? atoi(e) : 1;
    }();
    if (ra_env && p.nseg == 1 && L <= 512) {
        p.bpl = L <= 128 ? 2 : (L <= 256 ? 4 : 8);
        p.nslots = (int)ceil_div(L, p.bpl);
        p.threads = (int)ceil_div((int64_t)p.nslots * kCt, 32) * 32;
        p.ss = (int)ceil_div(L + 1, 4) * 4;  // bucket starts per tile
        p.cpl = coltile_ra_cpl();
        p.smem_ra = kCtStages * (p.cpl == 2 ? coltile_ra_stage_bytes<2 * kCt>(p.ss)
                                            : coltile_ra_stage_bytes<kCt>(p.ss));
        const int64_t cap = (int64_t)ids_sm_count() * coltile_ra_occ(p.bpl, p.cpl, p.threads, p.smem_ra);
        p.ngroups_ra = (int)tmax<int64_t>(ceil_div(cols, (int64_t)kCt * p.cpl), tmin<int64_t>(cols, cap));
        p.starts_stride = tmax<int64_t>(kStartsStride, p.ss);
    }
    return p;
}

}  // namespace

extern "C" size_t ids_countsketch_dense_workspace_bytes(int64_t rows, int64_t cols,
                                                        int64_t out_dim, int layout) {
    // worst case over the plans the kernel may choose
    const DensePlan p = plan_dense(rows, cols, out_dim, layout, 0, true, rows);
    const DensePlan p1 = plan_dense(rows, cols, out_dim, layout, 0, false, rows);
    const int nseg = max(p.nseg, p1.nseg);
    WsCount c;
    if (layout == IDS_COL_MAJOR && plan_coltile(rows, cols, out_dim, 0).use) {
        const ColTilePlan q = plan_coltile(rows, cols, out_dim, 0);
        const ColTilePlan qo = plan_coltile(rows, cols, out_dim, IDS_FLAG_ORDERED);
        c.take<double>((size_t)tmax(nseg, q.nseg) * out_dim * cols);
        c.take<int32_t>((size_t)rows);
        c.take<int32_t>((size_t)q.ntiles * kTT);
        c.take<int32_t>((size_t)q.ntiles * tmax(q.starts_stride, qo.starts_stride));
        return c.off + 256;
    }
    c.take<double>((size_t)nseg * out_dim * cols);
    if (layout == IDS_COL_MAJOR && p.global_acc) c.take<double>((size_t)p.units * p.nc * out_dim);
    return c.off + 256;
}

extern "C" int ids_countsketch_dense_f64(const double* A, int64_t rows, int64_t cols,
                                         int64_t ld, int layout, int64_t row0, int64_t in_dim,
                                         const int32_t* bucket, const int8_t* sign,
                                         const int32_t* order_signed, const int64_t* bstart,
                                         int64_t out_dim, double* Y, int accumulate, int flags,
                                         int32_t* nonfinite, void* workspace, size_t ws_bytes,
                                         void* stream) {
    if (rows < 1 || cols < 1 || out_dim < 1 || row0 < 0 || row0 + rows > in_dim ||
        (layout != IDS_ROW_MAJOR && layout != IDS_COL_MAJOR) ||
        ld < (layout == IDS_ROW_MAJOR ? cols : rows) || in_dim > 0x7fffffffLL) {
        ids_set_last_error("dense countsketch: bad arguments");
        return IDS_EINVAL;
    }
    cudaStream_t st = as_stream(stream);
    if (layout == IDS_COL_MAJOR) {
        const ColTilePlan q = plan_coltile(rows, cols, out_dim, flags);
        if (q.use) {
            WsCarve ws(workspace, ws_bytes);
            double* part = q.nseg > 1 ? ws.take<double>((size_t)q.nseg * out_dim * cols) : nullptr;
            int32_t* codes = ws.take<int32_t>((size_t)rows);
            int32_t* lists = ws.take<int32_t>((size_t)q.ntiles * kTT);
            int32_t* starts = ws.take<int32_t>((size_t)q.ntiles * q.starts_stride);
            if (!ws.ok()) {
                ids_set_last_error("dense countsketch: workspace too small");
                return IDS_EWORKSPACE;
            }
            const int64_t seg_stride = out_dim * cols;
            const unsigned gc = (unsigned)tmin<int64_t>(ceil_div(rows, 256), 148 * 8);
            row_codes_kernel<<<gc, 256, 0, st>>>(bucket, sign, row0, rows, codes);
            IDS_LAUNCH_CHECK();
            const int vec16 = ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && (ld % 2 == 0);
            double* out = q.nseg > 1 ? part : Y;
            const int init = (q.nseg == 1 && accumulate) ? 1 : 0;
            if (q.bpl && vec16) {
                tile_bucket_lists_kernel<kTT><<<(unsigned)q.ntiles, kCtThreads, 0, st>>>(
                    codes, rows, (int)out_dim, q.ss, lists, starts);
                IDS_LAUNCH_CHECK();
                const unsigned grid = (unsigned)q.ngroups_ra;
#define IDS_RA_LAUNCH(B, C)                                                                  \
    cs_coltile_ra_kernel<B, C><<<grid, q.threads + 32, q.smem_ra, st>>>(                     \
        A, ld, rows, cols, lists, starts, out_dim, q.nslots, q.ss, q.ngroups_ra, out, init)
                if (q.cpl == 2) {
                    if (q.bpl == 2) IDS_RA_LAUNCH(2, 2);
                    else if (q.bpl == 4) IDS_RA_LAUNCH(4, 2);
                    else IDS_RA_LAUNCH(8, 2);
                } else {
                    if (q.bpl == 2) IDS_RA_LAUNCH(2, 1);
                    else if (q.bpl == 4) IDS_RA_LAUNCH(4, 1);
                    else IDS_RA_LAUNCH(8, 1);
                }
#undef IDS_RA_LAUNCH
                IDS_LAUNCH_CHECK();
            } else {
                tile_slot_lists_kernel<<<(unsigned)q.ntiles, kCtThreads, 0, st>>>(codes, rows, lists,
                                                                                  starts);
                IDS_LAUNCH_CHECK();
                const unsigned grid = (unsigned)((int64_t)q.ngroups * q.nseg);
                IDS_CUDA_TRY(cudaFuncSetAttribute(cs_coltile_kernel,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)q.smem));
                cs_coltile_kernel<<<grid, kCtThreads, q.smem, st>>>(A, ld, rows, cols, lists, starts,
                                                                    out_dim, q.ngroups, q.nseg, vec16,
                                                                    out, seg_stride, init);
                IDS_LAUNCH_CHECK();
            }
            if (q.nseg > 1) {
                const unsigned g = (unsigned)tmin<int64_t>(ceil_div(seg_stride, 256), 148 * 8);
                seg_reduce_kernel<<<g, 256, 0, st>>>(part, q.nseg, seg_stride, seg_stride, Y,
                                                     accumulate);
                IDS_LAUNCH_CHECK();
            }
            if (nonfinite) {
                const unsigned g = (unsigned)tmin<int64_t>(ceil_div(seg_stride, 256), 148 * 4);
                nonfinite_scan_kernel<<<g, 256, 0, st>>>(Y, seg_stride, nonfinite);
                IDS_LAUNCH_CHECK();
            }
            return IDS_OK;
        }
    }
    const bool aligned2 = ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && (ld % 2 == 0) &&
                          (cols % 2 == 0);
    const DensePlan p = plan_dense(rows, cols, out_dim, layout, flags, aligned2,
                                   tmax<int64_t>(1, rows / out_dim));
    WsCarve ws(workspace, ws_bytes);
    double* part = p.nseg > 1 ? ws.take<double>((size_t)p.nseg * out_dim * cols) : nullptr;
    double* gacc = (layout == IDS_COL_MAJOR && p.global_acc)
                       ? ws.take<double>((size_t)p.units * p.nc * out_dim)
                       : nullptr;
    if (!ws.ok()) {
        ids_set_last_error("dense countsketch: workspace too small");
        return IDS_EWORKSPACE;
    }
    double* out = p.nseg > 1 ? part : Y;
    const int64_t seg_stride = out_dim * cols;
    const int init_from_out = (p.nseg == 1 && accumulate) ? 1 : 0;
    if (layout == IDS_ROW_MAJOR) {
        const int restrict_rows = (row0 != 0 || rows != in_dim) ? 1 : 0;
        const unsigned grid = (unsigned)ceil_div(p.units, kWarpsPerBlock);
        if (p.vec == 2)
            cs_rowmajor_kernel<2, 8><<<grid, kWarpsPerBlock * 32, 0, st>>>(
                A, ld, cols, row0, rows, restrict_rows, order_signed, bstart, out_dim,
                p.nchunks, p.nseg, out, seg_stride, init_from_out);
        else
            cs_rowmajor_kernel<1, 8><<<grid, kWarpsPerBlock * 32, 0, st>>>(
                A, ld, cols, row0, rows, restrict_rows, order_signed, bstart, out_dim,
                p.nchunks, p.nseg, out, seg_stride, init_from_out);
        IDS_LAUNCH_CHECK();
    } else {
        const unsigned grid = (unsigned)ceil_div(p.units, p.wpb);
        if (p.smem > 40 * 1024) {
            if (p.nc == 2)
                IDS_CUDA_TRY(cudaFuncSetAttribute(cs_colmajor_kernel<2, 4>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)p.smem));
            else
                IDS_CUDA_TRY(cudaFuncSetAttribute(cs_colmajor_kernel<1, 4>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)p.smem));
        }
        if (p.nc == 2)
            cs_colmajor_kernel<2, 4><<<grid, p.wpb * 32, p.smem, st>>>(
                A, ld, rows, cols, row0, bucket, sign, out_dim, p.ngroups, p.nseg, p.wpb, out,
                seg_stride, init_from_out, gacc);
        else
            cs_colmajor_kernel<1, 4><<<grid, p.wpb * 32, p.smem, st>>>(
                A, ld, rows, cols, row0, bucket, sign, out_dim, p.ngroups, p.nseg, p.wpb, out,
                seg_stride, init_from_out, gacc);
        IDS_LAUNCH_CHECK();
    }
    if (p.nseg > 1) {
        const unsigned g = (unsigned)tmin<int64_t>(ceil_div(seg_stride, 256), 148 * 8);
        seg_reduce_kernel<<<g, 256, 0, st>>>(part, p.nseg, seg_stride, seg_stride, Y, accumulate);
        IDS_LAUNCH_CHECK();
    }
    if (nonfinite) {
        const unsigned g = (unsigned)tmin<int64_t>(ceil_div(seg_stride, 256), 148 * 4);
        nonfinite_scan_kernel<<<g, 256, 0, st>>>(Y, seg_stride, nonfinite);
        IDS_LAUNCH_CHECK();
    }
    return IDS_OK;
}

extern "C" int ids_dense_has_nonfinite(const double* A, int64_t rows, int64_t cols, int64_t ld,
                                       int layout, int32_t* flag, void* stream) {
    if (rows < 0 || cols < 0) return IDS_EINVAL;
    if (rows == 0 || cols == 0) return IDS_OK;
    const int64_t outer = layout == IDS_ROW_MAJOR ? rows : cols;
    const int64_t inner = layout == IDS_ROW_MAJOR ? cols : rows;
    const unsigned g = (unsigned)tmin<int64_t>(ceil_div(outer * inner, 256), 148 * 16);
    dense_nonfinite_kernel<<<g, 256, 0, as_stream(stream)>>>(A, outer, inner, ld, flag);
    IDS_LAUNCH_CHECK();
    return IDS_OK;
}
