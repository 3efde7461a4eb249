// Shared helpers for the idsketch-b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/idsketch_b200.h"

#define IDS_CUDA_TRY(expr)                                   \
    do {                                                     \
        cudaError_t _e = (expr);                             \
        if (_e != cudaSuccess) {                             \
            ids_set_cuda_error(_e, __FILE__, __LINE__);      \
            return IDS_ECUDA;                                \
        }                                                    \
    } while (0)

#define IDS_LAUNCH_CHECK()                                   \
    do {                                                     \
        ids_count_launch();                                  \
        cudaError_t _e = cudaGetLastError();                 \
        if (_e != cudaSuccess) {                             \
            ids_set_cuda_error(_e, __FILE__, __LINE__);      \
            return IDS_ECUDA;                                \
        }                                                    \
    } while (0)

void ids_set_last_error(const char* msg);
void ids_set_cuda_error(cudaError_t e, const char* file, int line);
void ids_count_launch();

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// SM count of the current device (148 on B200), queried once per process:
// the planners size grids and per-CTA workspaces from it.
int ids_sm_count();

template <class T>
__host__ __device__ __forceinline__ T tmin(T a, T b) { return a < b ? a : b; }
template <class T>
__host__ __device__ __forceinline__ T tmax(T a, T b) { return a < b ? b : a; }

static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Simple bump allocator over a caller-owned workspace.
struct WsCarve {
    char* base;
    size_t cap;
    size_t off;
    __host__ WsCarve(void* b, size_t c) : base(static_cast<char*>(b)), cap(c), off(0) {}
    template <class T>
    __host__ T* take(size_t n) {
        off = align_up(off, 256);
        T* p = reinterpret_cast<T*>(base + off);
        off += n * sizeof(T);
        return p;
    }
    __host__ bool ok() const { return off <= cap; }
};

// Byte count the same carve sequence needs (workspace query helpers).
struct WsCount {
    size_t off = 0;
    template <class T>
    void take(size_t n) {
        off = align_up(off, 256);
        off += n * sizeof(T);
    }
};

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned warp_id() { return threadIdx.x >> 5; }

// Signed-row encoding used by the bucket index: row >= 0 with sign +1 is
// stored as row, sign -1 as ~row (negative).
__device__ __forceinline__ int32_t enc_row(int32_t row, int8_t s) { return s > 0 ? row : ~row; }
__device__ __forceinline__ int32_t dec_row(int32_t e) { return e >= 0 ? e : ~e; }

// Grid-wide barrier for cooperative (all-resident) kernels: one thread per
// CTA arrives on bar[0]; the waiters poll the generation word bar[1] with a
// nanosleep back-off, so CTAs parked at a barrier leave the SMs (and the L2
// slice of the counter) to the warps still working.  bar[] must be zeroed
// before the launch.  Pays where one CTA works while the others wait (the
// hash's phase B: ~10-20% faster than cooperative_groups' grid.sync());
// where all CTAs arrive together (CPQR) the spin barrier wakes faster.
__device__ __forceinline__ void ids_grid_bar(unsigned* bar, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g0 = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == nblocks - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            unsigned ns = 32;
            while (*gen == g0) {
                __nanosleep(ns);
                if (ns < 256) ns <<= 1;
            }
        }
        __threadfence();
    }
    __syncthreads();
}
