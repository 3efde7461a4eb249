// Complex fp64 helpers and in-register DFT kernels shared by the
// TensorSketch kernels (tensorsketch.cu, tensorsketch_split.cu).
#pragma once

#include <cuda_runtime.h>

namespace ids_fft {

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
__device__ __forceinline__ void dft<1>(double2*) {}  // length-1 transforms (N2 = 1)

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

// 16-point DFT in registers: 4 x DFT4, internal twiddles W16^(n2 k1), 4 x DFT4.
__device__ __forceinline__ void dft16(double2* x) {
    const double c = 0.92387953251128675613, s = 0.38268343236508977173;
    const double h = 0.70710678118654752440;
    double2 a[4][4];
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
        double2 t[4] = {x[n2], x[4 + n2], x[8 + n2], x[12 + n2]};
        dft<4>(t);
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) a[n2][k1] = t[k1];
    }
    a[1][1] = cmul(a[1][1], make_double2(c, -s));   // W^1
    a[1][2] = cmul(a[1][2], make_double2(h, -h));   // W^2
    a[1][3] = cmul(a[1][3], make_double2(s, -c));   // W^3
    a[2][1] = cmul(a[2][1], make_double2(h, -h));   // W^2
    a[2][2] = mul_mi(a[2][2]);                      // W^4 = -i
    a[2][3] = cmul(a[2][3], make_double2(-h, -h));  // W^6
    a[3][1] = cmul(a[3][1], make_double2(s, -c));   // W^3
    a[3][2] = cmul(a[3][2], make_double2(-h, -h));  // W^6
    a[3][3] = cmul(a[3][3], make_double2(-c, s));   // W^9
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
        double2 t[4] = {a[0][k1], a[1][k1], a[2][k1], a[3][k1]};
        dft<4>(t);
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) x[k1 + 4 * k2] = t[k2];
    }
}

template <>
__device__ __forceinline__ void dft<16>(double2* v) {
    dft16(v);
}

}  // namespace ids_fft
