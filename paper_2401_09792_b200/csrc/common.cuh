// Shared device helpers for the gwt B200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gwtk {

// complex element type per storage dtype: c64 -> float2, c128 -> double2
template <class R> struct CplxOf;
template <> struct CplxOf<float> { using type = float2; };
template <> struct CplxOf<double> { using type = double2; };

template <class R> using cplx_t = typename CplxOf<R>::type;

__host__ __device__ __forceinline__ float2 mk(float re, float im) { return make_float2(re, im); }
__host__ __device__ __forceinline__ double2 mk(double re, double im) { return make_double2(re, im); }

template <class C> __device__ __forceinline__ C cadd(C a, C b) { return mk(a.x + b.x, a.y + b.y); }
template <class C> __device__ __forceinline__ C csub(C a, C b) { return mk(a.x - b.x, a.y - b.y); }
template <class C> __device__ __forceinline__ C cmul(C a, C b) { return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
// a * conj(b)
template <class C> __device__ __forceinline__ C cmulc(C a, C b) { return mk(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y); }
// conj(a) * b
template <class C> __device__ __forceinline__ C cconjmul(C a, C b) { return mk(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x); }
template <class C> __device__ __forceinline__ C cconj(C a) { return mk(a.x, -a.y); }
// acc += a*b
template <class C> __device__ __forceinline__ void cfma(C& acc, C a, C b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
}
// acc += a*conj(b)
template <class C> __device__ __forceinline__ void cfmac(C& acc, C a, C b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(a.y, b.x, acc.y);
    acc.y = fma(-a.x, b.y, acc.y);
}
// acc += conj(a)*b
template <class C> __device__ __forceinline__ void cfmaconj(C& acc, C a, C b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(-a.y, b.x, acc.y);
}

__device__ __forceinline__ double2 to_d2(float2 a) { return make_double2(a.x, a.y); }
__device__ __forceinline__ double2 to_d2(double2 a) { return a; }
template <class C> __device__ __forceinline__ C from_d2(double2 a);
template <> __device__ __forceinline__ float2 from_d2<float2>(double2 a) { return make_float2((float)a.x, (float)a.y); }
template <> __device__ __forceinline__ double2 from_d2<double2>(double2 a) { return a; }

template <class C> __device__ __forceinline__ C czero() { return mk(decltype(C{}.x)(0), decltype(C{}.x)(0)); }

// exp(-j 2 pi f tau) with the phase argument reduced in binary64 first:
// f*tau is formed and its fractional part taken in fp64 so fp32 builds do not
// lose the ~600 rad phase.
__device__ __forceinline__ double2 phasor_neg(double f, double tau) {
    double x = f * tau;
    x = x - floor(x);
    double s, c;
    sincospi(2.0 * x, &s, &c);
    return make_double2(c, -s);
}

// conj(c_r(f)) for the fp32 kernels: binary64 argument reduction x = frac(f tau), then sincospif of the
// fp32 head xh = (float)x and a first-order rotation by the remainder 2 pi (x - xh) (|x - xh| <= 3e-8), so the
// phase carries ~1 ulp of fp32 instead of the 2e-7 rad of rounding the argument (a full binary64 sincospi
// measured no better on H~ at C4: the E / H~ accumulations dominate).
template <class T> __device__ __forceinline__ cplx_t<T> conj_coeff(double f, double tau);
template <> __device__ __forceinline__ float2 conj_coeff<float>(double f, double tau) {
    double x = f * tau;
    x -= floor(x);
    const float xh = (float)x;
    const float d = (float)(6.283185307179586 * (x - (double)xh));
    float s, c;
    sincospif(2.0f * xh, &s, &c);
    return make_float2(fmaf(-s, d, c), -fmaf(c, d, s));
}
template <> __device__ __forceinline__ double2 conj_coeff<double>(double f, double tau) { return phasor_neg(f, tau); }

// Topology helpers shared by the kernels: link = (k*J + i)*K + j, user = i*K + j.
struct Topo {
    int J, K, M, N, P, m, n, p, L;
    __host__ __device__ int users() const { return J * K; }
    __host__ __device__ int links() const { return J * J * K; }
};

// binary64 reciprocal: MUFU seed + two Newton steps (no division sequence on the QL's serial chain)
__device__ __forceinline__ double frcp(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = fma(y, fma(-x, y, 1.0), y);
    return fma(y, fma(-x, y, 1.0), y);
}

// binary64 reciprocal square root of a positive normal number: MUFU seed (~2^-22) + two Newton steps, no special-case
// branches (libdevice's rsqrt carries a slow path and was the top stall line of the QL chain)
__device__ __forceinline__ double frsqrt(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double hx = 0.5 * x;
    y = fma(y, fma(-hx * y, y, 0.5), y);
    return fma(y, fma(-hx * y, y, 0.5), y);
}


}  // namespace gwtk
