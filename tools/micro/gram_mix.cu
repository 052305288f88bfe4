// The k_rgram pair-Gram epilogue's arithmetic shape without TMEM: per iteration 4 + 8 complex operands (24 values),
// 32 complex accumulators (128 DFMA). MODE 0: operands loop-invariant registers (DFMA + register bandwidth only);
// MODE 1: operands converted from fp32 each iteration (24 F2F.F64.F32, as the epilogue does);
// MODE 2: operands produced by integer exponent rebias (no XU).  Prints DFMA/clk/SM per resident-warp count.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ double i2d(uint32_t b) {
    uint32_t hi = (((b & 0x7fffffffu) >> 3) + 0x38000000u) | (b & 0x80000000u);
    return __hiloint2double((int)hi, (int)(b << 29));
}
template <int MODE>
__global__ void k_mix(const float* in, double* out, int iters) {
    float xf[8], af[16];
    for (int i = 0; i < 8; ++i) xf[i] = in[(threadIdx.x + i) & 63];
    for (int i = 0; i < 16; ++i) af[i] = in[(threadIdx.x + 8 + i) & 63];
    double2 acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = make_double2(0.0, 0.0);
    double2 x[4], a[8];
#pragma unroll
    for (int z = 0; z < 4; ++z) x[z] = make_double2(xf[2 * z], xf[2 * z + 1]);
#pragma unroll
    for (int w = 0; w < 8; ++w) a[w] = make_double2(af[2 * w], af[2 * w + 1]);
    for (int it = 0; it < iters; ++it) {
        if (MODE == 1) {
#pragma unroll
            for (int z = 0; z < 4; ++z) x[z] = make_double2((double)xf[2 * z], (double)xf[2 * z + 1]);
        } else if (MODE == 2) {
#pragma unroll
            for (int z = 0; z < 4; ++z) x[z] = make_double2(i2d(__float_as_uint(xf[2 * z])), i2d(__float_as_uint(xf[2 * z + 1])));
        }
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            double2 av = a[w];
            if (MODE == 1) av = make_double2((double)af[2 * w], (double)af[2 * w + 1]);
            else if (MODE == 2) av = make_double2(i2d(__float_as_uint(af[2 * w])), i2d(__float_as_uint(af[2 * w + 1])));
#pragma unroll
            for (int z = 0; z < 4; ++z) {
                double2& c = acc[z * 8 + w];
                c.x = fma(x[z].x, av.x, c.x);
                c.x = fma(x[z].y, av.y, c.x);
                c.y = fma(x[z].y, av.x, c.y);
                c.y = fma(-x[z].x, av.y, c.y);
            }
        }
        if (MODE != 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i) xf[i] = __uint_as_float(__float_as_uint(xf[i]) ^ (it & 1));
#pragma unroll
            for (int i = 0; i < 16; ++i) af[i] = __uint_as_float(__float_as_uint(af[i]) ^ (it & 1));
        }
    }
    double t = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) t += acc[i].x + acc[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int MODE>
void run(const float* in, double* out, int sms) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 1 << 12;
    for (int thr : {64, 128, 256}) {
        float ms = 0;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0); k_mix<MODE><<<sms, thr>>>(in, out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        printf("mode %d threads/SM %4d: %.1f DFMA/clk/SM\n", MODE, thr, 128.0 * iters * thr / (ms * 1e-3) / 1.965e9);
    }
}
int main() {
    float* in; double* out;
    cudaMalloc(&in, 64 * 4); cudaMalloc(&out, 148 * 1024 * 8);
    float h[64]; for (int i = 0; i < 64; ++i) h[i] = 1.0f + i * 0.01f;
    cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>(in, out, sms); run<1>(in, out, sms); run<2>(in, out, sms);
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
