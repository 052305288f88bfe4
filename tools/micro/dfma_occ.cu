// DFMA throughput vs resident warps per SM (B200): 8 / 16 / 32 warps, 8 or 16 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k_dfma(const double* in, double* out, int iters) {
    double a = in[threadIdx.x & 7], b = in[(threadIdx.x + 1) & 7];
    double s[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) s[c] = c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) s[c] = fma(a, b, s[c]);
    }
    double t = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) t += s[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
    double *din, *out;
    cudaMalloc(&din, 64 * 8); cudaMalloc(&out, 148 * 1024 * 8); cudaMemset(din, 0, 64 * 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 1 << 13;
    for (int thr : {128, 256, 512, 1024}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0); k_dfma<16><<<sms, thr>>>(din, out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double ops = 16.0 * iters * sms * thr;
            if (rep) printf("threads/SM %4d (16 chains): %.1f DFMA/clk/SM\n", thr, ops / (ms * 1e-3) / sms / 1.965e9);
            cudaEventRecord(e0); k_dfma<4><<<sms, thr>>>(din, out, iters * 4); cudaEventRecord(e1); cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            ops = 16.0 * iters * sms * thr;
            if (rep) printf("threads/SM %4d (4 chains):  %.1f DFMA/clk/SM\n", thr, ops / (ms * 1e-3) / sms / 1.965e9);
        }
    }
    return 0;
}
