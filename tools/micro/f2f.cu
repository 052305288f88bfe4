// Throughput probe: F2F.F64.F32 conversions vs DFMA vs FFMA per SM per clock (B200).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_f2f(const float* in, double* out, int iters) {
    float a = in[threadIdx.x], b = in[threadIdx.x + 1], c = in[threadIdx.x + 2], d = in[threadIdx.x + 3];
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    for (int i = 0; i < iters; ++i) {
        s0 += (double)a; s1 += (double)b; s2 += (double)c; s3 += (double)d;
        a += 1.0f; b += 1.0f; c += 1.0f; d += 1.0f;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
__global__ void k_dfma(const double* in, double* out, int iters) {
    double a = in[threadIdx.x], b = in[threadIdx.x + 1];
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0, s6 = 0, s7 = 0;
    for (int i = 0; i < iters; ++i) {
        s0 = fma(a, b, s0); s1 = fma(a, b, s1); s2 = fma(a, b, s2); s3 = fma(a, b, s3);
        s4 = fma(a, b, s4); s5 = fma(a, b, s5); s6 = fma(a, b, s6); s7 = fma(a, b, s7);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3 + s4 + s5 + s6 + s7;
}
int main() {
    float* fin; double *din, *out;
    cudaMalloc(&fin, 4096); cudaMalloc(&din, 8192); cudaMalloc(&out, 148 * 8 * 1024 * 8);
    cudaMemset(fin, 0, 4096); cudaMemset(din, 0, 8192);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 1 << 14, blocks = sms * 8, thr = 256;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0); k_f2f<<<blocks, thr>>>(fin, out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = 4.0 * iters * blocks * thr;
        printf("F2F.F64.F32: %.1f Gop/s = %.1f per SM per clk (clk %d kHz)\n", ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk * 1e3), clk);
        cudaEventRecord(e0); k_dfma<<<blocks, thr>>>(din, out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        ops = 8.0 * iters * blocks * thr;
        printf("DFMA: %.1f Gop/s = %.1f per SM per clk\n", ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk * 1e3));
    }
    return 0;
}
