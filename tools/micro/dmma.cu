// DMMA (mma.sync.m8n8k4.f64) throughput vs resident warps per SM on B200, beside DFMA (tools/micro/dfma_occ.cu).
// Decides whether the binary64 Gram epilogue of k_rgram can move from DFMA onto the FP64 tensor path.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(const double* in, double* out, int iters) {
    double a = in[threadIdx.x & 7], b = in[(threadIdx.x + 1) & 7];
    double s[CH][2];
#pragma unroll
    for (int c = 0; c < CH; ++c) s[c][0] = s[c][1] = c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) dmma(s[c], a, b);
    }
    double t = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) t += s[c][0] + s[c][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

// DMMA fed by F2F conversions of fp32 values (the epilogue's shape: one fp32 pair per lane per k-chunk)
template <int CH>
__global__ void k_dmma_cvt(const float* in, double* out, int iters) {
    float a = in[threadIdx.x & 7], b = in[(threadIdx.x + 1) & 7];
    double s[CH][2];
#pragma unroll
    for (int c = 0; c < CH; ++c) s[c][0] = s[c][1] = c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const double da = (double)(a + (float)c), db = (double)b;
            dmma(s[c], da, db);
            dmma(s[c], db, da);
        }
        a += 1e-7f;
    }
    double t = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) t += s[c][0] + s[c][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
    double *din, *out;
    float* fin;
    cudaMalloc(&din, 64 * 8);
    cudaMalloc(&fin, 64 * 4);
    cudaMalloc(&out, 148 * 2048 * 8);
    cudaMemset(din, 0, 64 * 8);
    cudaMemset(fin, 0, 64 * 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 1 << 12;
    for (int thr : {64, 128, 256, 512, 1024}) {
        for (int rep = 0; rep < 2; ++rep) {
            float ms;
            cudaEventRecord(e0);
            k_dmma<8><<<sms, thr>>>(din, out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            double fmas = 8.0 * iters * sms * (thr / 32) * 256;
            if (rep) printf("threads/SM %4d dmma 8 chains: %.1f FMA/clk/SM  (%.1f TFLOP/s)\n", thr, fmas / (ms * 1e-3) / sms / 1.965e9, 2 * fmas / (ms * 1e-3) / 1e12);
            cudaEventRecord(e0);
            k_dmma<2><<<sms, thr>>>(din, out, iters * 4);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep) printf("threads/SM %4d dmma 2 chains: %.1f FMA/clk/SM\n", thr, fmas / (ms * 1e-3) / sms / 1.965e9);
            cudaEventRecord(e0);
            k_dmma_cvt<4><<<sms, thr>>>(fin, out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep) printf("threads/SM %4d dmma+cvt 4 chains: %.1f FMA/clk/SM\n", thr, fmas / (ms * 1e-3) / sms / 1.965e9);
        }
    }
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
