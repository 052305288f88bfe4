// tcgen05.mma kind::tf32 pacing probe: cycles per MMA (M = 128, K = 8) against N, the shared-memory operand
// layout (no swizzle / 32 / 64 / 128-byte swizzle) and the A operand source (shared or tensor memory).
// Timing only: the operands are whatever shared memory holds. nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2401_09792_b200/csrc/tc_sm100.cuh"
using namespace gwtk;

__device__ __forceinline__ uint64_t desc_sw(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem), "r"(a_tmem), "l"(bdesc),
                 "r"(idesc), "r"(acc));
}

// mode: layout code 0 none, 6 = 32B, 4 = 64B, 2 = 128B; ts: A from TMEM; KS k-steps per accumulator group
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
    return pred != 0;
}

// whole warp walks the loop, the MMA is issued under elect.sync (no divergent region around the uniform-datapath
// instruction), descriptors advance by constant adds, k-steps unrolled
template <int KS>
__global__ void __launch_bounds__(128, 1) probe_elect(int N, int iters, long long* out) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x;
    for (int i = tid; i < 160 * 1024 / 4; i += 128) reinterpret_cast<float*>(smem)[i] = 1.0f + (i % 7) * 0.125f;
    if (tid < 32) tc::tmem_alloc(&tbase, 512);
    if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
    tc::fence_async_shared();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tb = tbase;
    if (tid < 32) {
        const uint32_t a0 = tc::smem_u32(smem), b0 = a0 + 64 * 1024;
        const uint32_t idesc = tc::idesc_tf32(128, N);
        const uint64_t da = tc::smem_desc(a0, 128, KS * 256), db = tc::smem_desc(b0, 128, KS * 256);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint32_t d = tb + (uint32_t)((it & 1) * N);
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < KS; ++kk) {
                    if (kk == 0) asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(da), "l"(db), "r"(idesc));
                    else asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(da + 16 * kk), "l"(db + 16 * kk), "r"(idesc));
                }
            }
            __syncwarp();
        }
        if (elect_one()) tc::commit(&bar);
        __syncwarp();
        tc::mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (blockIdx.x == 0 && tid == 0) out[0] = t1 - t0;
    }
    __syncthreads();
    if (tid < 32) tc::tmem_dealloc(tb, 512);
}

__global__ void __launch_bounds__(128, 1) probe(int N, int layout, int ts, int iters, int ksteps, long long* out) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x;
    for (int i = tid; i < 160 * 1024 / 4; i += 128) reinterpret_cast<float*>(smem)[i] = 1.0f + (i % 7) * 0.125f;
    if (tid < 32) tc::tmem_alloc(&tbase, 512);
    if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
    tc::fence_async_shared();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tb = tbase;
    if (tid == 0) {
        // row pitch inside an 8-row group: no swizzle -> core matrices (LBO 128 between K cores, SBO = ksteps*256);
        // swizzled K-major: SBO = 8 * swizzle bytes, K advance = +32 bytes inside the atom
        const uint32_t swb = layout == 2 ? 128 : layout == 4 ? 64 : layout == 6 ? 32 : 0;
        const uint32_t sbo = swb ? 8 * swb : (uint32_t)ksteps * 256;
        const uint32_t lbo = swb ? 16 : 128;
        const uint32_t a0 = tc::smem_u32(smem), b0 = a0 + 64 * 1024;
        const uint32_t idesc = tc::idesc_tf32(128, N);
        const int kin = swb ? swb / 32 : ksteps;  // k-steps reachable inside one atom / tile
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            for (int kk = 0; kk < ksteps; ++kk) {
                const int ka = kk % kin, kb = kk / kin;
                const uint32_t koff = swb ? (uint32_t)ka * 32 + (uint32_t)kb * 16 * 1024 : (uint32_t)kk * 256;
                const uint64_t da = desc_sw(a0 + koff, lbo, sbo, layout);
                const uint64_t db = desc_sw(b0 + koff, lbo, sbo, layout);
                const uint32_t d = tb + (uint32_t)((it & 1) * N);
                if (ts) mma_ts(d, tb + 256 + 8 * kk, db, idesc, kk > 0);
                else tc::mma_tf32(d, da, db, idesc, kk > 0);
            }
        }
        tc::commit(&bar);
        tc::mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    __syncthreads();
    if (tid < 32) tc::tmem_dealloc(tb, 512);
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    const int iters = 2000, ks = 6;
    cudaFuncSetAttribute(probe_elect<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    for (int N : {32, 64, 128, 256}) {
        probe_elect<6><<<148, 128, 160 * 1024>>>(N, iters, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h = 0;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("elect, unrolled, no swizzle N %3d: %.1f cycles / MMA (floor %d)  %s\n", N, (double)h / (iters * ks), 128 * N / 256,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    for (int ts = 0; ts < 2; ++ts)
        for (int layout : {0})
            for (int N : {32, 64, 128, 256}) {
                probe<<<148, 128, 160 * 1024>>>(N, layout, ts, iters, ks, d);
                cudaError_t e = cudaDeviceSynchronize();
                long long h = 0;
                cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
                printf("A %s layout %d N %3d: %.1f cycles / MMA (floor %d)  %s\n", ts ? "tmem" : "smem", layout, N,
                       (double)h / (iters * ks), 128 * N / 256, e == cudaSuccess ? "" : cudaGetErrorString(e));
                if (e != cudaSuccess) return 1;
            }
    return 0;
}
