// tcgen05 (5th-gen tensor core) kernels, sm_100a.
//
// k_tc_gemm_test: one 128x128 fp32 tile C = A * B^T (A, B row-major with K contiguous)
// through tcgen05.mma.kind::tf32 with operands staged in the canonical K-major layout
// and the accumulator in TMEM; optional 3xTF32 split (hi*hi + hi*lo + lo*hi) for
// ~fp32 accuracy. Used to validate the descriptor/TMEM plumbing (tests/test_tc.py) that
// the batched complex Gram kernel builds on.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "tc_sm100.cuh"

namespace gwtk {

template <bool SPLIT3>
__global__ void __launch_bounds__(128) k_tc_gemm_test(int K, const float* __restrict__ A, const float* __restrict__ B,
                                                      float* __restrict__ C) {
    constexpr int KC = 32, ROWS = 128;
    constexpr uint32_t TILE = ROWS * KC * 4;  // 16 KB
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* sAh = smem;
    unsigned char* sAl = smem + TILE;
    unsigned char* sBh = smem + 2 * TILE;
    unsigned char* sBl = smem + 3 * TILE;
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    if (warp == 0) tc::tmem_alloc(&tmem_base, 128);
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        tc::fence_barrier_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t taddr = tmem_base;
    constexpr uint32_t idesc = tc::idesc_tf32(128, 128);
    uint32_t phase = 0;
    for (int k0 = 0; k0 < K; k0 += KC) {
        for (int idx = tid; idx < ROWS * KC; idx += blockDim.x) {
            const int r = idx / KC, k = idx % KC;
            const float a = (k0 + k < K) ? A[(size_t)r * K + k0 + k] : 0.f;
            const float b = (k0 + k < K) ? B[(size_t)r * K + k0 + k] : 0.f;
            float ah, al, bh, bl;
            tc::split_tf32(a, ah, al);
            tc::split_tf32(b, bh, bl);
            const uint32_t off = tc::kmajor_off(r, k, KC);
            *reinterpret_cast<float*>(sAh + off) = SPLIT3 ? ah : a;
            *reinterpret_cast<float*>(sBh + off) = SPLIT3 ? bh : b;
            *reinterpret_cast<float*>(sAl + off) = al;
            *reinterpret_cast<float*>(sBl + off) = bl;
        }
        tc::fence_async_shared();
        __syncthreads();
        if (tid == 0) {
            tc::fence_after_sync();
            const uint32_t ah = tc::smem_u32(sAh), al = tc::smem_u32(sAl), bh = tc::smem_u32(sBh), bl = tc::smem_u32(sBl);
            constexpr uint32_t LBO = 128, SBO = (KC / 4) * 128;
#pragma unroll
            for (int s = 0; s < KC / 8; ++s) {
                const uint32_t o = s * 256;
                const uint32_t acc = (k0 > 0 || s > 0) ? 1u : 0u;
                tc::mma_tf32(taddr, tc::smem_desc(ah + o, LBO, SBO), tc::smem_desc(bh + o, LBO, SBO), idesc, acc);
                if (SPLIT3) {
                    tc::mma_tf32(taddr, tc::smem_desc(ah + o, LBO, SBO), tc::smem_desc(bl + o, LBO, SBO), idesc, 1u);
                    tc::mma_tf32(taddr, tc::smem_desc(al + o, LBO, SBO), tc::smem_desc(bh + o, LBO, SBO), idesc, 1u);
                }
            }
            tc::commit(&mbar);
        }
        tc::mbar_wait(&mbar, phase);
        phase ^= 1;
    }
    tc::fence_after_sync();
    for (int c0 = 0; c0 < 128; c0 += 16) {
        float v[16];
        tc::tmem_ld16(taddr + ((uint32_t)(32 * warp) << 16) + c0, v);
        const int row = 32 * warp + lane;
#pragma unroll
        for (int i = 0; i < 16; ++i) C[(size_t)row * 128 + c0 + i] = v[i];
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(taddr, 128);
}

// ---------------------------------------------------------------------------
// Batched complex Hermitian rank-k update on the tensor cores (c64 data, 3xTF32):
//   Out[set](x, y) = sum_{links of set} sum_t V(x,t) conj(V(y,t)),  x, y < D (GramDesc addressing)
// as two real GEMMs over K' = 2t (re/im interleaved):
//   Re S = Wh Wh^T,  Im S = Wt Wh^T,  Wh(x, 2t..2t+1) = (Vr, Vi),  Wt(x, 2t..2t+1) = (Vi, -Vr).
// CTA = one 128 x 128 output tile of one set; TMEM holds Re (cols 0..127) and Im (128..255);
// K chunks of 32 real (16 complex) are staged by all 256 threads (split into tf32 hi + lo),
// double-buffered so the single MMA-issuing thread overlaps the next chunk's staging.
__device__ __forceinline__ int tc_set_size(const Topo& t, int kind) {
    switch (kind) {
        case FI_USER: return t.J;
        case FI_BASE: return t.J * t.K;
        case FI_LINK: return 1;
        default: return t.links();
    }
}
__device__ __forceinline__ int tc_set_link(const Topo& t, int kind, int s, int r) {
    switch (kind) {
        case FI_USER: {
            const int i = s / t.K, j = s % t.K;
            return (r * t.J + i) * t.K + j;
        }
        case FI_BASE: return s * t.J * t.K + r;
        case FI_LINK: return s;
        default: return r;
    }
}

__global__ void __launch_bounds__(256) k_gram_tc(Topo t, GramDesc d, int sets_per_group, const float2* __restrict__ V,
                                                 float2* __restrict__ out) {
    constexpr int KC = 32, TILE_R = 128;
    constexpr uint32_t TB = TILE_R * KC * 4;  // 16 KB per operand tile
    extern __shared__ __align__(1024) unsigned char smem[];
    // per stage: Ah Al (Wh of x-rows), Th Tl (Wt of x-rows), Bh Bl (Wh of y-rows)
    __shared__ uint64_t mbar[2];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int64_t set = blockIdx.y;
    const int64_t g = set / sets_per_group;
    const int s = (int)(set % sets_per_group);
    const int tiles = (d.D + TILE_R - 1) / TILE_R;
    const int x0 = (blockIdx.x % tiles) * TILE_R, y0 = (blockIdx.x / tiles) * TILE_R;
    const bool diag = x0 == y0;
    if (warp == 0) tc::tmem_alloc(&tmem_base, 256);
    if (tid == 0) {
        tc::mbar_init(&mbar[0], 1);
        tc::mbar_init(&mbar[1], 1);
        tc::fence_barrier_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tre = tmem_base, tim = tmem_base + 128;
    constexpr uint32_t idesc = tc::idesc_tf32(128, 128);
    const int nl = tc_set_size(t, d.set_kind);
    const int Tn = d.T1 * d.T2;
    const int64_t ktot = (int64_t)nl * Tn;  // complex reduction length
    const int nchunks = (int)((ktot + KC / 2 - 1) / (KC / 2));
    uint32_t phase[2] = {0, 0};
    for (int ch = 0; ch < nchunks; ++ch) {
        const int st = ch & 1;
        unsigned char* base = smem + (size_t)st * 6 * TB;
        if (ch >= 2) {  // wait until the MMAs that read this stage (chunk ch-2) are done
            tc::mbar_wait(&mbar[st], phase[st]);
            phase[st] ^= 1;
        }
        // stage 16 complex columns of the x-tile and y-tile rows
        for (int idx = tid; idx < TILE_R * (KC / 2); idx += blockDim.x) {
            const int tc_ = idx % (KC / 2), r = idx / (KC / 2);
            const int64_t kt = (int64_t)ch * (KC / 2) + tc_;
            float2 vx = make_float2(0.f, 0.f), vy = make_float2(0.f, 0.f);
            if (kt < ktot) {
                const int li = (int)(kt / Tn), tt = (int)(kt % Tn);
                const int l = tc_set_link(t, d.set_kind, s, li);
                const float2* vb = V + (g * t.links() + l) * d.v_item +
                                   (int64_t)(tt % d.T1) * d.t1s + (int64_t)(tt / d.T1) * d.t2s;
                if (x0 + r < d.D) vx = vb[(int64_t)(x0 + r) * d.xs];
                if (!diag && y0 + r < d.D) vy = vb[(int64_t)(y0 + r) * d.xs];
            }
            const int k = 2 * tc_;
            const uint32_t o0 = tc::kmajor_off(r, k, KC), o1 = tc::kmajor_off(r, k + 1, KC);
            float h, l_;
            tc::split_tf32(vx.x, h, l_);
            *reinterpret_cast<float*>(base + 0 * TB + o0) = h;
            *reinterpret_cast<float*>(base + 1 * TB + o0) = l_;
            *reinterpret_cast<float*>(base + 3 * TB + o1) = -h;
            *reinterpret_cast<float*>(base + 4 * TB + o1) = -l_;
            tc::split_tf32(vx.y, h, l_);
            *reinterpret_cast<float*>(base + 0 * TB + o1) = h;
            *reinterpret_cast<float*>(base + 1 * TB + o1) = l_;
            *reinterpret_cast<float*>(base + 3 * TB + o0) = h;
            *reinterpret_cast<float*>(base + 4 * TB + o0) = l_;
            if (!diag) {
                tc::split_tf32(vy.x, h, l_);
                *reinterpret_cast<float*>(base + 2 * TB + o0) = h;
                *reinterpret_cast<float*>(base + 5 * TB + o0) = l_;
                tc::split_tf32(vy.y, h, l_);
                *reinterpret_cast<float*>(base + 2 * TB + o1) = h;
                *reinterpret_cast<float*>(base + 5 * TB + o1) = l_;
            }
        }
        tc::fence_async_shared();
        __syncthreads();
        if (tid == 0) {
            tc::fence_after_sync();
            const uint32_t ah = tc::smem_u32(base), al = ah + TB;
            const uint32_t bh = diag ? ah : ah + 2 * TB, bl = diag ? al : ah + 5 * TB;
            const uint32_t th = ah + 3 * TB, tl = ah + 4 * TB;
            constexpr uint32_t LBO = 128, SBO = (KC / 4) * 128;
#pragma unroll
            for (int k8 = 0; k8 < KC / 8; ++k8) {
                const uint32_t o = k8 * 256;
                const uint32_t acc = (ch > 0 || k8 > 0) ? 1u : 0u;
                const uint64_t dbh = tc::smem_desc(bh + o, LBO, SBO), dbl = tc::smem_desc(bl + o, LBO, SBO);
                tc::mma_tf32(tre, tc::smem_desc(ah + o, LBO, SBO), dbh, idesc, acc);
                tc::mma_tf32(tre, tc::smem_desc(ah + o, LBO, SBO), dbl, idesc, 1u);
                tc::mma_tf32(tre, tc::smem_desc(al + o, LBO, SBO), dbh, idesc, 1u);
                tc::mma_tf32(tim, tc::smem_desc(th + o, LBO, SBO), dbh, idesc, acc);
                tc::mma_tf32(tim, tc::smem_desc(th + o, LBO, SBO), dbl, idesc, 1u);
                tc::mma_tf32(tim, tc::smem_desc(tl + o, LBO, SBO), dbh, idesc, 1u);
            }
            tc::commit(&mbar[st]);
        }
    }
    // drain: the last one or two chunks' commits
    for (int st = 0; st < 2; ++st) {
        const int used = nchunks > st ? (nchunks - 1 - st) / 2 + 1 : 0;  // chunks that used stage st
        const int waited = nchunks > st + 2 ? (nchunks - st - 2 + 1) / 2 : 0;
        if (used > waited) tc::mbar_wait(&mbar[st], phase[st]);
    }
    tc::fence_after_sync();
    // epilogue: warps 0-3 read Re, warps 4-7 read Im; warp w owns TMEM lanes 32*(w%4)..
    const int q = warp % 4;
    const bool im = warp >= 4;
    const int x = x0 + 32 * q + lane;
    float2* ob = out + set * (int64_t)d.D * d.D;
    for (int c0 = 0; c0 < 128; c0 += 16) {
        float v[16];
        tc::tmem_ld16((im ? tim : tre) + ((uint32_t)(32 * q) << 16) + c0, v);
        if (x < d.D) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int y = y0 + c0 + i;
                if (y < d.D) {
                    float* o = reinterpret_cast<float*>(ob + x + (int64_t)d.D * y);
                    o[im ? 1 : 0] = v[i];
                }
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem_base, 256);
}

cudaError_t launch_gram_tc(const Topo& t, const GramDesc& d, int64_t ngroups, int sets_per_group, const void* V,
                           void* out, cudaStream_t st) {
    const size_t sm = 2 * 6 * 128 * 32 * 4;  // 192 KB: two stages x six 16 KB operand tiles
    cudaError_t e = cudaFuncSetAttribute(k_gram_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    const int tiles = (d.D + 127) / 128;
    dim3 grid(tiles * tiles, (unsigned)(ngroups * sets_per_group));
    k_gram_tc<<<grid, 256, sm, st>>>(t, d, sets_per_group, (const float2*)V, (float2*)out);
    return cudaGetLastError();
}

}  // namespace gwtk

// Debug/validation entry (device pointers): C[128][128] = A[128][K] * B[128][K]^T.
extern "C" int gwt_debug_tc_gemm(int K, const float* A, const float* B, float* C, int split3) {
    using namespace gwtk;
    const size_t sm = 4 * 128 * 32 * 4;
    cudaError_t e;
    if (split3) {
        e = cudaFuncSetAttribute(k_tc_gemm_test<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e == cudaSuccess) k_tc_gemm_test<true><<<1, 128, sm>>>(K, A, B, C);
    } else {
        e = cudaFuncSetAttribute(k_tc_gemm_test<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e == cudaSuccess) k_tc_gemm_test<false><<<1, 128, sm>>>(K, A, B, C);
    }
    if (e != cudaSuccess) return (int)e;
    e = cudaDeviceSynchronize();
    return (int)e;
}
