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

// ---------------------------------------------------------------------------------------------
// Tucker Gram on the tensor cores for unfoldings whose rows are contiguous blocks of T1 complex values
// (GramDesc xs == T1, t1s == 1): the transmit-mode Gram of W2 = Y1 x1 A^H ([link][p][N][m], T1 = m,
// decompose.cpp:160-176), Out[set](x, y) = sum over the set's links and t2 of V(x, :) V(y, :)^H.
//
// One CTA per (128-row x strip, set): the B operand is rows [0, nb) with nb = 128 (xt + 1) (so the strip
// covers every y <= x, the lower triangle, with no wasted tile) and the A operand is the strip's own rows,
// i.e. the last 128 rows of the B tile (descriptor offset, no separate A tile). Per (link, t2) chunk the nb
// rows are ONE contiguous block of nb T1 complex values:
//   warp 8 (one thread): TMA bulk copy of the raw block (cp.async.bulk, 3 raw stages);
//   warps 0-7          : convert raw -> canonical K-major tf32 tiles, 3xTF32 split: B = [vr, vi] and
//                        P = [-vi, vr], hi / lo each (2 tile stages);
//   warp 9 (one thread): 12 tcgen05.mma per chunk (M = 128, N = nb <= 256, K = 2 T1):
//                        Re += A_h B_h + A_h B_l + A_l B_h, Im += A_h P_h + A_h P_l + A_l P_h, TMEM;
//   warps 0-7          : epilogue, TMEM -> Gram strip (Re warps 0-3, Im warps 4-7).
// N = 256 halves the shared-memory operand bytes per MAC of 128 x 128 tiles (the previous form was
// shared-pipe bound at 52 % with the tensor pipe at 34 %).
namespace {
constexpr int kGT = 128;
constexpr int kGTThreads = 320;
constexpr int kGMaxRows = 256;
}  // namespace

template <int T1>
__global__ void __launch_bounds__(kGTThreads, 1) k_gram_tcb(Topo t, GramDesc d, int sets_per_group,
                                                           const float2* __restrict__ V, float2* __restrict__ out) {
    constexpr int KC = 2 * T1;                             // real K per chunk
    constexpr uint32_t TILE = kGMaxRows * KC * 4;          // one operand tile of up to 256 rows (bytes)
    constexpr uint32_t RAW = kGMaxRows * T1 * 8;           // one raw block of up to 256 rows
    constexpr uint32_t SBO = (KC / 4) * 128;
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* raw = smem;                              // [3] RAW each
    unsigned char* tiles = smem + 3 * RAW;                  // [2][Bh Bl Ph Pl] TILE each
    __shared__ uint64_t raw_full[3], raw_empty[3], tile_full[2], tile_empty[2], acc_full;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int64_t set = blockIdx.y;
    const int64_t g = set / sets_per_group;
    const int s = (int)(set % sets_per_group);
    const int xt = blockIdx.x, x0 = xt * kGT;
    const int nb = min(kGT * (xt + 1), d.D);                // B rows: [0, nb)
    const int nbp = (nb + 15) / 16 * 16;                     // MMA N (multiple of 16)
    const int nl = tc_set_size(t, d.set_kind);
    const int nch = nl * d.T2;
    if (warp == 0) tc::tmem_alloc(&tmem_base, 512);
    if (tid == 0) {
        for (int i = 0; i < 3; ++i) {
            tc::mbar_init(&raw_full[i], 1);
            tc::mbar_init(&raw_empty[i], 256);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&tile_full[i], 256);
            tc::mbar_init(&tile_empty[i], 1);
        }
        tc::mbar_init(&acc_full, 1);
        tc::fence_barrier_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tre = tmem_base, tim = tmem_base + 256;
    if (warp == 8) {
        // ---------------- TMA producer
        if (lane == 0) {
            const uint32_t bytes = (uint32_t)nb * T1 * 8;
            for (int c = 0; c < nch; ++c) {
                const int st = c % 3, use = c / 3;
                if (use > 0) tc::mbar_wait(&raw_empty[st], (use - 1) & 1);
                const int li = c / d.T2, t2 = c % d.T2;
                const int l = tc_set_link(t, d.set_kind, s, li);
                tc::mbar_arrive_expect_tx(&raw_full[st], bytes);
                tc::bulk_g2s(raw + (size_t)st * RAW, V + (g * t.links() + l) * d.v_item + (int64_t)t2 * d.t2s, bytes,
                             &raw_full[st]);
            }
        }
        __syncwarp();
    } else if (warp == 9) {
        // ---------------- MMA issuer: the whole warp waits, one elected lane issues (under elect.sync the
        // UTCHMMAs compile back to back; in a `lane == 0` region each sits in an ELECT / BRA.U.ANY loop, ~240
        // cycles per MMA on the lone thread against the 128-cycle floor of N = 256, tools/micro/mma_fetch.cu)
        const uint32_t idesc = tc::idesc_tf32(kGT, nbp);
        const uint32_t aoff = (uint32_t)(x0 / 8) * SBO;  // the strip's rows inside the B tiles
        for (int c = 0; c < nch; ++c) {
            const int st = c & 1, use = c >> 1;
            tc::mbar_wait(&tile_full[st], use & 1);
            tc::fence_after_sync();
            if (tc::elect_one()) {
                const uint32_t b0 = tc::smem_u32(tiles + (size_t)st * 4 * TILE);
                const uint64_t dBh = tc::smem_desc(b0, 128, SBO), dBl = tc::smem_desc(b0 + TILE, 128, SBO);
                const uint64_t dPh = tc::smem_desc(b0 + 2 * TILE, 128, SBO), dPl = tc::smem_desc(b0 + 3 * TILE, 128, SBO);
                const uint64_t dAh = tc::smem_desc(b0 + aoff, 128, SBO), dAl = tc::smem_desc(b0 + TILE + aoff, 128, SBO);
                const uint32_t acc0 = c > 0 ? 1u : 0u;
#pragma unroll
                for (int kk = 0; kk < KC / 8; ++kk) {
                    const uint64_t o = (uint64_t)kk * 16;  // 256-byte k-step in the 16-byte address field
                    const uint32_t acc = kk > 0 ? 1u : acc0;
                    tc::mma_tf32(tre, dAh + o, dBh + o, idesc, acc);
                    tc::mma_tf32(tre, dAh + o, dBl + o, idesc, 1u);
                    tc::mma_tf32(tre, dAl + o, dBh + o, idesc, 1u);
                    tc::mma_tf32(tim, dAh + o, dPh + o, idesc, acc);
                    tc::mma_tf32(tim, dAh + o, dPl + o, idesc, 1u);
                    tc::mma_tf32(tim, dAl + o, dPh + o, idesc, 1u);
                }
                tc::commit(&tile_empty[st]);
                if (c == nch - 1) tc::commit(&acc_full);
            }
            __syncwarp();
        }
    } else {
        // ---------------- converters (256 threads): 16-byte units (2 complex) of the raw block
        const int units = nbp * T1 / 2;
        for (int c = 0; c < nch; ++c) {
            const int rs = c % 3, ru = c / 3, ts = c & 1, tu = c >> 1;
            tc::mbar_wait(&raw_full[rs], ru & 1);
            if (tu > 0) tc::mbar_wait(&tile_empty[ts], (tu - 1) & 1);
            const float4* rv = reinterpret_cast<const float4*>(raw + (size_t)rs * RAW);
            unsigned char* tb = tiles + (size_t)ts * 4 * TILE;
            for (int u = tid; u < units; u += 256) {
                const int r = u / (T1 / 2), k4 = (u % (T1 / 2)) * 4;  // row, first real K of the unit
                const uint32_t o = (uint32_t)((r >> 3) * SBO + (k4 >> 2) * 128 + (r & 7) * 16);
                const float4 v = r < nb ? rv[u] : make_float4(0.f, 0.f, 0.f, 0.f);
                float4 h, l;
                tc::split_tf32_rn(v.x, h.x, l.x);
                tc::split_tf32_rn(v.y, h.y, l.y);
                tc::split_tf32_rn(v.z, h.z, l.z);
                tc::split_tf32_rn(v.w, h.w, l.w);
                *reinterpret_cast<float4*>(tb + o) = h;
                *reinterpret_cast<float4*>(tb + TILE + o) = l;
                // P = [-vi, vr] per complex
                *reinterpret_cast<float4*>(tb + 2 * TILE + o) = make_float4(-h.y, h.x, -h.w, h.z);
                *reinterpret_cast<float4*>(tb + 3 * TILE + o) = make_float4(-l.y, l.x, -l.w, l.z);
            }
            tc::fence_async_shared();
            tc::mbar_arrive(&tile_full[ts]);
            tc::mbar_arrive(&raw_empty[rs]);
        }
        // ---------------- epilogue: rows x of the strip, columns y < nb (the strictly lower part and the whole
        // diagonal block, as the CUDA-core Gram writes them)
        tc::mbar_wait(&acc_full, 0);
        tc::fence_after_sync();
        const int q = warp % 4;
        const bool im = warp >= 4;
        const int x = x0 + 32 * q + lane;
        float2* ob = out + set * (int64_t)d.D * d.D;
        for (int c0 = 0; c0 < nbp; c0 += 16) {
            float v[16];
            tc::tmem_ld16((im ? tim : tre) + ((uint32_t)(32 * q) << 16) + c0, v);
            if (x < d.D) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int y = c0 + i;
                    if (y < nb && (y <= x || y >= x0)) reinterpret_cast<float*>(ob + x + (int64_t)d.D * y)[im ? 1 : 0] = v[i];
                }
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (warp == 0) tc::tmem_dealloc(tmem_base, 512);
}

bool gram_tc_fits(const GramDesc& d) {
    return d.xs == d.T1 && d.t1s == 1 && (d.T1 == 4 || d.T1 == 8) && d.D >= 128 && d.D <= kGMaxRows && d.D % 8 == 0;
}

cudaError_t launch_gram_tc(const Topo& t, const GramDesc& d, int64_t ngroups, int sets_per_group, const void* V,
                           void* out, cudaStream_t st) {
    if (!gram_tc_fits(d)) return cudaErrorNotSupported;
    const int strips = (d.D + kGT - 1) / kGT;
    dim3 grid(strips, (unsigned)(ngroups * sets_per_group));
    cudaError_t e;
#define GWT_GTC(TT)                                                                                                \
    do {                                                                                                           \
        const size_t sm = 3 * (size_t)kGMaxRows * TT * 8 + 2 * 4 * (size_t)kGMaxRows * 2 * TT * 4;                 \
        e = cudaFuncSetAttribute(k_gram_tcb<TT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);            \
        if (e != cudaSuccess) return e;                                                                            \
        k_gram_tcb<TT><<<grid, kGTThreads, sm, st>>>(t, d, sets_per_group, (const float2*)V, (float2*)out);        \
    } while (0)
    if (d.T1 == 8) GWT_GTC(8);
    else GWT_GTC(4);
#undef GWT_GTC
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
