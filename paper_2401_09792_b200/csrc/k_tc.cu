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

// ---------------------------------------------------------------------------
// K1 on the tensor cores (c64): per link and subcarrier tile the rebuild
// H~(f) = sum_q G(:,:,q) E_q(f) is one real GEMM with interleaved re/im rows,
//   out[2r][f]   = sum_q  Gr(r,q) Er(q,f) - Gi(r,q) Ei(q,f)   (Re H~(r, f))
//   out[2r+1][f] = sum_q  Gi(r,q) Er(q,f) + Gr(r,q) Ei(q,f)   (Im H~(r, f))
// A' = [[Gr, -Gi]; [Gi, Gr]] (2mn x 2p, row pairs), B' = [Er; Ei] (2p x N), 3xTF32 with the
// fp32 accumulator in TMEM. A' is staged once per CTA (persistent over the link's subcarriers);
// per tile the CUDA cores form the phasors and E (= C^T conj(c(f))) straight into the B' operand,
// one thread issues RB*3*(2p/8) MMAs, and the epilogue streams TMEM rows to H~ (row 2r+i is
// float 2r+i of the link's m*n complex block: consecutive lanes write consecutive floats).
template <int RB, int N>
__global__ void __launch_bounds__(256) k_rebuild_tc(Topo t, int Fc, int64_t f0, int frange, const float2* __restrict__ Cd,
                                                    const float2* __restrict__ G, const double* __restrict__ tau,
                                                    const double* __restrict__ freqs, float* __restrict__ H) {
    constexpr int NT = 256;
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int P = t.P, p = t.p, mn = t.m * t.n, links = t.links();
    const int KP = 2 * p, KC = (KP + 7) / 8 * 8;
    const uint32_t TA = (uint32_t)RB * 128 * KC * 4, TB = (uint32_t)N * KC * 4;
    unsigned char* sAh = smem;
    unsigned char* sAl = smem + TA;
    unsigned char* sBh = smem + 2 * TA;
    unsigned char* sBl = sBh + TB;
    float2* ph = reinterpret_cast<float2*>(sBl + TB);  // [P][N]
    float2* sC = ph + (size_t)P * N;                   // [p][P] (C_l column-major P x p)
    double* st = reinterpret_cast<double*>(sC + (size_t)P * p);
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int l = blockIdx.x;
    const int64_t g = blockIdx.y;
    const int64_t gl = g * links + l;
    if (warp == 0) tc::tmem_alloc(&tmem_base, RB * N < 32 ? 32 : RB * N);
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        tc::fence_barrier_init();
    }
    // A' (hi/lo) from G_l: G_l(r, q) at G[gl*mn*p + r + mn*q]
    const float2* Gl = G + gl * (int64_t)mn * p;
    // zero the padding, then scatter G_l in its native (coalesced) order: element (r, q) feeds
    // A'[2r][q] = Gr, A'[2r][p+q] = -Gi, A'[2r+1][q] = Gi, A'[2r+1][p+q] = Gr
    for (int idx = tid; idx < RB * 128 * KC; idx += NT) {
        const int R = idx / KC, k = idx % KC;
        if (R >= 2 * mn || k >= KP) {
            const uint32_t o = tc::kmajor_off(R, k, KC);
            *reinterpret_cast<float*>(sAh + o) = 0.f;
            *reinterpret_cast<float*>(sAl + o) = 0.f;
        }
    }
    for (int idx = tid; idx < mn * p; idx += NT) {
        const int r = idx % mn, q = idx / mn;
        const float2 gv = Gl[idx];
        const float vals[4] = {gv.x, -gv.y, gv.y, gv.x};
        const int rows[4] = {2 * r, 2 * r, 2 * r + 1, 2 * r + 1};
        const int ks[4] = {q, p + q, q, p + q};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            float hi, lo;
            tc::split_tf32(vals[u], hi, lo);
            const uint32_t o = tc::kmajor_off(rows[u], ks[u], KC);
            *reinterpret_cast<float*>(sAh + o) = hi;
            *reinterpret_cast<float*>(sAl + o) = lo;
        }
    }
    const float2* Cl = Cd + gl * (int64_t)P * p;
    for (int e = tid; e < P * p; e += NT) sC[e] = Cl[e];
    for (int e = tid; e < P; e += NT) st[e] = tau[gl * P + e];
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tbase = tmem_base;
    constexpr uint32_t idesc = tc::idesc_tf32(128, N);
    const uint32_t LBO = 128, SBO = (uint32_t)(KC / 4) * 128;
    const uint32_t ah = tc::smem_u32(sAh), al = tc::smem_u32(sAl), bh = tc::smem_u32(sBh), bl = tc::smem_u32(sBl);
    uint32_t phase = 0;
    const int fbeg = blockIdx.z * frange, fend = min(Fc, fbeg + frange);
    const int64_t fstride = (int64_t)links * mn * 2;  // floats between subcarriers
    for (int ft0 = fbeg; ft0 < fend; ft0 += N) {
        const int nf = min(N, fend - ft0);
        for (int idx = tid; idx < P * N; idx += NT) {
            const int r = idx / N, f = idx % N;
            ph[idx] = f < nf ? conj_coeff<float>(freqs[f0 + ft0 + f], st[r]) : make_float2(0.f, 0.f);
        }
        __syncthreads();
        // B' rows = subcarriers, K' = [Er (q < p) | Ei (q >= p)] (hi/lo), zero padding k >= 2p
        for (int idx = tid; idx < p * N; idx += NT) {
            const int q = idx / N, f = idx % N;
            const float2* cq = sC + (size_t)P * q;
            float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
            int r = 0;
            for (; r + 1 < P; r += 2) {
                cfma(a0, cq[r], ph[r * N + f]);
                cfma(a1, cq[r + 1], ph[(r + 1) * N + f]);
            }
            if (r < P) cfma(a0, cq[r], ph[r * N + f]);
            const float2 e = make_float2(a0.x + a1.x, a0.y + a1.y);
            float hi, lo;
            tc::split_tf32(e.x, hi, lo);
            uint32_t o = tc::kmajor_off(f, q, KC);
            *reinterpret_cast<float*>(sBh + o) = hi;
            *reinterpret_cast<float*>(sBl + o) = lo;
            tc::split_tf32(e.y, hi, lo);
            o = tc::kmajor_off(f, p + q, KC);
            *reinterpret_cast<float*>(sBh + o) = hi;
            *reinterpret_cast<float*>(sBl + o) = lo;
        }
        for (int idx = tid; idx < N * (KC - KP); idx += NT) {
            const int f = idx / (KC - KP), k = KP + idx % (KC - KP);
            const uint32_t o = tc::kmajor_off(f, k, KC);
            *reinterpret_cast<float*>(sBh + o) = 0.f;
            *reinterpret_cast<float*>(sBl + o) = 0.f;
        }
        tc::fence_async_shared();
        __syncthreads();
        if (tid == 0) {
            tc::fence_after_sync();
#pragma unroll
            for (int b = 0; b < RB; ++b) {
                const uint32_t d = tbase + (uint32_t)(b * N);
                const uint32_t ab = ah + (uint32_t)b * 16 * SBO, alb = al + (uint32_t)b * 16 * SBO;
                for (int k8 = 0; k8 < KC / 8; ++k8) {
                    const uint32_t o = k8 * 256;
                    const uint64_t dbh = tc::smem_desc(bh + o, LBO, SBO), dbl = tc::smem_desc(bl + o, LBO, SBO);
                    tc::mma_tf32(d, tc::smem_desc(ab + o, LBO, SBO), dbh, idesc, k8 > 0 ? 1u : 0u);
                    tc::mma_tf32(d, tc::smem_desc(ab + o, LBO, SBO), dbl, idesc, 1u);
                    tc::mma_tf32(d, tc::smem_desc(alb + o, LBO, SBO), dbh, idesc, 1u);
                }
            }
            tc::commit(&mbar);
        }
        tc::mbar_wait(&mbar, phase);
        phase ^= 1;
        tc::fence_after_sync();
        // epilogue: warp w reads TMEM lanes 32(w%4).. (rows b*128 + 32(w%4) + lane) of each row block,
        // warps 0-3 the first half of the subcarrier columns, warps 4-7 the second
        const int wq = warp & 3, ch = warp >> 2;
#pragma unroll
        for (int b = 0; b < RB; ++b) {
            const int R = b * 128 + 32 * wq + lane;
            float* hb = H + ((g * Fc + ft0) * links + l) * (int64_t)mn * 2 + R;
#pragma unroll 1
            for (int c0 = ch * (N / 2); c0 < (ch + 1) * (N / 2); c0 += 16) {
                float v[16];
                tc::tmem_ld16(tbase + (uint32_t)(b * N + c0) + ((uint32_t)(32 * wq) << 16), v);
                if (R < 2 * mn) {
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        if (c0 + i < nf) hb[(int64_t)(c0 + i) * fstride] = v[i];
                }
            }
        }
        tc::fence_before_sync();
        __syncthreads();  // TMEM and B' free for the next tile
    }
    if (warp == 0) tc::tmem_dealloc(tbase, RB * N < 32 ? 32 : RB * N);
}

// Warp-specialised variant of k_rebuild_tc: per CTA (link, group), tiles of N subcarriers flow
// through a 2-stage pipeline
//   producers (warps 0-7): phasors -> E -> B' stage s (hi/lo, K-major)   --bfull[s]-->
//   MMA thread (warp 12):  3xTF32 MMAs into TMEM accumulator s          --afull[s]--> / --bempty[s]-->
//   epilogue (warps 8-11): TMEM -> registers -> H~ rows in HBM          --aempty[s]-->
// so the CUDA-core work of tile t+1, the tensor-core work of tile t and the stores of tile t-1
// overlap inside the CTA.
template <int RB, int N>
__global__ void __launch_bounds__(416, 1) k_rebuild_ws(Topo t, int Fc, int64_t f0, const float2* __restrict__ Cd,
                                                       const float2* __restrict__ G, const double* __restrict__ tau,
                                                       const double* __restrict__ freqs, float* __restrict__ H) {
    constexpr int NPROD = 256, NEPI = 128;
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint64_t bfull[2], bempty[2], afull[2], aempty[2];
    __shared__ uint32_t tmem_base;
    const int P = t.P, p = t.p, mn = t.m * t.n, links = t.links();
    const int KP = 2 * p, KC = (KP + 7) / 8 * 8;
    const uint32_t TA = (uint32_t)RB * 128 * KC * 4, TB = (uint32_t)N * KC * 4;
    unsigned char* sAh = smem;
    unsigned char* sAl = smem + TA;
    unsigned char* sB = smem + 2 * TA;  // [stage][hi, lo] each TB
    float2* ph = reinterpret_cast<float2*>(sB + 4 * TB);  // [P][N]
    float2* sC = ph + (size_t)P * N;                        // [p][P]
    double* st = reinterpret_cast<double*>(sC + (size_t)P * p);
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int l = blockIdx.x;
    const int64_t g = blockIdx.y;
    const int64_t gl = g * links + l;
    if (warp == 0) tc::tmem_alloc(&tmem_base, 4 * RB * N >= 32 ? 2 * RB * N : 32);
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            tc::mbar_init(&bfull[s], NPROD);
            tc::mbar_init(&bempty[s], 1);
            tc::mbar_init(&afull[s], 1);
            tc::mbar_init(&aempty[s], NEPI);
        }
        tc::fence_barrier_init();
    }
    // A' (hi/lo) from G_l, zero padding, C_l and delays (all threads)
    const float2* Gl = G + gl * (int64_t)mn * p;
    for (int idx = tid; idx < RB * 128 * KC; idx += blockDim.x) {
        const int R = idx / KC, k = idx % KC;
        if (R >= 2 * mn || k >= KP) {
            const uint32_t o = tc::kmajor_off(R, k, KC);
            *reinterpret_cast<float*>(sAh + o) = 0.f;
            *reinterpret_cast<float*>(sAl + o) = 0.f;
        }
    }
    for (int idx = tid; idx < mn * p; idx += blockDim.x) {
        const int r = idx % mn, q = idx / mn;
        const float2 gv = Gl[idx];
        const float vals[4] = {gv.x, -gv.y, gv.y, gv.x};
        const int rows[4] = {2 * r, 2 * r, 2 * r + 1, 2 * r + 1};
        const int ks[4] = {q, p + q, q, p + q};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            float hi, lo;
            tc::split_tf32(vals[u], hi, lo);
            const uint32_t o = tc::kmajor_off(rows[u], ks[u], KC);
            *reinterpret_cast<float*>(sAh + o) = hi;
            *reinterpret_cast<float*>(sAl + o) = lo;
        }
    }
    const float2* Cl = Cd + gl * (int64_t)P * p;
    for (int e = tid; e < P * p; e += blockDim.x) sC[e] = Cl[e];
    for (int e = tid; e < P; e += blockDim.x) st[e] = tau[gl * P + e];
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tbase = tmem_base;
    const int ntiles = (Fc + N - 1) / N;
    if (warp < 8) {
        // ---------------- producers
        for (int ti = 0; ti < ntiles; ++ti) {
            const int s = ti & 1, u = ti >> 1;
            const int ft0 = ti * N, nf = min(N, Fc - ft0);
            tc::named_bar(1, NPROD);  // previous tile's E finished reading ph
            for (int idx = tid; idx < P * N; idx += NPROD) {
                const int r = idx / N, f = idx % N;
                ph[idx] = f < nf ? conj_coeff<float>(freqs[f0 + ft0 + f], st[r]) : make_float2(0.f, 0.f);
            }
            tc::named_bar(1, NPROD);
            if (u > 0) tc::mbar_wait(&bempty[s], (u - 1) & 1);
            unsigned char* bh = sB + (size_t)s * 2 * TB;
            unsigned char* bl = bh + TB;
            for (int idx = tid; idx < p * N; idx += NPROD) {
                const int q = idx / N, f = idx % N;
                const float2* cq = sC + (size_t)P * q;
                float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
                int r = 0;
                for (; r + 1 < P; r += 2) {
                    cfma(a0, cq[r], ph[r * N + f]);
                    cfma(a1, cq[r + 1], ph[(r + 1) * N + f]);
                }
                if (r < P) cfma(a0, cq[r], ph[r * N + f]);
                const float2 e = make_float2(a0.x + a1.x, a0.y + a1.y);
                float hi, lo;
                tc::split_tf32(e.x, hi, lo);
                uint32_t o = tc::kmajor_off(f, q, KC);
                *reinterpret_cast<float*>(bh + o) = hi;
                *reinterpret_cast<float*>(bl + o) = lo;
                tc::split_tf32(e.y, hi, lo);
                o = tc::kmajor_off(f, p + q, KC);
                *reinterpret_cast<float*>(bh + o) = hi;
                *reinterpret_cast<float*>(bl + o) = lo;
            }
            for (int idx = tid; idx < N * (KC - KP); idx += NPROD) {
                const int f = idx / (KC - KP), k = KP + idx % (KC - KP);
                const uint32_t o = tc::kmajor_off(f, k, KC);
                *reinterpret_cast<float*>(bh + o) = 0.f;
                *reinterpret_cast<float*>(bl + o) = 0.f;
            }
            tc::fence_async_shared();
            tc::mbar_arrive(&bfull[s]);
        }
    } else if (warp == 12) {
        // ---------------- MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc = tc::idesc_tf32(128, N);
            const uint32_t LBO = 128, SBO = (uint32_t)(KC / 4) * 128;
            const uint32_t ah = tc::smem_u32(sAh), al = tc::smem_u32(sAl);
            for (int ti = 0; ti < ntiles; ++ti) {
                const int s = ti & 1, u = ti >> 1;
                tc::mbar_wait(&bfull[s], u & 1);
                if (u > 0) tc::mbar_wait(&aempty[s], (u - 1) & 1);
                tc::fence_after_sync();
                const uint32_t bh = tc::smem_u32(sB + (size_t)s * 2 * TB), bl = bh + TB;
#pragma unroll
                for (int b = 0; b < RB; ++b) {
                    const uint32_t d = tbase + (uint32_t)((s * RB + b) * N);
                    const uint32_t ab = ah + (uint32_t)b * 16 * SBO, alb = al + (uint32_t)b * 16 * SBO;
                    for (int k8 = 0; k8 < KC / 8; ++k8) {
                        const uint32_t o = k8 * 256;
                        const uint64_t dbh = tc::smem_desc(bh + o, LBO, SBO), dbl = tc::smem_desc(bl + o, LBO, SBO);
                        tc::mma_tf32(d, tc::smem_desc(ab + o, LBO, SBO), dbh, idesc, k8 > 0 ? 1u : 0u);
                        tc::mma_tf32(d, tc::smem_desc(ab + o, LBO, SBO), dbl, idesc, 1u);
                        tc::mma_tf32(d, tc::smem_desc(alb + o, LBO, SBO), dbh, idesc, 1u);
                    }
                }
                tc::commit(&bempty[s]);
                tc::commit(&afull[s]);
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue (warps 8..11 -> TMEM lane quarters 0..3)
        const int wq = warp & 3;
        const int64_t fstride = (int64_t)links * mn * 2;
        for (int ti = 0; ti < ntiles; ++ti) {
            const int s = ti & 1, u = ti >> 1;
            const int ft0 = ti * N, nf = min(N, Fc - ft0);
            tc::mbar_wait(&afull[s], u & 1);
            tc::fence_after_sync();
#pragma unroll
            for (int b = 0; b < RB; ++b) {
                const int R = b * 128 + 32 * wq + lane;
                float* hb = H + ((g * Fc + ft0) * links + l) * (int64_t)mn * 2 + R;
#pragma unroll
                for (int c0 = 0; c0 < N; c0 += 16) {
                    float v[16];
                    tc::tmem_ld16(tbase + (uint32_t)((s * RB + b) * N + c0) + ((uint32_t)(32 * wq) << 16), v);
                    if (R < 2 * mn) {
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            if (c0 + i < nf) hb[(int64_t)(c0 + i) * fstride] = v[i];
                    }
                }
            }
            tc::fence_before_sync();
            tc::mbar_arrive(&aempty[s]);
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (warp == 0) tc::tmem_dealloc(tbase, 4 * RB * N >= 32 ? 2 * RB * N : 32);
}

// c64 rebuild on the tensor cores when 2*m*n <= 256 and (2p) % 8 == 0 fits; returns
// cudaErrorNotSupported otherwise (caller uses the CUDA-core kernel)
cudaError_t launch_rebuild_tc(const Topo& t, int ngroups, int Fc, int64_t f0, const void* Cd, const void* G,
                              const double* tau, const double* freqs, void* H, cudaStream_t st) {
    constexpr int N = 32;
    const int mn = t.m * t.n, KC = (2 * t.p + 7) / 8 * 8;
    const int RB = (2 * mn + 127) / 128;
    if (RB > 2 || KC > 64) return cudaErrorNotSupported;
    const size_t sm = (size_t)2 * RB * 128 * KC * 4 + (size_t)2 * N * KC * 4 + (size_t)t.P * N * 8 + (size_t)t.P * t.p * 8 +
                      (size_t)t.P * 8;
    if (sm > 200 * 1024) return cudaErrorNotSupported;
    const int64_t base = (int64_t)ngroups * t.links();
    int nz = (int)std::max<int64_t>(1, std::min<int64_t>((148 * 4 + base - 1) / base, (Fc + N - 1) / N));
    int frange = (Fc + nz - 1) / nz;
    frange = (frange + N - 1) / N * N;
    nz = (Fc + frange - 1) / frange;
    cudaError_t e;
    const char* mode = std::getenv("GWT_REBUILD_TC");
    if (!(mode && std::atoi(mode) == 2)) {  // warp-specialised pipeline
        constexpr int NW = 32;
        const size_t smw = (size_t)2 * RB * 128 * KC * 4 + (size_t)4 * NW * KC * 4 + (size_t)t.P * NW * 8 +
                           (size_t)t.P * t.p * 8 + (size_t)t.P * 8;
        dim3 gw(t.links(), ngroups);
        if (RB == 1) {
            e = cudaFuncSetAttribute(k_rebuild_ws<1, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smw);
            if (e != cudaSuccess) return e;
            k_rebuild_ws<1, NW><<<gw, 416, smw, st>>>(t, Fc, f0, (const float2*)Cd, (const float2*)G, tau, freqs, (float*)H);
        } else {
            e = cudaFuncSetAttribute(k_rebuild_ws<2, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smw);
            if (e != cudaSuccess) return e;
            k_rebuild_ws<2, NW><<<gw, 416, smw, st>>>(t, Fc, f0, (const float2*)Cd, (const float2*)G, tau, freqs, (float*)H);
        }
        return cudaGetLastError();
    }
    dim3 grid(t.links(), ngroups, nz);
    if (RB == 1) {
        e = cudaFuncSetAttribute(k_rebuild_tc<1, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
        k_rebuild_tc<1, N><<<grid, 256, sm, st>>>(t, Fc, f0, frange, (const float2*)Cd, (const float2*)G, tau, freqs,
                                                  (float*)H);
    } else {
        e = cudaFuncSetAttribute(k_rebuild_tc<2, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
        k_rebuild_tc<2, N><<<grid, 256, sm, st>>>(t, Fc, f0, frange, (const float2*)Cd, (const float2*)G, tau, freqs,
                                                  (float*)H);
    }
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
