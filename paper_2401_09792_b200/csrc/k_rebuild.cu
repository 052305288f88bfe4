// Stage R of the compressed-form SINR for large cores (m n >= 256: C3, C4, C5), complex64.
//
// Reference: assemble_channel_compressed (proj/src/channel.cpp:189-208) for every link at
// every subcarrier: d = C^H c, H~ = G x3 conj(d) — per link a GEMM
//     H~[f](x) = sum_q G(x, q) E(q, f),   E(q, f) = sum_r C(r, q) conj(c_r(f)),
// M = m n rows, K = p, N = subcarriers. Output layout [g][f][link][n][m] (m fastest).
//
// SGEMM-style tiling (CUDA cores, fp32 FMA): one CTA per (64-subcarrier tile, link, group),
// blockIdx.x fastest so the subcarrier tiles of a link run together and its core stays in L2.
//  1. phasors conj(c_r(f)) for the tile (binary64 argument reduction) and E = C^T c* into smem;
//  2. per 128-row chunk of G (staged in smem with coalesced loads): 256 threads, each a 4 x 8
//     (rows x subcarriers) register tile; per q step 4 conflict-free G loads and 4 broadcast
//     16-byte E loads feed 32 complex FMAs; stores are 256-byte row runs per subcarrier.
#include "kernels.cuh"

namespace gwtk {

namespace {
constexpr int kFT = 64;     // subcarriers per CTA
constexpr int kRows = 128;  // rows per chunk
constexpr int kNT = 256;
}  // namespace

__global__ void __launch_bounds__(kNT, 2) k_rebuild_mm(Topo t, int Fc, int64_t f0, const float2* __restrict__ Cd,
                                                       const float2* __restrict__ G, const double* __restrict__ tau,
                                                       const double* __restrict__ freqs, float2* __restrict__ H) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int P = t.P, p = t.p, mn = t.m * t.n, links = t.links();
    float2* sE = reinterpret_cast<float2*>(smem_raw);                 // [p][kFT]
    float2* sG = sE + (size_t)p * kFT;                                // [p][kRows] (chunk), aliased by phasors
    float2* ph = sG;                                                  // [P][kFT] during the E phase
    float2* sC = sG + (size_t)max(p * kRows, P * kFT);                // [q][P] (C_l column-major P x p)
    double* st = reinterpret_cast<double*>(sC + (size_t)P * p);       // [P]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int l = blockIdx.y;
    const int64_t g = blockIdx.z;
    const int64_t gl = g * links + l;
    const int ft0 = blockIdx.x * kFT, nf = min(kFT, Fc - ft0);
    const float2* Cl = Cd + gl * (int64_t)P * p;
    for (int e = tid; e < P * p; e += kNT) sC[e] = Cl[e];
    for (int e = tid; e < P; e += kNT) st[e] = tau[gl * P + e];
    __syncthreads();
    for (int e = tid; e < P * kFT; e += kNT) {
        const int r = e / kFT, f = e % kFT;
        ph[e] = f < nf ? conj_coeff<float>(freqs[f0 + ft0 + f], st[r]) : make_float2(0.f, 0.f);
    }
    __syncthreads();
    // E(q, f): thread per (q, f) pairs, two partial sums for ILP
    for (int e = tid; e < p * kFT; e += kNT) {
        const int q = e / kFT, f = e % kFT;
        const float2* cq = sC + (size_t)q * P;
        float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
        int r = 0;
        for (; r + 1 < P; r += 2) {
            cfma(a0, cq[r], ph[r * kFT + f]);
            cfma(a1, cq[r + 1], ph[(r + 1) * kFT + f]);
        }
        if (r < P) cfma(a0, cq[r], ph[r * kFT + f]);
        sE[e] = make_float2(a0.x + a1.x, a0.y + a1.y);
    }
    const float2* Gl = G + gl * (int64_t)mn * p;
    const int64_t fstride = (int64_t)links * mn;  // H~ stride between subcarriers (complex elements)
    float2* hb = H + ((g * Fc + ft0) * links + l) * (int64_t)mn;
    const int fb = warp * 8;  // this warp's 8 subcarriers
    for (int r0 = 0; r0 < mn; r0 += kRows) {
        const int nr = min(kRows, mn - r0);
        __syncthreads();  // E complete (first pass) / previous chunk consumed
        for (int e = tid; e < p * kRows; e += kNT) {
            const int q = e / kRows, r = e % kRows;
            sG[e] = r < nr ? Gl[(size_t)q * mn + r0 + r] : make_float2(0.f, 0.f);
        }
        __syncthreads();
        float2 acc[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int f = 0; f < 8; ++f) acc[i][f] = make_float2(0.f, 0.f);
#pragma unroll 2
        for (int q = 0; q < p; ++q) {
            float2 gv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) gv[i] = sG[q * kRows + lane + 32 * i];
            const float4* e4 = reinterpret_cast<const float4*>(sE + q * kFT + fb);
#pragma unroll
            for (int f2 = 0; f2 < 4; ++f2) {
                const float4 ev = e4[f2];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    cfma(acc[i][2 * f2], gv[i], make_float2(ev.x, ev.y));
                    cfma(acc[i][2 * f2 + 1], gv[i], make_float2(ev.z, ev.w));
                }
            }
        }
#pragma unroll
        for (int f = 0; f < 8; ++f) {
            if (fb + f < nf) {
                float2* hp = hb + (int64_t)(fb + f) * fstride + r0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int r = lane + 32 * i;
                    if (r < nr) hp[r] = acc[i][f];
                }
            }
        }
    }
}

bool rebuild_mm_fits(const Topo& t) {
    const size_t sm = sizeof(float2) * ((size_t)t.p * kFT + std::max<size_t>((size_t)t.p * kRows, (size_t)t.P * kFT) +
                                        (size_t)t.P * t.p) + 8 * (size_t)t.P;
    return t.m * t.n >= 256 && sm <= 110 * 1024;
}

cudaError_t launch_rebuild_mm(const Topo& t, int ngroups, int Fc, int64_t f0, const void* Cd, const void* G,
                              const double* tau, const double* freqs, void* H, cudaStream_t st) {
    if (!rebuild_mm_fits(t)) return cudaErrorNotSupported;
    const size_t sm = sizeof(float2) * ((size_t)t.p * kFT + std::max<size_t>((size_t)t.p * kRows, (size_t)t.P * kFT) +
                                        (size_t)t.P * t.p) + 8 * (size_t)t.P;
    cudaError_t e = cudaFuncSetAttribute(k_rebuild_mm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    dim3 grid((Fc + kFT - 1) / kFT, t.links(), ngroups);
    k_rebuild_mm<<<grid, kNT, sm, st>>>(t, Fc, f0, (const float2*)Cd, (const float2*)G, tau, freqs, (float2*)H);
    return cudaGetLastError();
}

}  // namespace gwtk
