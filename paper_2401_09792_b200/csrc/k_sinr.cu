// Compressed-form SINR stage (hot path b), sm_100a.
//
// Reference semantics: run_compressed_pipeline (proj/src/sinr.cpp:296-326) =
//   assemble_all_compressed (sinr.cpp:147-160 / channel.cpp:189-208)
//   -> precoders_compressed (truncated_svd, sinr.cpp:162-182)
//   -> per user covariance_compressed (:184-203), woodbury_inverse_apply (:205-227),
//      filter_compressed (:229-240), sinr_compressed/stream_sinrs (:242-254, :28-43),
// batched over F coefficient grids (subcarriers) and many groups.
//
// B200 formulation: everything after the rebuild is expressed
// through m x m Gram matrices, so no n-length vector is ever materialised:
//   serving Gram  A_u = H~_{iij} H~_{iij}^H              -> eig -> U, lambda (sigma^2)
//   precoder      V_u = H~^H U Lambda^{-1/2} (never formed)
//   pair Gram     X_{u,(k,l)} = H~_{kij} H~_{kkl}^H       (interferer k, its user l)
//   covariance    Q = s^2 I + U_L Lambda_L U_L^H + sum X P_{kl} X^H,
//                 P_{kl} = U'_L Lambda'^{-1}_L U'^H_L
//   filter/SINR   w_r = Q^{-1} g_r, g_r = sqrt(lambda_r) u_r;
//                 gamma_r = g_r^H Q^{-1} g_r (Cholesky + forward solve)
//                 signal_r = gamma_r^2, SINR_r = gamma_r / (1 - gamma_r)
// which equals the reference's W~ = (1/s^2)(HV - T HV) route algebraically.
#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"
#include "small_linalg.cuh"

namespace gwtk {


// ---------------------------------------------------------------------------
// K1: rebuild H~(f) = sum_q G(:,:,q) * E[q][f],
//     E[q][f] = sum_r C(r,q) * conj(c_r(f)),  c_r(f) = exp(+j 2 pi f tau_r) or explicit.
// grid (ceil(Fc/FT), links, groups); one CTA per (link, subcarrier tile).
#ifdef GWT_PHASE_TIMERS
__device__ long long g_rb_phase[4];
extern "C" int gwt_debug_rebuild_phases(long long* out4) {
    return (int)cudaMemcpyFromSymbol(out4, g_rb_phase, 4 * sizeof(long long));
}
#define GWT_CLK(v) const long long v = clock64()
#else
#define GWT_CLK(v)
#endif
template <class T, int FT>
__global__ void __launch_bounds__(128) k_rebuild(Topo t, int Fc, int64_t f0, int64_t Ftot,
                                                 const cplx_t<T>* __restrict__ Cd, const cplx_t<T>* __restrict__ G,
                                                 const double* __restrict__ tau, const double* __restrict__ freqs,
                                                 const cplx_t<T>* __restrict__ coeffs, cplx_t<T>* __restrict__ H) {
    using C = cplx_t<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* ph = reinterpret_cast<C*>(smem_raw);  // [P][FT]
    C* E = ph + t.P * FT;                    // [p][FT]
    const int g = blockIdx.z, l = blockIdx.y, ft0 = blockIdx.x * FT;
    const int nf = min(FT, Fc - ft0);
    const int links = t.links();
    const int64_t gl = (int64_t)g * links + l;
    GWT_CLK(c0);
    for (int idx = threadIdx.x; idx < t.P * FT; idx += blockDim.x) {
        const int r = idx / FT, f = idx % FT;
        C v = czero<C>();
        if (f < nf) {
            const int64_t fa = f0 + ft0 + f;
            if (coeffs) {
                v = cconj(coeffs[(((int64_t)g * Ftot + fa) * links + l) * t.P + r]);
            } else {
                v = conj_coeff<T>(freqs[fa], tau[gl * t.P + r]);
            }
        }
        ph[idx] = v;
    }
    __syncthreads();
    GWT_CLK(c1);
    const C* Cl = Cd + gl * t.P * t.p;
    for (int idx = threadIdx.x; idx < t.p * FT; idx += blockDim.x) {
        const int q = idx / FT, f = idx % FT;
        C acc = czero<C>();
        for (int r = 0; r < t.P; ++r) cfma(acc, Cl[r + t.P * q], ph[r * FT + f]);
        E[idx] = acc;
    }
    __syncthreads();
    GWT_CLK(c2);
    const int mn = t.m * t.n;
    const C* Gl = G + gl * mn * t.p;
    for (int row = threadIdx.x; row < mn; row += blockDim.x) {
        C acc[FT];
#pragma unroll
        for (int f = 0; f < FT; ++f) acc[f] = czero<C>();
        const C* gp = Gl + row;
        for (int q = 0; q < t.p; ++q, gp += mn) {
            const C gv = *gp;
            if constexpr (sizeof(C) == 8) {
                // two complex64 per 128-bit shared load (E row is 16-byte aligned)
                const float4* e4 = reinterpret_cast<const float4*>(E + q * FT);
#pragma unroll
                for (int f = 0; f < FT / 2; ++f) {
                    const float4 ev = e4[f];
                    cfma(acc[2 * f], gv, C{ev.x, ev.y});
                    cfma(acc[2 * f + 1], gv, C{ev.z, ev.w});
                }
            } else {
#pragma unroll
                for (int f = 0; f < FT; ++f) cfma(acc[f], gv, E[q * FT + f]);
            }
        }
#pragma unroll
        for (int f = 0; f < FT; ++f)
            if (f < nf) H[(((int64_t)g * Fc + ft0 + f) * links + l) * mn + row] = acc[f];
    }
#ifdef GWT_PHASE_TIMERS
    if (blockIdx.x == 3 && blockIdx.y == 5 && blockIdx.z == 7 && threadIdx.x == 0) {
        const long long c3 = clock64();
        g_rb_phase[0] = c1 - c0;
        g_rb_phase[1] = c2 - c1;
        g_rb_phase[2] = c3 - c2;
    }
#endif
}

// K1 (persistent per link): one CTA per (link, group, subcarrier range) keeps the link's delay
// factor C_l (P x p), core G_l (mn x p) and delays in shared memory and walks its subcarriers in
// tiles of FT: phasors -> E (p x FT) -> H~ rows. Every global read happens once per CTA; the inner
// loops only touch shared memory (E read as 16-byte pairs of subcarriers). 128 threads; work items
// (row, 8-subcarrier block) for the rebuild, (q, subcarrier pair) for E.
template <class T, int FT>
__global__ void __launch_bounds__(128) k_rebuild_link(Topo t, int Fc, int64_t f0, int64_t Ftot, int frange,
                                                      const cplx_t<T>* __restrict__ Cd, const cplx_t<T>* __restrict__ G,
                                                      const double* __restrict__ tau, const double* __restrict__ freqs,
                                                      cplx_t<T>* __restrict__ H) {
    using C = cplx_t<T>;
    constexpr int NT = 128, FB = 8, NB = FT / FB;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int P = t.P, p = t.p, mn = t.m * t.n, links = t.links();
    C* ph = reinterpret_cast<C*>(smem_raw);   // [P][FT]
    C* E = ph + (size_t)P * FT;               // [p][FT]
    C* sG = E + (size_t)p * FT;               // [p][mn]
    C* sC = sG + (size_t)p * mn;              // [p][P]  (C_l column-major P x p)
    double* st = reinterpret_cast<double*>(sC + (size_t)p * P);  // [P]
    const int l = blockIdx.x;
    const int64_t g = blockIdx.y;
    const int64_t gl = g * links + l;
    const int tid = threadIdx.x;
    const C* Gl = G + gl * (int64_t)mn * p;
    const C* Cl = Cd + gl * (int64_t)P * p;
    for (int e = tid; e < mn * p; e += NT) sG[e] = Gl[e];
    for (int e = tid; e < P * p; e += NT) sC[e] = Cl[e];
    for (int e = tid; e < P; e += NT) st[e] = tau[gl * P + e];
    const int fbeg = blockIdx.z * frange, fend = min(Fc, fbeg + frange);
    const int64_t fstride = (int64_t)links * mn;  // H~ stride between subcarriers
    for (int ft0 = fbeg; ft0 < fend; ft0 += FT) {
        const int nf = min(FT, fend - ft0);
        __syncthreads();  // previous tile's E consumed (and staging done on the first pass)
        for (int idx = tid; idx < P * FT; idx += NT) {
            const int r = idx / FT, f = idx % FT;
            ph[idx] = f < nf ? conj_coeff<T>(freqs[f0 + ft0 + f], st[r]) : czero<C>();
        }
        __syncthreads();
        // E[q][f..f+1] = sum_r C_l(r, q) ph[r][f..f+1]
        for (int idx = tid; idx < p * (FT / 2); idx += NT) {
            const int q = idx / (FT / 2), f = 2 * (idx % (FT / 2));
            const C* cq = sC + (size_t)P * q;
            C a0 = czero<C>(), a1 = czero<C>(), b0 = czero<C>(), b1 = czero<C>();
            int r = 0;
            for (; r + 1 < P; r += 2) {
                const C c0 = cq[r], c1 = cq[r + 1];
                cfma(a0, c0, ph[r * FT + f]);
                cfma(a1, c0, ph[r * FT + f + 1]);
                cfma(b0, c1, ph[(r + 1) * FT + f]);
                cfma(b1, c1, ph[(r + 1) * FT + f + 1]);
            }
            if (r < P) {
                cfma(a0, cq[r], ph[r * FT + f]);
                cfma(a1, cq[r], ph[r * FT + f + 1]);
            }
            E[q * FT + f] = cadd(a0, b0);
            E[q * FT + f + 1] = cadd(a1, b1);
        }
        __syncthreads();
        for (int w = tid; w < mn * NB; w += NT) {
            const int row = w % mn, fb = (w / mn) * FB;
            C acc[FB];
#pragma unroll
            for (int f = 0; f < FB; ++f) acc[f] = czero<C>();
            for (int q = 0; q < p; ++q) {
                const C gv = sG[(size_t)q * mn + row];
                const C* eq = E + q * FT + fb;
                if constexpr (sizeof(C) == 8) {
                    const float4* e4 = reinterpret_cast<const float4*>(eq);
#pragma unroll
                    for (int f = 0; f < FB / 2; ++f) {
                        const float4 ev = e4[f];
                        cfma(acc[2 * f], gv, C{ev.x, ev.y});
                        cfma(acc[2 * f + 1], gv, C{ev.z, ev.w});
                    }
                } else {
#pragma unroll
                    for (int f = 0; f < FB; ++f) cfma(acc[f], gv, eq[f]);
                }
            }
            C* hp = H + ((g * Fc + ft0 + fb) * links + l) * (int64_t)mn + row;
#pragma unroll
            for (int f = 0; f < FB; ++f, hp += fstride)
                if (fb + f < nf) *hp = acc[f];
        }
    }
}

// K1 v2 (register-blocked; the default for c64/c128 when p <= 32): ncu showed k_rebuild_link
// limited by the L1/shared-memory pipe (l1tex 83 %, FMA pipe 49 %): every cMAC of H~ = G E re-read
// one G entry and half an E pair. Here each thread keeps an RB x 8 block of H~ (RB rows 32 apart,
// 8 subcarriers) in registers, so one q step costs RB conflict-free G loads + 4 broadcast 16-byte E
// loads for 32*RB FFMA; E = C^T ph is blocked as (subcarrier, half of the q range) with two q per
// 16-byte broadcast load of the transposed C. Phasors are formed once per (tap, subcarrier) tile
// entry (binary64 argument reduction, conj_coeff). One CTA per (subcarrier tile range, link, group).
template <class T, int FT, int RB, int PH, bool GS>
__global__ void __launch_bounds__(128) k_rebuild_rb(Topo t, int Fc, int64_t f0, int tpc,
                                                    const cplx_t<T>* __restrict__ Cd, const cplx_t<T>* __restrict__ G,
                                                    const double* __restrict__ tau, const double* __restrict__ freqs,
                                                    cplx_t<T>* __restrict__ H) {
    using C = cplx_t<T>;
    constexpr int NT = 128, QG = NT / FT;  // q groups in the E phase
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int P = t.P, p = t.p, mn = t.m * t.n, links = t.links();
    const int pp = QG * PH;  // padded q extent (C^T row length, E rows)
    C* ph = reinterpret_cast<C*>(smem_raw);  // [P][FT]
    C* E = ph + (size_t)P * FT;              // [pp][FT]
    C* sG = E + (size_t)pp * FT;             // [p][mn]
    C* sCt = sG + (GS ? (size_t)p * mn : 0);  // [P][pp]  (transposed C_l, zero padded)
    double* st = reinterpret_cast<double*>(sCt + (size_t)P * pp);  // [P]
    const int l = blockIdx.y;
    const int64_t g = blockIdx.z;
    const int64_t gl = g * links + l;
    const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
    const C* Gl = G + gl * (int64_t)mn * p;
    const C* Cl = Cd + gl * (int64_t)P * p;
    if constexpr (GS)
        for (int e = tid; e < mn * p; e += NT) sG[e] = Gl[e];
    for (int e = tid; e < P * pp; e += NT) {
        const int r = e / pp, q = e % pp;
        sCt[e] = q < p ? Cl[r + (size_t)P * q] : czero<C>();
    }
    for (int e = tid; e < P; e += NT) st[e] = tau[gl * P + e];
    const int ntile = (Fc + FT - 1) / FT;
    const int tbeg = blockIdx.x * tpc, tend = min(ntile, tbeg + tpc);
    const int64_t fstride = (int64_t)links * mn;  // H~ stride between subcarriers
    const int nrb = (mn + 32 * RB - 1) / (32 * RB);
    for (int tile = tbeg; tile < tend; ++tile) {
        const int ft0 = tile * FT, nf = min(FT, Fc - ft0);
        __syncthreads();  // previous tile's ph/E consumed (and staging done on the first pass)
        {
            const int f = tid % FT;
            const double fr = f < nf ? freqs[f0 + ft0 + f] : 0.0;
            for (int r = tid / FT; r < P; r += QG) ph[r * FT + f] = f < nf ? conj_coeff<T>(fr, st[r]) : czero<C>();
        }
        __syncthreads();
        {
            const int f = tid % FT, q0 = (tid / FT) * PH;
            C acc[PH];
#pragma unroll
            for (int i = 0; i < PH; ++i) acc[i] = czero<C>();
            for (int r = 0; r < P; ++r) {
                const C x = ph[r * FT + f];
                const C* cr = sCt + (size_t)r * pp + q0;
                if constexpr (sizeof(C) == 8 && PH % 2 == 0) {
                    const float4* c4 = reinterpret_cast<const float4*>(cr);  // pp, q0 even: 16-byte aligned
#pragma unroll
                    for (int i = 0; i < PH / 2; ++i) {
                        const float4 cv = c4[i];
                        cfma(acc[2 * i], C{cv.x, cv.y}, x);
                        cfma(acc[2 * i + 1], C{cv.z, cv.w}, x);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < PH; ++i) cfma(acc[i], cr[i], x);
                }
            }
#pragma unroll
            for (int i = 0; i < PH; ++i) E[(q0 + i) * FT + f] = acc[i];
        }
        __syncthreads();
        for (int item = warp; item < nrb * (FT / 8); item += NT / 32) {
            const int rb = item % nrb, fb = (item / nrb) * 8;
            if (fb >= nf) continue;
            const int row0 = rb * 32 * RB + lane;
            C acc[RB][8];
#pragma unroll
            for (int u = 0; u < RB; ++u)
#pragma unroll
                for (int f = 0; f < 8; ++f) acc[u][f] = czero<C>();
            for (int q = 0; q < p; ++q) {
                C gv[RB];
#pragma unroll
                for (int u = 0; u < RB; ++u) {
                    const int row = row0 + 32 * u;
                    if constexpr (GS) gv[u] = row < mn ? sG[(size_t)q * mn + row] : czero<C>();
                    else gv[u] = row < mn ? __ldg(Gl + (size_t)q * mn + row) : czero<C>();
                }
                const C* eq = E + q * FT + fb;
                if constexpr (sizeof(C) == 8) {
                    const float4* e4 = reinterpret_cast<const float4*>(eq);
#pragma unroll
                    for (int f2 = 0; f2 < 4; ++f2) {
                        const float4 ev = e4[f2];
#pragma unroll
                        for (int u = 0; u < RB; ++u) {
                            cfma(acc[u][2 * f2], gv[u], C{ev.x, ev.y});
                            cfma(acc[u][2 * f2 + 1], gv[u], C{ev.z, ev.w});
                        }
                    }
                } else {
#pragma unroll
                    for (int f = 0; f < 8; ++f) {
                        const C ev = eq[f];
#pragma unroll
                        for (int u = 0; u < RB; ++u) cfma(acc[u][f], gv[u], ev);
                    }
                }
            }
            C* hp = H + ((g * Fc + ft0 + fb) * links + l) * (int64_t)mn;
#pragma unroll
            for (int f = 0; f < 8; ++f, hp += fstride)
                if (fb + f < nf)
#pragma unroll
                    for (int u = 0; u < RB; ++u) {
                        const int row = row0 + 32 * u;
                        if (row < mn) hp[row] = acc[u][f];
                    }
        }
    }
}

template <class T, int FT, int RB, int PH, bool GS>
static cudaError_t launch_rebuild_rb_t(const Topo& t, int ngroups, int Fc, int64_t f0, const void* Cd, const void* G,
                                       const double* tau, const double* freqs, void* H, cudaStream_t st) {
    using C = cplx_t<T>;
    const int pp = (128 / FT) * PH, mn = t.m * t.n;
    const size_t sm = sizeof(C) * ((size_t)t.P * FT + (size_t)pp * FT + (GS ? (size_t)t.p * mn : 0) + (size_t)t.P * pp) +
                      8 * (size_t)t.P;
    if (sm > 200 * 1024) return cudaErrorNotSupported;
    cudaError_t e = cudaFuncSetAttribute(k_rebuild_rb<T, FT, RB, PH, GS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sm);
    if (e != cudaSuccess) return e;
    const int ntile = (Fc + FT - 1) / FT;
    const int64_t base = (int64_t)ngroups * t.links();
    // tiles per CTA: as many as keeps >= ~6 CTAs per SM in the grid (amortises the C/G staging),
    // then evened out so no CTA gets a short remainder
    int tpc = (int)std::max<int64_t>(1, std::min<int64_t>(ntile, (base * ntile) / (148 * 6)));
    const int nz = (ntile + tpc - 1) / tpc;
    tpc = (ntile + nz - 1) / nz;
    dim3 grid((ntile + tpc - 1) / tpc, t.links(), ngroups);
    k_rebuild_rb<T, FT, RB, PH, GS><<<grid, 128, sm, st>>>(t, Fc, f0, tpc, (const C*)Cd, (const C*)G, tau, freqs, (C*)H);
    return cudaGetLastError();
}

// dispatch: RB by the row count (mn a multiple of 96 -> 3, of 64 -> 2, else 1), PH by p; G staged in
// shared memory when it is small (<= 32 KB), else read through L1/L2 (C3/C4: 60-200 KB per link)
template <class T, int FT>
static cudaError_t launch_rebuild_rb(const Topo& t, int ngroups, int Fc, int64_t f0, const void* Cd, const void* G,
                                     const double* tau, const double* freqs, void* H, cudaStream_t st) {
    constexpr int QG = 128 / FT;
    const int mn = t.m * t.n;
    const int ph = (t.p + QG - 1) / QG;
    const int rb = (sizeof(T) == 4 && mn % 96 == 0) ? 3 : (mn % 64 == 0 ? 2 : 1);
    const char* gse = std::getenv("GWT_REBUILD_GSMEM");
    const bool gs = gse ? std::atoi(gse) != 0 : (size_t)mn * t.p * sizeof(cplx_t<T>) <= 32 * 1024;
#define GWT_RB(RBV, PHV)                                                                                        \
    if (rb == RBV && ph <= PHV)                                                                                 \
        return gs ? launch_rebuild_rb_t<T, FT, RBV, PHV, true>(t, ngroups, Fc, f0, Cd, G, tau, freqs, H, st)   \
                  : launch_rebuild_rb_t<T, FT, RBV, PHV, false>(t, ngroups, Fc, f0, Cd, G, tau, freqs, H, st);
    if (QG == 2) {
        GWT_RB(3, 6) GWT_RB(3, 8) GWT_RB(3, 12) GWT_RB(3, 16) GWT_RB(2, 6) GWT_RB(2, 8) GWT_RB(2, 12) GWT_RB(2, 16)
        GWT_RB(1, 8) GWT_RB(1, 16)
    } else {
        GWT_RB(3, 4) GWT_RB(3, 6) GWT_RB(3, 8) GWT_RB(2, 4) GWT_RB(2, 6) GWT_RB(2, 8) GWT_RB(1, 4) GWT_RB(1, 8)
    }
#undef GWT_RB
    return cudaErrorNotSupported;
}

// scope slot s of user (i,j) -> (k,l), mirroring scope_pairs (sinr.cpp:47-62)
__device__ __forceinline__ void scope_slot(const Topo& t, int scope, int i, int j, int s, int& k, int& l) {
    if (scope == 0) {  // full: all (k,l) k-major
        k = s / t.K;
        l = s % t.K;
    } else {  // paper_experiment: (i,j) then (k,0) for k != i ascending
        if (s == 0) {
            k = i;
            l = j;
        } else {
            k = s - 1;
            if (k >= i) ++k;
            l = 0;
        }
    }
}
__device__ __forceinline__ int serving_slot(const Topo& t, int scope, int i, int j) {
    return scope == 0 ? i * t.K + j : 0;
}

// ---------------------------------------------------------------------------
// K2: pair Grams X_{u,s} = H~_{k,i,j} H~_{k,k,l}^H (m x m, fp64 accumulation)
// one warp per (group, subcarrier, user); lanes over (slot, a, b) entries.
template <class T>
__global__ void __launch_bounds__(128) k_pair_gram(Topo t, int scope, int S, int Fc, int64_t f0, int64_t Ftot,
                                                   int64_t items, const cplx_t<T>* __restrict__ H,
                                                   double2* __restrict__ PG) {
    using C = cplx_t<T>;
    const int64_t item = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (item >= items) return;
    const int lane = threadIdx.x & 31;
    const int users = t.users(), links = t.links();
    const int u = (int)(item % users);
    const int64_t gf = item / users;  // g*Fc + f
    const int i = u / t.K, j = u % t.K;
    const int m = t.m, n = t.n, mn = m * n;
    const C* Hgf = H + gf * links * mn;
    const int total = S * m * m;
    const int64_t orow = ((gf / Fc) * Ftot + f0 + gf % Fc) * users + u;  // row in the all-subcarrier PG
    for (int e = lane; e < total; e += 32) {
        const int s = e / (m * m);
        const int ab = e % (m * m);
        const int a = ab % m, b = ab / m;
        int k, l;
        scope_slot(t, scope, i, j, s, k, l);
        const C* h1 = Hgf + (int64_t)((k * t.J + i) * t.K + j) * mn;  // receive link (k,i,j)
        const C* h2 = Hgf + (int64_t)((k * t.J + k) * t.K + l) * mn;  // partner's serving link (k,k,l)
        double2 acc0 = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
        int c = 0;
#pragma unroll 4
        for (; c + 1 < n; c += 2) {
            cfmac(acc0, to_d2(h1[a + m * c]), to_d2(h2[b + m * c]));
            cfmac(acc1, to_d2(h1[a + m * (c + 1)]), to_d2(h2[b + m * (c + 1)]));
        }
        if (c < n) cfmac(acc0, to_d2(h1[a + m * c]), to_d2(h2[b + m * c]));
        PG[(orow * S + s) * m * m + a + m * b] = make_double2(acc0.x + acc1.x, acc0.y + acc1.y);
    }
}

// K2 (paper scope): the item's 2J-1 links (J receive links (k,i,j), J-1 partner links (k,k,0))
// are staged into shared memory with coalesced loads, then each lane computes one Gram entry.
template <class T, int M>
__global__ void __launch_bounds__(128) k_pair_gram_staged(Topo t, int Fc, int64_t f0, int64_t Ftot, int64_t items,
                                                          const cplx_t<T>* __restrict__ H, double2* __restrict__ PG) {
    using C = cplx_t<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    const int64_t item = (int64_t)blockIdx.x * (blockDim.x / 32) + warp;
    const int J = t.J, users = t.users(), links = t.links();
    const int mn = M * t.n, nl = 2 * J - 1;
    double2* sh = reinterpret_cast<double2*>(smem_raw) + (size_t)warp * nl * mn;  // binary64 once, at staging
    if (item >= items) return;
    const int u = (int)(item % users);
    const int64_t gf = item / users;
    const int i = u / t.K, j = u % t.K;
    const C* Hgf = H + gf * links * mn;
    for (int li = 0; li < nl; ++li) {
        int l;
        if (li < J) l = (li * J + i) * t.K + j;  // receive link (k = li, i, j)
        else {
            int k = li - J;
            if (k >= i) ++k;
            l = (k * J + k) * t.K;  // partner (k, k, 0)
        }
        const C* src = Hgf + (int64_t)l * mn;
        double2* dst = sh + li * mn;
        for (int e = lane; e < mn; e += 32) dst[e] = to_d2(src[e]);
    }
    __syncwarp();
    const int64_t orow = ((gf / Fc) * Ftot + f0 + gf % Fc) * users + u;
    constexpr int MM = M * M;
    for (int e = lane; e < J * MM; e += 32) {
        const int s = e / MM, ab = e % MM, a = ab % M, b = ab / M;
        // slot 0: serving (i,i,j) with itself; slot s>0: cell k (k-th cell != i) receive link vs partner
        int kcell = s == 0 ? i : (s - 1 < i ? s - 1 : s);
        const double2* h1 = sh + kcell * mn;
        const double2* h2 = s == 0 ? h1 : sh + (J + s - 1) * mn;
        double2 acc0 = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
        int c = 0;
        for (; c + 1 < t.n; c += 2) {
            cfmac(acc0, h1[a + M * c], h2[b + M * c]);
            cfmac(acc1, h1[a + M * (c + 1)], h2[b + M * (c + 1)]);
        }
        if (c < t.n) cfmac(acc0, h1[a + M * c], h2[b + M * c]);
        PG[(orow * J + s) * MM + ab] = make_double2(acc0.x + acc1.x, acc0.y + acc1.y);
    }
}

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(sdst)), "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// K2 (paper scope, c64), persistent and double-buffered: each CTA walks (group, subcarrier) slices
// with stride gridDim.x; slice it+1's H~(f) block (contiguous links*m*n complex64) is fetched with
// cp.async into a raw buffer while slice it is converted once to binary64 and reduced into the J
// pair Grams of every user (one thread per Gram entry).
template <int M>
__global__ void __launch_bounds__(256) k_pair_gram_pipe(Topo t, int Fc, int64_t f0, int64_t Ftot, int64_t nslices,
                                                        const float2* __restrict__ H, double2* __restrict__ PG) {
    constexpr int MM = M * M;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int J = t.J, K = t.K, links = t.links(), users = t.users();
    const int n = t.n, mn = M * n, tot = links * mn;  // complex elements per slice (tot % 2 == 0 checked)
    float2* raw[2] = {reinterpret_cast<float2*>(smem_raw), reinterpret_cast<float2*>(smem_raw) + tot};
    double2* sh = reinterpret_cast<double2*>(smem_raw + 2 * (size_t)tot * sizeof(float2));
    const int nchunk = tot / 2;  // 16-byte chunks per slice
    auto fetch = [&](int64_t sl, float2* dst) {
        if (sl < nslices) {
            const float2* src = H + sl * (int64_t)tot;  // slice = g * Fc + f (H~ layout [g][Fc][links][mn])
            for (int c = threadIdx.x; c < nchunk; c += blockDim.x) cp_async16(dst + 2 * c, src + 2 * c);
        }
        cp_async_commit();
    };
    int64_t sl = blockIdx.x;
    fetch(sl, raw[0]);
    for (int it = 0; sl < nslices; ++it, sl += gridDim.x) {
        fetch(sl + gridDim.x, raw[(it + 1) & 1]);
        cp_async_wait1();
        __syncthreads();
        const float2* r = raw[it & 1];
        for (int e = threadIdx.x; e < tot; e += blockDim.x) sh[e] = make_double2(r[e].x, r[e].y);
        __syncthreads();
        const int64_t g = sl / Fc, f = sl % Fc;
        const int64_t orow0 = (g * Ftot + f0 + f) * users;
        for (int e = threadIdx.x; e < users * J * MM; e += blockDim.x) {
            const int u = e / (J * MM), s = (e / MM) % J, ab = e % MM, a = ab % M, b = ab / M;
            const int i = u / K, j = u % K;
            int lx, ly;
            if (s == 0) {
                lx = ly = (i * J + i) * K + j;
            } else {
                const int k = s - 1 < i ? s - 1 : s;
                lx = (k * J + i) * K + j;
                ly = (k * J + k) * K;
            }
            const double2* h1 = sh + (size_t)lx * mn + a;
            const double2* h2 = sh + (size_t)ly * mn + b;
            double2 acc0 = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
            int c = 0;
            for (; c + 1 < n; c += 2) {
                cfmac(acc0, h1[M * c], h2[M * c]);
                cfmac(acc1, h1[M * (c + 1)], h2[M * (c + 1)]);
            }
            if (c < n) cfmac(acc0, h1[M * c], h2[M * c]);
            PG[((orow0 + u) * J + s) * MM + ab] = make_double2(acc0.x + acc1.x, acc0.y + acc1.y);
        }
        __syncthreads();  // sh and raw[it&1] reused by the next iterations
    }
}

// K2 (paper scope, whole subcarrier): one CTA per (group, subcarrier) stages every link of that
// H~(f) (one contiguous links*m*n block, 16-byte vector loads, converted to binary64 once) and
// computes all users' J pair Grams, one thread per Gram entry. No partner link is read twice.
template <class T, int M>
__global__ void __launch_bounds__(256) k_pair_gram_gf(Topo t, int Fc, int64_t f0, int64_t Ftot, int LS,
                                                      const cplx_t<T>* __restrict__ H, double2* __restrict__ PG) {
    // LS: padded per-link stride (LS % 8 == 4) so the two Gram tasks of a warp, which read different
    // links at the same offsets, hit disjoint shared-memory banks
    using C = cplx_t<T>;
    constexpr int MM = M * M;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* sh = reinterpret_cast<double2*>(smem_raw);  // [links][LS]
    const int J = t.J, K = t.K, links = t.links(), users = t.users();
    const int n = t.n, mn = M * n;
    const int f = blockIdx.x;
    const int64_t g = blockIdx.y;
    const C* Hf = H + ((g * Fc + f) * links) * (int64_t)mn;
    const int tot = links * mn;
    if (sizeof(C) == 8 && (mn % 2) == 0) {
        // all of a thread's 16-byte loads are issued before the first conversion/store: the staging
        // phase was HBM-latency bound with one load in flight per thread (ncu: long-scoreboard stalls
        // on the store line)
        constexpr int U = 4;
        const float4* h4 = reinterpret_cast<const float4*>(Hf);
        const int n4 = tot / 2;
        for (int e0 = threadIdx.x; e0 < n4; e0 += U * blockDim.x) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = e0 + u * blockDim.x;
                if (e < n4) v[u] = __ldg(h4 + e);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = e0 + u * blockDim.x;
                if (e < n4) {
                    const int l = (2 * e) / mn, r = (2 * e) % mn;
                    sh[l * LS + r] = make_double2(v[u].x, v[u].y);
                    sh[l * LS + r + 1] = make_double2(v[u].z, v[u].w);
                }
            }
        }
    } else {
        for (int e = threadIdx.x; e < tot; e += blockDim.x) sh[(e / mn) * LS + e % mn] = to_d2(Hf[e]);
    }
    __syncthreads();
    const int64_t orow0 = (g * Ftot + f0 + f) * users;
    for (int e = threadIdx.x; e < users * J * MM; e += blockDim.x) {
        const int u = e / (J * MM), s = (e / MM) % J, ab = e % MM, a = ab % M, b = ab / M;
        const int i = u / K, j = u % K;
        int lx, ly;
        if (s == 0) {
            lx = ly = (i * J + i) * K + j;  // serving (i,i,j)
        } else {
            const int k = s - 1 < i ? s - 1 : s;  // s-th cell != i (scope_pairs order)
            lx = (k * J + i) * K + j;
            ly = (k * J + k) * K;
        }
        const double2* h1 = sh + (size_t)lx * LS + a;
        const double2* h2 = sh + (size_t)ly * LS + b;
        double2 acc0 = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
        int c = 0;
        for (; c + 1 < n; c += 2) {
            cfmac(acc0, h1[M * c], h2[M * c]);
            cfmac(acc1, h1[M * (c + 1)], h2[M * (c + 1)]);
        }
        if (c < n) cfmac(acc0, h1[M * c], h2[M * c]);
        PG[((orow0 + u) * J + s) * MM + ab] = make_double2(acc0.x + acc1.x, acc0.y + acc1.y);
    }
}

// ---------------------------------------------------------------------------
// K1+K2 fused (opt-in GWT_SINR_PATH=rg; measured slower than K1 -> K2 on C2): one CTA (512
// threads) per (group, FT-subcarrier tile): phasors -> E -> every link's H~ for the tile (binary64
// in shared memory) -> the J pair Grams of every user, 4 threads per (user, slot, subcarrier).
template <int M>
__host__ __device__ inline size_t rg_smem(const Topo& t, int FT, int csize) {
    const size_t hd = (size_t)t.links() * M * t.n * FT * 16;
    const size_t ph = (size_t)t.links() * t.P * FT * csize;
    return (hd > ph ? hd : ph) + (size_t)t.links() * t.p * FT * csize;
}

template <class T, int M, int FT>
__global__ void __launch_bounds__(512, 1) k_rebuild_pg(Topo t, int Fc, int64_t f0, int64_t Ftot, int64_t pf0, int64_t pfs,
                                                     const cplx_t<T>* __restrict__ Cd, const cplx_t<T>* __restrict__ G,
                                                     const double* __restrict__ tau, const double* __restrict__ freqs,
                                                     const cplx_t<T>* __restrict__ coeffs, double2* __restrict__ PG) {
    using C = cplx_t<T>;
    constexpr int NT = 512, MM = M * M;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int J = t.J, K = t.K, links = t.links(), users = t.users();
    const int n = t.n, mn = M * n, P = t.P, p = t.p;
    double2* Hd = reinterpret_cast<double2*>(smem_raw);  // [links][mn][FT]   (phases 3-4)
    C* Ph = reinterpret_cast<C*>(smem_raw);              // [links][P][FT]    (phases 1-2, aliases Hd)
    const size_t hd_bytes = (size_t)links * mn * FT * 16, ph_bytes = (size_t)links * P * FT * sizeof(C);
    C* E = reinterpret_cast<C*>(smem_raw + (hd_bytes > ph_bytes ? hd_bytes : ph_bytes));  // [links][p][FT]
    const int64_t g = blockIdx.y;
    const int ft0 = blockIdx.x * FT;
    const int nf = min(FT, Fc - ft0);
    const int tid = threadIdx.x;
    for (int idx = tid; idx < links * P * FT; idx += NT) {
        const int l = idx / (P * FT), r = (idx / FT) % P, f = idx % FT;
        C v = czero<C>();
        if (f < nf) {
            const int64_t fa = f0 + ft0 + f;
            v = coeffs ? cconj(coeffs[((g * Ftot + fa) * links + l) * P + r])
                       : conj_coeff<T>(freqs[fa], tau[(g * links + l) * P + r]);
        }
        Ph[idx] = v;
    }
    __syncthreads();
    for (int idx = tid; idx < links * p * FT; idx += NT) {
        const int l = idx / (p * FT), q = (idx / FT) % p, f = idx % FT;
        const C* Cl = Cd + ((g * links + l) * P) * (int64_t)p + (int64_t)P * q;
        const C* ph = Ph + (size_t)l * P * FT + f;
        C acc = czero<C>();
        for (int r = 0; r < P; ++r) cfma(acc, Cl[r], ph[r * FT]);
        E[idx] = acc;
    }
    __syncthreads();
    for (int rg = tid; rg < links * mn; rg += NT) {
        const int l = rg / mn, row = rg % mn;
        const C* Gl = G + (g * links + l) * (int64_t)mn * p + row;
        const C* e = E + (size_t)l * p * FT;
        C acc[FT];
#pragma unroll
        for (int f = 0; f < FT; ++f) acc[f] = czero<C>();
        for (int q = 0; q < p; ++q) {
            const C gv = Gl[(int64_t)mn * q];
#pragma unroll
            for (int f = 0; f < FT; ++f) cfma(acc[f], gv, e[q * FT + f]);
        }
        double2* h = Hd + (size_t)rg * FT;
#pragma unroll
        for (int f = 0; f < FT; ++f) h[f] = to_d2(acc[f]);
    }
    __syncthreads();
    const int ntask = users * J * FT * 4;
    for (int w = tid; w < ntask; w += NT) {
        const int h = w & 3, f = (w >> 2) % FT, task = (w >> 2) / FT;
        const int u = task / J, s = task % J;
        const int i = u / K, j = u % K;
        int lx, ly;
        if (s == 0) {
            lx = ly = (i * J + i) * K + j;
        } else {
            const int k = s - 1 < i ? s - 1 : s;
            lx = (k * J + i) * K + j;
            ly = (k * J + k) * K;
        }
        const double2* hx = Hd + (size_t)lx * mn * FT + f;
        const double2* hy = Hd + (size_t)ly * mn * FT + f;
        double2 acc[M][M];
#pragma unroll
        for (int a = 0; a < M; ++a)
#pragma unroll
            for (int b = 0; b < M; ++b) acc[a][b] = make_double2(0.0, 0.0);
        for (int c = h; c < n; c += 4) {
            double2 xa[M], yb[M];
#pragma unroll
            for (int a = 0; a < M; ++a) {
                xa[a] = hx[(size_t)(a + M * c) * FT];
                yb[a] = hy[(size_t)(a + M * c) * FT];
            }
#pragma unroll
            for (int a = 0; a < M; ++a)
#pragma unroll
                for (int b = 0; b < M; ++b) cfmac(acc[a][b], xa[a], yb[b]);
        }
#pragma unroll
        for (int a = 0; a < M; ++a)
#pragma unroll
            for (int b = 0; b < M; ++b)
#pragma unroll
                for (int o = 1; o < 4; o <<= 1) {
                    acc[a][b].x += __shfl_xor_sync(0xffffffffu, acc[a][b].x, o);
                    acc[a][b].y += __shfl_xor_sync(0xffffffffu, acc[a][b].y, o);
                }
        if (f < nf) {
            double2* o = PG + (((g * pfs + pf0 + ft0 + f) * users + u) * J + s) * MM;
#pragma unroll
            for (int e = 0; e < MM; ++e)
                if ((e & 3) == h) o[e] = acc[e % M][e / M];
        }
    }
}

template <class T>
cudaError_t launch_rebuild_pg(const Topo& t, int ngroups, int Fc, int64_t f0, int64_t Ftot, int64_t pf0, int64_t pfs,
                              const void* Cd, const void* G, const double* tau, const double* freqs, const void* coeffs,
                              double2* PG, cudaStream_t st) {
    constexpr int FT = 8;
    if (t.m > 4) return cudaErrorNotSupported;
    const size_t cs = sizeof(cplx_t<T>);
    dim3 grid((Fc + FT - 1) / FT, ngroups);
    cudaError_t e = cudaErrorNotSupported;
    switch (t.m) {
#define GWT_RPG(MM)                                                                                                   \
    case MM: {                                                                                                        \
        const size_t sm = rg_smem<MM>(t, FT, (int)cs);                                                                \
        if (sm > 227 * 1024) return cudaErrorNotSupported;                                                            \
        e = cudaFuncSetAttribute(k_rebuild_pg<T, MM, FT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);     \
        if (e != cudaSuccess) return e;                                                                               \
        k_rebuild_pg<T, MM, FT><<<grid, 512, sm, st>>>(t, Fc, f0, Ftot, pf0, pfs, (const cplx_t<T>*)Cd,              \
                                                       (const cplx_t<T>*)G, tau, freqs, (const cplx_t<T>*)coeffs, PG); \
        return cudaGetLastError();                                                                                    \
    }
        GWT_RPG(1) GWT_RPG(2) GWT_RPG(3) GWT_RPG(4)
#undef GWT_RPG
    }
    return e;
}
bool rebuild_pg_fits(const Topo& t, size_t csize) {
    if (t.m > 4) return false;
    switch (t.m) {
        case 1: return rg_smem<1>(t, 8, (int)csize) <= 227 * 1024;
        case 2: return rg_smem<2>(t, 8, (int)csize) <= 227 * 1024;
        case 3: return rg_smem<3>(t, 8, (int)csize) <= 227 * 1024;
        default: return rg_smem<4>(t, 8, (int)csize) <= 227 * 1024;
    }
}
template cudaError_t launch_rebuild_pg<float>(const Topo&, int, int, int64_t, int64_t, int64_t, int64_t, const void*,
                                              const void*, const double*, const double*, const void*, double2*,
                                              cudaStream_t);
template cudaError_t launch_rebuild_pg<double>(const Topo&, int, int, int64_t, int64_t, int64_t, int64_t, const void*,
                                               const void*, const double*, const double*, const void*, double2*,
                                               cudaStream_t);

// ---------------------------------------------------------------------------
// K3a: precoder per (group, subcarrier, user): eig of the serving Gram ->
// top-L eigenpairs (descending). EG layout per item: lambda[L] (padded to even) then U[M][L]
// column-major (M x L), fp64.
template <int M>
__device__ __forceinline__ void precoder_item(const Topo& t, int scope, int S, int64_t item, const double2* PG,
                                              double* EG, int64_t eg_item) {
    const int L = t.L;
    const int u = (int)(item % t.users());
    const int i = u / t.K, j = u % t.K;
    const int ss = serving_slot(t, scope, i, j);
    const double2* src = PG + (item * S + ss) * M * M;
    double2 A[M][M], V[M][M];
#pragma unroll
    for (int b = 0; b < M; ++b)
#pragma unroll
        for (int a = 0; a < M; ++a) A[a][b] = src[a + M * b];
    // Hermitian part (exact Gram up to rounding)
#pragma unroll
    for (int a = 0; a < M; ++a) {
        A[a][a].y = 0.0;
#pragma unroll
        for (int b = a + 1; b < M; ++b) {
            const double2 v = make_double2(0.5 * (A[a][b].x + A[b][a].x), 0.5 * (A[a][b].y - A[b][a].y));
            A[a][b] = v;
            A[b][a] = make_double2(v.x, -v.y);
        }
    }
    jacobi_herm<M>(A, V);
    double lam[M];
    int rank[M];
#pragma unroll
    for (int r = 0; r < M; ++r) lam[r] = A[r][r].x;
#pragma unroll
    for (int r = 0; r < M; ++r) {
        int rk = 0;
#pragma unroll
        for (int s = 0; s < M; ++s) rk += (lam[s] > lam[r] || (lam[s] == lam[r] && s < r)) ? 1 : 0;
        rank[r] = rk;
    }
    const int Lp = (L + 1) & ~1;  // keep the U block 16-byte aligned
    double* dst = EG + eg_item * (int64_t)(Lp + 2 * M * L);
    double2* du = reinterpret_cast<double2*>(dst + Lp);
#pragma unroll
    for (int r = 0; r < M; ++r) {
        if (rank[r] < L) {
            dst[rank[r]] = fmax(lam[r], 0.0);
#pragma unroll
            for (int a = 0; a < M; ++a) du[a + M * rank[r]] = V[a][r];
        }
    }
}

template <int M>
__global__ void __launch_bounds__(128) k_precoder_eig(Topo t, int scope, int S, int64_t items,
                                                      const double2* __restrict__ PG, double* __restrict__ EG) {
    const int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= items) return;
    precoder_item<M>(t, scope, S, item, PG, EG, item);
}

// ---------------------------------------------------------------------------
// K3b: covariance, Cholesky (with the reference's PD and condition checks),
// filter and per-stream SINR; one thread per (group, subcarrier, user).
template <int M>
__device__ __forceinline__ void mmse_item(const Topo& t, int scope, int S, int64_t item, double sigma, int fc,
                                          int64_t Ftot, int64_t f0, const double2* PG, const double* EG,
                                          int64_t eg_item, double* sinr, double* signal, int* status) {
    const int L = t.L;
    const int users = t.users();
    const int u = (int)(item % users);
    const int64_t gf = item / users;
    const int i = u / t.K, j = u % t.K;
    const int Lp = (L + 1) & ~1;
    const int64_t eg_stride = Lp + 2 * M * L;
    const double* own = EG + eg_item * eg_stride;
    const double2* ownU = reinterpret_cast<const double2*>(own + Lp);
    int st = 0;
    double2 Q[M][M];
    const double s2 = sigma * sigma;
#pragma unroll
    for (int a = 0; a < M; ++a)
#pragma unroll
        for (int b = 0; b < M; ++b) Q[a][b] = make_double2(a == b ? s2 : 0.0, 0.0);
    // serving term U_L Lambda_L U_L^H  (= (H~ V)(H~ V)^H)
    for (int r = 0; r < L; ++r) {
        const double lr = own[r];
        double2 ur[M];
#pragma unroll
        for (int a = 0; a < M; ++a) ur[a] = ownU[a + M * r];
#pragma unroll
        for (int a = 0; a < M; ++a)
#pragma unroll
            for (int b = 0; b < M; ++b) {
                double2 v = make_double2(0, 0);
                cfmac(v, ur[a], ur[b]);
                Q[a][b].x += lr * v.x;
                Q[a][b].y += lr * v.y;
            }
    }
    // interferer terms (X P X^H) for every non-serving scope slot
    const int ss = serving_slot(t, scope, i, j);
    for (int s = 0; s < S; ++s) {
        if (s == ss) continue;
        int k, l;
        scope_slot(t, scope, i, j, s, k, l);
        const int64_t pidx = (eg_item / users) * users + (k * t.K + l);
        const double* pe = EG + pidx * eg_stride;
        const double2* pU = reinterpret_cast<const double2*>(pe + Lp);
        const double2* X = PG + (item * S + s) * M * M;
        double2 Xr[M][M];
#pragma unroll
        for (int b = 0; b < M; ++b)
#pragma unroll
            for (int a = 0; a < M; ++a) Xr[a][b] = X[a + M * b];
        for (int r = 0; r < L; ++r) {
            const double lr = pe[r];
            if (!(lr > 0.0)) {
                st = st ? st : 5;
                continue;
            }
            const double sc = 1.0 / sqrt(lr);
            double2 z[M];  // z = X u'_r / sqrt(lambda'_r)  (= H~_{kij} v_{kl,r})
#pragma unroll
            for (int a = 0; a < M; ++a) {
                double2 acc = make_double2(0, 0);
#pragma unroll
                for (int b = 0; b < M; ++b) cfma(acc, Xr[a][b], pU[b + M * r]);
                z[a] = make_double2(acc.x * sc, acc.y * sc);
            }
#pragma unroll
            for (int a = 0; a < M; ++a)
#pragma unroll
                for (int b = 0; b < M; ++b) cfmac(Q[a][b], z[a], z[b]);
        }
    }
    // non-finite check (check_finite(q, "woodbury_inverse_apply"))
    bool finite = true;
#pragma unroll
    for (int a = 0; a < M; ++a)
#pragma unroll
        for (int b = 0; b < M; ++b) finite = finite && isfinite(Q[a][b].x) && isfinite(Q[a][b].y);
    // Cholesky, lower, in place (Eigen::LLT semantics)
    bool pd = finite;
    double dmax = 0.0, dmin = 1e308;
#pragma unroll
    for (int c = 0; c < M; ++c) {
        double d = Q[c][c].x;
#pragma unroll
        for (int k2 = 0; k2 < c; ++k2) d -= Q[c][k2].x * Q[c][k2].x + Q[c][k2].y * Q[c][k2].y;
        pd = pd && (d > 0.0);
        const double lcc = sqrt(fmax(d, 1e-300));
        dmax = fmax(dmax, lcc);
        dmin = fmin(dmin, lcc);
        Q[c][c] = make_double2(lcc, 0.0);
        const double inv = 1.0 / lcc;
#pragma unroll
        for (int r = c + 1; r < M; ++r) {
            double2 s = Q[r][c];
#pragma unroll
            for (int k2 = 0; k2 < c; ++k2) {
                const double2 pr = make_double2(Q[r][k2].x * Q[c][k2].x + Q[r][k2].y * Q[c][k2].y,
                                                Q[r][k2].y * Q[c][k2].x - Q[r][k2].x * Q[c][k2].y);
                s.x -= pr.x;
                s.y -= pr.y;
            }
            Q[r][c] = make_double2(s.x * inv, s.y * inv);
        }
    }
    if (!finite) st = 4;
    else if (!pd) st = 1;
    else if ((dmax / dmin) * (dmax / dmin) > 1e14) st = 2;
    // output row: items are (g, f in chunk, u); outputs are [g][Ftot][users]
    const int64_t g = gf / fc, fl = gf % fc;
    const int64_t orow = (g * Ftot + f0 + fl) * users + u;
    double* so = sinr + orow * L;
    double* sg = signal + orow * L;
    for (int r = 0; r < L; ++r) {
        double gamma = 0.0;
        const double lr = own[r];
        if (st != 1 && st != 2 && st != 4) {
            double2 y[M];
#pragma unroll
            for (int a = 0; a < M; ++a) {
                double2 acc = ownU[a + M * r];
#pragma unroll
                for (int k2 = 0; k2 < a; ++k2) {
                    double2 pr = make_double2(0, 0);
                    cfma(pr, Q[a][k2], y[k2]);
                    acc.x -= pr.x;
                    acc.y -= pr.y;
                }
                y[a] = make_double2(acc.x / Q[a][a].x, acc.y / Q[a][a].x);
            }
            double nn = 0.0;
#pragma unroll
            for (int a = 0; a < M; ++a) nn += y[a].x * y[a].x + y[a].y * y[a].y;
            gamma = lr * nn;  // g^H Q^{-1} g
        }
        const double sp = gamma * gamma;
        double den = gamma * (1.0 - gamma);  // w^H Q w - |w^H g|^2
        if (den <= -1e-12 && st == 0) st = 3;
        den = fmax(den, 2.2250738585072014e-308);
        so[r] = sp / den;
        sg[r] = sp;
    }
    status[orow] = st;
}

template <int M>
__global__ void __launch_bounds__(128) k_mmse(Topo t, int scope, int S, int64_t items, double sigma, int fc,
                                              int64_t Ftot, int64_t f0, const double2* __restrict__ PG,
                                              const double* __restrict__ EG,
                                              double* __restrict__ sinr, double* __restrict__ signal,
                                              int* __restrict__ status) {
    const int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= items) return;
    mmse_item<M>(t, scope, S, item, sigma, fc, Ftot, f0, PG, EG, item, sinr, signal, status);
}

// K3 fused: a CTA holds whole (group, subcarrier) slices (users x SL threads); the precoders go to
// shared memory and the MMSE phase reads its partners' from there (no EG round trip through HBM).
template <int M>
__global__ void __launch_bounds__(128, 3) k_small_fused(Topo t, int scope, int S, int64_t items, double sigma, int fc,
                                                     int64_t Ftot, int64_t f0, const double2* __restrict__ PG,
                                                     double* __restrict__ sinr, double* __restrict__ signal,
                                                     int* __restrict__ status) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* eg = reinterpret_cast<double*>(smem_raw);
    const int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool on = item < items;
    if (on) precoder_item<M>(t, scope, S, item, PG, eg, threadIdx.x);
    __syncthreads();
    if (on) mmse_item<M>(t, scope, S, item, sigma, fc, Ftot, f0, PG, eg, threadIdx.x, sinr, signal, status);
}

// ---------------------------------------------------------------------------
// K3 for m > 4 (C3/C4: m = 8): one CTA per SPC (group, subcarrier) slices, 8 lanes per user
// (lane = matrix column), all matrices in fp64.
//  a) precoder: parallel cyclic Jacobi on the serving Gram (round-robin pairing, 7 rounds of 4
//     disjoint rotations per sweep; the rotation of jacobi_herm / the reference test oracle),
//     columns exchanged between partner lanes by shuffles; eigenpairs ranked and kept in smem.
//  b) MMSE: lane j builds column j of Q (partners' precoders read from smem), right-looking
//     Cholesky with the reference's PD / condition / finite checks, one lane per stream solves
//     L y = u_r for gamma_r.
template <class V>
__device__ __forceinline__ V sel8(const V (&a)[8], int i) {
    V r = a[0];
#pragma unroll
    for (int k = 1; k < 8; ++k)
        if (k == i) r = a[k];
    return r;
}
__device__ __forceinline__ double2 shfl_d2(double2 v, int src) {
    return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}
__host__ __device__ constexpr int rr_partner(int i, int r) {  // round-robin pairing of 8 indices, round r < 7
    return i == 7 ? r : (i == r ? 7 : ((2 * r - i) % 7 + 7) % 7);
}

template <int M>
__global__ void __launch_bounds__(256) k_small_grp(Topo t, int scope, int S, int64_t nslices, int spc, double sigma,
                                                   int fc, int64_t Ftot, int64_t f0, const double2* __restrict__ PG,
                                                   double* __restrict__ sinr, double* __restrict__ signal,
                                                   int* __restrict__ status) {
    constexpr int MM = M * M;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int users = t.users(), L = t.L;
    const int tid = threadIdx.x, lane = tid & 31, j = tid & 7, base = lane & ~7;
    const int sl_local = tid / (users * 8), u = (tid / 8) % users;
    const int64_t sl = (int64_t)blockIdx.x * spc + sl_local;
    // per slice: U [users][8][8] double2, L-factor scratch [users][8][8] double2, lambda [users][8]
    const size_t per_slice = (size_t)users * (64 * 16 * 2 + 8 * 8);
    double2* sU = reinterpret_cast<double2*>(smem_raw + sl_local * per_slice);
    double2* sL = sU + (size_t)users * 64;
    double* slam = reinterpret_cast<double*>(sL + (size_t)users * 64);
    const bool valid = sl_local < spc && sl < nslices;
    const int64_t item = (sl < nslices ? sl : 0) * users + u;
    const int i_cell = u / t.K, j_user = u % t.K;
    // ---- a) precoder eig of the serving Gram (symmetrised), lane j holds column j
    double2 acol[8], vcol[8];
    {
        const int ss = serving_slot(t, scope, i_cell, j_user);
        const double2* src = PG + (item * S + ss) * MM;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            double2 a = make_double2(0.0, 0.0);
            if (valid && i < M && j < M) {
                const double2 x = src[i + M * j], y = src[j + M * i];
                a = make_double2(0.5 * (x.x + y.x), 0.5 * (x.y - y.y));
                if (i == j) a.y = 0.0;
            }
            acol[i] = a;
            vcol[i] = make_double2(i == j ? 1.0 : 0.0, 0.0);
        }
    }
    for (int sweep = 0; sweep < 32; ++sweep) {
        double off = 0.0, dia = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (i < j) off += acol[i].x * acol[i].x + acol[i].y * acol[i].y;
            if (i == j) dia += acol[i].x * acol[i].x;
        }
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            off += __shfl_xor_sync(0xffffffffu, off, o);
            dia += __shfl_xor_sync(0xffffffffu, dia, o);
        }
        const bool conv = off <= kJacobiTol * dia || off == 0.0;
        if (__all_sync(0xffffffffu, conv)) break;
#pragma unroll
        for (int r = 0; r < 7; ++r) {
            const int q = rr_partner(j, r);
            const bool lead = j < q;
            double2 pc[8], pv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                pc[i] = shfl_d2(acol[i], base + q);
                pv[i] = shfl_d2(vcol[i], base + q);
            }
            // rotation parameters from the leader's column and the other lane's diagonal
            const double2 app = lead ? sel8(acol, j) : sel8(pc, q);
            const double2 aqq = lead ? sel8(pc, q) : sel8(acol, j);
            const double2 aqp = lead ? sel8(acol, q) : sel8(pc, j);  // A[q][p] of the leader's column
            const double2 apq = make_double2(aqp.x, -aqp.y);
            double c = 1.0, sn = 0.0, phr = 1.0, phi = 0.0;
            const double b2 = apq.x * apq.x + apq.y * apq.y;
            if (b2 > 1e-300) {
                const double rb = rsqrt(b2);
                phr = apq.x * rb;
                phi = apq.y * rb;
                const float tau = (float)((aqq.x - app.x) * (0.5 * rb));
                const float tf = copysignf(1.0f, tau) / (fabsf(tau) + sqrtf(fmaf(tau, tau, 1.0f)));
                const double tt = (double)tf;
                c = rsqrt(fma(tt, tt, 1.0));
                sn = tt * c;
            }
            const double2 uqp = make_double2(-sn * phr, sn * phi), uqq = make_double2(c * phr, -c * phi);
            // A <- A U and V <- V U: columns p (leader) and q
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double2 na, nv;
                if (lead) {
                    na = make_double2(c * acol[i].x, c * acol[i].y);
                    cfma(na, pc[i], uqp);
                    nv = make_double2(c * vcol[i].x, c * vcol[i].y);
                    cfma(nv, pv[i], uqp);
                } else {
                    na = make_double2(sn * pc[i].x, sn * pc[i].y);
                    cfma(na, acol[i], uqq);
                    nv = make_double2(sn * pv[i].x, sn * pv[i].y);
                    cfma(nv, vcol[i], uqq);
                }
                acol[i] = na;
                vcol[i] = nv;
            }
            // A <- U^H A: rows p, q of my column for every pair of this round (parameters from leaders)
#pragma unroll
            for (int pp = 0; pp < 8; ++pp) {
                const int qq = rr_partner(pp, r);
                if (pp < qq) {
                    const double cl = __shfl_sync(0xffffffffu, c, base + pp);
                    const double sl2 = __shfl_sync(0xffffffffu, sn, base + pp);
                    const double pr = __shfl_sync(0xffffffffu, phr, base + pp);
                    const double pi = __shfl_sync(0xffffffffu, phi, base + pp);
                    const double2 up = make_double2(-sl2 * pr, sl2 * pi), uq = make_double2(cl * pr, -cl * pi);
                    const double2 apc = acol[pp], aqc = acol[qq];
                    double2 np = make_double2(cl * apc.x, cl * apc.y);
                    cfmaconj(np, up, aqc);
                    double2 nq = make_double2(sl2 * apc.x, sl2 * apc.y);
                    cfmaconj(nq, uq, aqc);
                    acol[pp] = np;
                    acol[qq] = nq;
                }
            }
        }
    }
    // rank eigenvalues (descending, lower index first on ties) and keep the top L
    {
        const double lam = sel8(acol, j).x;
        int rank = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const double lk = __shfl_sync(0xffffffffu, lam, base + k);
            if (k < M && j < M) rank += (lk > lam || (lk == lam && k < j)) ? 1 : 0;
        }
        if (valid && j < M && rank < L) {
            slam[u * 8 + rank] = fmax(lam, 0.0);
#pragma unroll
            for (int i = 0; i < 8; ++i) sU[(u * 8 + rank) * 8 + i] = vcol[i];
        }
    }
    __syncthreads();
    // ---- b) covariance column j, Cholesky, per-stream gamma
    int st = 0;
    const double s2 = sigma * sigma;
    double2 qcol[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) qcol[i] = make_double2(i == j ? s2 : 0.0, 0.0);
    if (valid && j < M) {
        for (int r = 0; r < L; ++r) {
            const double lr = slam[u * 8 + r];
            const double2* ur = sU + (u * 8 + r) * 8;
            const double2 uj = ur[j];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double2 v = make_double2(0.0, 0.0);
                cfmac(v, ur[i], uj);
                qcol[i].x += lr * v.x;
                qcol[i].y += lr * v.y;
            }
        }
    }
    const int ss = serving_slot(t, scope, i_cell, j_user);
    for (int s = 0; s < S; ++s) {
        if (s == ss) continue;
        int k, l;
        scope_slot(t, scope, i_cell, j_user, s, k, l);
        const int pu = k * t.K + l;
        double2 xrow[8];
        const double2* X = PG + (item * S + s) * MM;
#pragma unroll
        for (int b = 0; b < 8; ++b) xrow[b] = (valid && j < M && b < M) ? X[j + M * b] : make_double2(0.0, 0.0);
        for (int r = 0; r < L; ++r) {  // warp-uniform trip count: every lane reaches the shuffles
            const double lr = valid ? slam[pu * 8 + r] : 1.0;
            const bool ok = lr > 0.0;
            if (!ok) st = st ? st : 5;
            const double sc = ok ? 1.0 / sqrt(lr) : 0.0;
            const double2* ur = sU + (pu * 8 + r) * 8;
            double2 zj = make_double2(0.0, 0.0);
            if (valid && ok) {
#pragma unroll
                for (int b = 0; b < 8; ++b) cfma(zj, xrow[b], ur[b]);
            }
            zj = make_double2(zj.x * sc, zj.y * sc);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const double2 zi = shfl_d2(zj, base + i);
                cfmac(qcol[i], zi, zj);
            }
        }
    }
    // non-finite check over the item's Q (check_finite(q, "woodbury_inverse_apply"))
    bool finite;
    {
        bool fin = true;
#pragma unroll
        for (int i = 0; i < 8; ++i) fin = fin && isfinite(qcol[i].x) && isfinite(qcol[i].y);
        const unsigned bad = __ballot_sync(0xffffffffu, !fin);
        finite = ((bad >> base) & 0xffu) == 0u;
    }
    // right-looking Cholesky (Eigen::LLT semantics: d_c = Q_cc - sum_k |L_ck|^2 > 0), lane = column
    bool pd = finite;
    double dmax = 0.0, dmin = 1e308;
#pragma unroll
    for (int kc = 0; kc < M; ++kc) {
        double dh = 0.0;
        if (j == kc) {
            dh = qcol[kc].x;
            const double lkk = sqrt(fmax(dh, 1e-300));
            qcol[kc] = make_double2(lkk, 0.0);
            const double inv = 1.0 / lkk;
#pragma unroll
            for (int i = kc + 1; i < 8; ++i) qcol[i] = make_double2(qcol[i].x * inv, qcol[i].y * inv);
        }
        const double d = __shfl_sync(0xffffffffu, dh, base + kc);
        double2 lk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) lk[i] = shfl_d2(qcol[i], base + kc);
        pd = pd && (d > 0.0);
        dmax = fmax(dmax, lk[kc].x);
        dmin = fmin(dmin, lk[kc].x);
        if (j > kc && j < M) {
            const double2 ljv = sel8(lk, j);  // L[j][kc]
#pragma unroll
            for (int i = kc + 1; i < 8; ++i) {
                if (i >= j) {  // Q[i][j] -= L[i][kc] conj(L[j][kc])
                    qcol[i].x -= lk[i].x * ljv.x + lk[i].y * ljv.y;
                    qcol[i].y -= lk[i].y * ljv.x - lk[i].x * ljv.y;
                }
            }
        }
    }
    if (valid && j < M)
#pragma unroll
        for (int i = 0; i < 8; ++i) sL[(u * 8 + j) * 8 + i] = qcol[i];  // column j of L
    __syncwarp();
    if (!finite) st = 4;
    else if (!pd) st = 1;
    else if ((dmax / dmin) * (dmax / dmin) > 1e14) st = 2;
    const int64_t gf = item / users;
    const int64_t g = gf / fc, fl = gf % fc;
    const int64_t orow = (g * Ftot + f0 + fl) * users + u;
    if (valid && j < L) {
        const int r = j;
        double gamma = 0.0;
        const double lr = slam[u * 8 + r];
        if (st != 1 && st != 2 && st != 4) {
            const double2* ur = sU + (u * 8 + r) * 8;
            double2 y[8];
#pragma unroll
            for (int a = 0; a < 8; ++a) {
                if (a < M) {
                    double2 acc = ur[a];
#pragma unroll
                    for (int k2 = 0; k2 < a; ++k2) {
                        double2 pr = make_double2(0, 0);
                        cfma(pr, sL[(u * 8 + k2) * 8 + a], y[k2]);
                        acc.x -= pr.x;
                        acc.y -= pr.y;
                    }
                    const double laa = sL[(u * 8 + a) * 8 + a].x;
                    y[a] = make_double2(acc.x / laa, acc.y / laa);
                } else {
                    y[a] = make_double2(0.0, 0.0);
                }
            }
            double nn = 0.0;
#pragma unroll
            for (int a = 0; a < 8; ++a) nn += y[a].x * y[a].x + y[a].y * y[a].y;
            gamma = lr * nn;
        }
        const double sp = gamma * gamma;
        double den = gamma * (1.0 - gamma);
        if (den <= -1e-12 && st == 0) st = 3;
        den = fmax(den, 2.2250738585072014e-308);
        sinr[orow * L + r] = sp / den;
        signal[orow * L + r] = sp;
    }
    // status: lanes agree on 5/4/1/2; a negative denominator (3) can come from any stream lane
    {
        const unsigned any3 = __ballot_sync(0xffffffffu, st == 3);
        if (valid && j == 0) status[orow] = (st == 0 && ((any3 >> base) & 0xffu)) ? 3 : st;
    }
}

// ---------------------------------------------------------------------------
// Fused compressed-SINR path (paper_experiment scope), two kernels:
//  k_rebuild_gram: one CTA per (group, user batch, subcarrier tile). H~ is
//    rebuilt tile by tile into shared memory and consumed there: per user the
//    serving Gram A_u and one cross Gram X_{u,k} per other cell (fp64), so H~
//    never touches HBM. Output: GU[g][f][user][J][m*m].
//  k_sinr_solve: one CTA per (group, subcarrier tile), one thread per
//    (user, subcarrier): eig of A_u (Jacobi), the partner projectors P_{k0}
//    exchanged through shared memory, covariance, Cholesky, SINR.
struct FusedShape {
    int B, FT, fsplit;
};

// Shared-memory tile layouts (bank-conflict free for the access patterns below):
//   Ph [nl][P][FT] conj(c_r(f)),  E [nl][p][FT],  H~ tile [m*n][FT+1] (subcarrier fastest, padded)
// A CTA is split into NG independent groups of WG threads (named barriers), each group
// rebuilding nl (<= 2) links at a time: phasors -> E -> H~ -> Grams, every phase fully parallel.

__device__ __forceinline__ void group_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <class T, int M, int FT, int FPT>
__device__ __forceinline__ void group_rebuild(const Topo& t, int lane, int WG, int bar_id, int nl, const int* lids,
                                              int ft0, int Fc, int64_t f0, int64_t Ftot, int64_t gidx,
                                              const cplx_t<T>* __restrict__ Cd, const cplx_t<T>* __restrict__ G,
                                              const double* __restrict__ tau, const double* __restrict__ freqs,
                                              const cplx_t<T>* __restrict__ coeffs, cplx_t<T>* Ph, cplx_t<T>* Es,
                                              cplx_t<T>* const* dst) {
    using C = cplx_t<T>;
    constexpr int LD = FT + 1;
    const int links = t.links();
    const int PF = t.P * FT, pF = t.p * FT;
    for (int idx = lane; idx < nl * PF; idx += WG) {
        const int li = idx / PF, rem = idx % PF, r = rem / FT, f = rem % FT;
        const int64_t gl = gidx * links + lids[li];
        C v = czero<C>();
        if (ft0 + f < Fc) {
            const int64_t fa = f0 + ft0 + f;
            v = coeffs ? cconj(coeffs[((gidx * Ftot + fa) * links + lids[li]) * t.P + r])
                       : conj_coeff<T>(freqs[fa], tau[gl * t.P + r]);
        }
        Ph[idx] = v;
    }
    group_bar(bar_id, WG);
    for (int idx = lane; idx < nl * pF; idx += WG) {
        const int li = idx / pF, rem = idx % pF, q = rem / FT, f = rem % FT;
        const C* Cl = Cd + (gidx * links + lids[li]) * t.P * t.p + (int64_t)t.P * q;
        const C* ph = Ph + li * PF + f;
        C acc = czero<C>();
        for (int r = 0; r < t.P; ++r) cfma(acc, Cl[r], ph[r * FT]);
        Es[idx] = acc;
    }
    group_bar(bar_id, WG);
    const int mn = M * t.n;
    constexpr int FS = FT / FPT;
    for (int idx = lane; idx < nl * mn * FS; idx += WG) {
        const int li = idx / (mn * FS), rem = idx % (mn * FS), row = rem % mn, fb = (rem / mn) * FPT;
        const C* Gl = G + (gidx * links + lids[li]) * mn * t.p + row;
        const C* e = Es + li * pF + fb;
        C acc[FPT];
#pragma unroll
        for (int ff = 0; ff < FPT; ++ff) acc[ff] = czero<C>();
        for (int q = 0; q < t.p; ++q) {
            const C gv = Gl[(int64_t)mn * q];
#pragma unroll
            for (int ff = 0; ff < FPT; ++ff) cfma(acc[ff], gv, e[q * FT + ff]);
        }
        C* d = dst[li] + row * LD + fb;
#pragma unroll
        for (int ff = 0; ff < FPT; ++ff) d[ff] = acc[ff];
    }
    group_bar(bar_id, WG);
}

// Gram tasks of one user: serving (Hermitian, M(M+1)/2 entries) and `ncross` cross Grams (M*M each)
// out[f*ostride + slot*MM + a + M b] = sum_c Hx[a + M c][f] conj(Hy[b + M c][f])  (fp64 accumulation)
template <class T, int M, int FT>
__device__ __forceinline__ void group_grams(int lane, int WG, int bar_id, int n, int Fvalid, const cplx_t<T>* Hs,
                                            int ncross, const cplx_t<T>* const* Hc, const cplx_t<T>* const* Hp,
                                            const int* slot, double2* out, int64_t ostride) {
    constexpr int LD = FT + 1, MM = M * M, HS = M * (M + 1) / 2;
    const int total = FT * (HS + ncross * MM);
    for (int idx = lane; idx < total; idx += WG) {
        const int f = idx % FT;
        int e = idx / FT;
        const cplx_t<T>*hx, *hy;
        int a, b, sl;
        bool herm = e < HS;
        if (herm) {
            a = 0;
            while (e >= M - a) { e -= M - a; ++a; }
            b = a + e;
            hx = Hs;
            hy = Hs;
            sl = 0;
        } else {
            e -= HS;
            const int c = e / MM;
            e %= MM;
            a = e % M;
            b = e / M;
            hx = Hc[c];
            hy = Hp[c];
            sl = slot[c];
        }
        if (f >= Fvalid) continue;
        const cplx_t<T>* px = hx + a * LD + f;
        const cplx_t<T>* py = hy + b * LD + f;
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll 4
        for (int c = 0; c < n; ++c) cfmac(acc, to_d2(px[M * LD * c]), to_d2(py[M * LD * c]));
        double2* o = out + f * ostride + sl * MM;
        o[a + M * b] = acc;
        if (herm && a != b) o[b + M * a] = make_double2(acc.x, -acc.y);
    }
    group_bar(bar_id, WG);
}

template <class T, int M, int FT, int FPT>
__global__ void __launch_bounds__(256) k_rebuild_gram(Topo t, FusedShape fs, int Fc, int64_t f0, int64_t Ftot,
                                                      const cplx_t<T>* __restrict__ Cd,
                                                      const cplx_t<T>* __restrict__ G, const double* __restrict__ tau,
                                                      const double* __restrict__ freqs, int uniform, double df,
                                                      const cplx_t<T>* __restrict__ coeffs, double2* __restrict__ GU) {
    using C = cplx_t<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int LD = FT + 1;
    const int J = t.J, K = t.K, B = fs.B;
    const int WG = fs.fsplit;  // threads per group
    const int NG = blockDim.x / WG;
    const int mn = M * t.n, MM = M * M;
    const size_t tile = (size_t)mn * LD;
    const size_t per_group = 2 * tile + (size_t)2 * FT * (t.P + t.p);
    C* Hpart = reinterpret_cast<C*>(smem_raw);  // [J][mn][LD]
    const int grp = threadIdx.x / WG, lane = threadIdx.x % WG, bar_id = 1 + grp;
    C* gw = Hpart + (size_t)J * tile + grp * per_group;
    C* Hw0 = gw;
    C* Hw1 = gw + tile;
    C* Ph = gw + 2 * tile;
    C* Es = Ph + (size_t)2 * FT * t.P;
    const int64_t gidx = blockIdx.z;
    const int ft0 = blockIdx.x * FT;
    const int Fvalid = min(FT, Fc - ft0);
    const int u0 = blockIdx.y * B;
    const int users = t.users();
    auto link_id = [&](int k, int i, int j) { return (k * J + i) * K + j; };
    const int64_t fstride = (int64_t)users * J * MM;
    double2* gbase = GU + ((gidx * Fc + ft0) * users) * (int64_t)J * MM;
    // partner links (k,k,0), round-robin over groups, into Hpart
    for (int k = grp; k < J; k += NG) {
        int lid[2] = {link_id(k, k, 0), 0};
        C* dst[2] = {Hpart + (size_t)k * tile, nullptr};
        group_rebuild<T, M, FT, FPT>(t, lane, WG, bar_id, 1, lid, ft0, Fc, f0, Ftot, gidx, Cd, G, tau, freqs, coeffs,
                                     Ph, Es, dst);
    }
    __syncthreads();
    const int ubeg = u0, uend = min(users, u0 + B);
    for (int u = ubeg + grp; u < uend; u += NG) {
        const int i = u / K, j = u % K;
        // cross links (k,i,j), k != i, in slot order; the serving link rides along when j != 0
        int kc = 0;
        int cross_k[8];
        for (int k = 0; k < J && kc < 8; ++k)
            if (k != i) cross_k[kc++] = k;
        const C* hs = Hpart + (size_t)i * tile;
        int done = 0;
        bool serving_pending = true;
        while (serving_pending || done < kc) {
            int lid[2];
            C* dst[2];
            int nl = 0;
            const C* Hc[2];
            const C* Hp[2];
            int slot[2];
            int ncross = 0;
            bool with_serving = false;
            if (serving_pending && j != 0) {
                lid[nl] = link_id(i, i, j);
                dst[nl] = Hw0;
                ++nl;
                hs = Hw0;
                with_serving = true;
            } else if (serving_pending) {
                with_serving = true;  // serving link is the partner tile Hpart[i]
            }
            while (nl < 2 && done < kc) {
                const int k = cross_k[done];
                lid[nl] = link_id(k, i, j);
                dst[nl] = nl == 0 ? Hw0 : Hw1;
                Hc[ncross] = dst[nl];
                Hp[ncross] = Hpart + (size_t)k * tile;
                slot[ncross] = 1 + done;
                ++ncross;
                ++nl;
                ++done;
            }
            if (nl > 0)
                group_rebuild<T, M, FT, FPT>(t, lane, WG, bar_id, nl, lid, ft0, Fc, f0, Ftot, gidx, Cd, G, tau, freqs,
                                             coeffs, Ph, Es, dst);
            if (with_serving) {
                group_grams<T, M, FT>(lane, WG, bar_id, t.n, Fvalid, hs, ncross, Hc, Hp, slot,
                                      gbase + (int64_t)u * J * MM, fstride);
            } else {
                // cross-only round: reuse the Gram routine with a dummy serving slot skipped
                constexpr int LDc = FT + 1;
                const int total = FT * ncross * MM;
                for (int idx = lane; idx < total; idx += WG) {
                    const int f = idx % FT;
                    int e = idx / FT;
                    const int c = e / MM;
                    e %= MM;
                    const int a = e % M, b = e / M;
                    if (f >= Fvalid) continue;
                    const C* px = Hc[c] + a * LDc + f;
                    const C* py = Hp[c] + b * LDc + f;
                    double2 acc = make_double2(0.0, 0.0);
                    for (int cc = 0; cc < t.n; ++cc) cfmac(acc, to_d2(px[M * LDc * cc]), to_d2(py[M * LDc * cc]));
                    gbase[(int64_t)u * J * MM + f * fstride + slot[c] * MM + a + M * b] = acc;
                }
                group_bar(bar_id, WG);
            }
            serving_pending = false;
        }
    }
}

// ---------------------------------------------------------------------------
// Whole-group rebuild + Grams (paper scope, small groups: all links of a group fit in shared
// memory): one CTA per (group, FT subcarriers); every phase runs over ALL links at once, so
// the CTA never serialises on per-link barriers. H~ stays in shared memory; output GU as above.
template <class T, int M, int FT>
__global__ void __launch_bounds__(256) k_sinr_group(Topo t, int Fc, int64_t f0, int64_t Ftot,
                                                    const cplx_t<T>* __restrict__ Cd, const cplx_t<T>* __restrict__ G,
                                                    const double* __restrict__ tau, const double* __restrict__ freqs,
                                                    const cplx_t<T>* __restrict__ coeffs, double2* __restrict__ GU) {
    using C = cplx_t<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int LD = FT + 1, MM = M * M, HS = M * (M + 1) / 2;
    const int J = t.J, K = t.K, links = t.links(), users = t.users();
    const int mn = M * t.n, P = t.P, p = t.p;
    C* H = reinterpret_cast<C*>(smem_raw);      // [links][mn][LD]   (phases 3-4)
    C* Ph = H;                                   // [links][P][FT]    (phases 1-2, aliases H)
    C* E = H + (size_t)links * mn * LD;          // [links][p][FT]
    const int64_t gidx = blockIdx.y;
    const int ft0 = blockIdx.x * FT;
    const int Fvalid = min(FT, Fc - ft0);
    const int tid = threadIdx.x, nt = blockDim.x;
    // 1. conj(c_r(f)) for every link
    for (int idx = tid; idx < links * P * FT; idx += nt) {
        const int l = idx / (P * FT), r = (idx / FT) % P, f = idx % FT;
        C v = czero<C>();
        if (f < Fvalid) {
            const int64_t fa = f0 + ft0 + f;
            v = coeffs ? cconj(coeffs[((gidx * Ftot + fa) * links + l) * P + r])
                       : conj_coeff<T>(freqs[fa], tau[(gidx * links + l) * P + r]);
        }
        Ph[idx] = v;
    }
    __syncthreads();
    // 2. E_l[q][f] = sum_r C_l(r,q) conj(c_r(f))
    for (int idx = tid; idx < links * p * FT; idx += nt) {
        const int l = idx / (p * FT), q = (idx / FT) % p, f = idx % FT;
        const C* Cl = Cd + ((gidx * links + l) * P) * (int64_t)p + (int64_t)P * q;
        const C* ph = Ph + (size_t)l * P * FT + f;
        C acc = czero<C>();
        for (int r = 0; r < P; ++r) cfma(acc, Cl[r], ph[r * FT]);
        E[idx] = acc;
    }
    __syncthreads();
    // 3. H~_l[row][f] = sum_q G_l[row + mn q] E_l[q][f], all links, one row x FT subcarriers per thread
    for (int rg = tid; rg < links * mn; rg += nt) {
        const int l = rg / mn, row = rg % mn;
        const C* Gl = G + (gidx * links + l) * (int64_t)mn * p + row;
        const C* e = E + (size_t)l * p * FT;
        C acc[FT];
#pragma unroll
        for (int f = 0; f < FT; ++f) acc[f] = czero<C>();
        for (int q = 0; q < p; ++q) {
            const C gv = Gl[(int64_t)mn * q];
#pragma unroll
            for (int f = 0; f < FT; ++f) cfma(acc[f], gv, e[q * FT + f]);
        }
        C* h = H + (size_t)rg * LD;
#pragma unroll
        for (int f = 0; f < FT; ++f) h[f] = acc[f];
    }
    __syncthreads();
    // 4. Grams per user: serving (Hermitian) + one cross Gram per other cell (fp64 accumulation)
    const int per_user = HS + (J - 1) * MM;
    const int64_t fstride = (int64_t)users * J * MM;
    double2* gbase = GU + ((gidx * Fc + ft0) * users) * (int64_t)J * MM;
    for (int idx = tid; idx < users * per_user * FT; idx += nt) {
        const int f = idx % FT;
        int e = (idx / FT) % per_user;
        const int u = idx / (FT * per_user);
        if (f >= Fvalid) continue;
        const int i = u / K, j = u % K;
        const C *hx, *hy;
        int a, b, slot;
        const bool herm = e < HS;
        if (herm) {
            a = 0;
            while (e >= M - a) { e -= M - a; ++a; }
            b = a + e;
            hx = hy = H + (size_t)((i * J + i) * K + j) * mn * LD;
            slot = 0;
        } else {
            e -= HS;
            const int c = e / MM;
            e %= MM;
            a = e % M;
            b = e / M;
            const int k = c < i ? c : c + 1;  // c-th cell != i
            hx = H + (size_t)((k * J + i) * K + j) * mn * LD;
            hy = H + (size_t)((k * J + k) * K + 0) * mn * LD;
            slot = 1 + c;
        }
        const C* px = hx + a * LD + f;
        const C* py = hy + b * LD + f;
        double2 acc0 = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
        int c = 0;
        for (; c + 1 < t.n; c += 2) {
            cfmac(acc0, to_d2(px[M * LD * c]), to_d2(py[M * LD * c]));
            cfmac(acc1, to_d2(px[M * LD * (c + 1)]), to_d2(py[M * LD * (c + 1)]));
        }
        if (c < t.n) cfmac(acc0, to_d2(px[M * LD * c]), to_d2(py[M * LD * c]));
        const double2 acc = make_double2(acc0.x + acc1.x, acc0.y + acc1.y);
        double2* o = gbase + f * fstride + (int64_t)u * J * MM + slot * MM;
        o[a + M * b] = acc;
        if (herm && a != b) o[b + M * a] = make_double2(acc.x, -acc.y);
    }
}

template <class T, int M>
static size_t group_smem(const Topo& t, int FT) {
    const size_t cs = sizeof(cplx_t<T>);
    const size_t hbytes = cs * (size_t)t.links() * M * t.n * (FT + 1);
    const size_t phbytes = cs * (size_t)t.links() * t.P * FT;
    return std::max(hbytes, phbytes) + cs * (size_t)t.links() * t.p * FT;
}

template <int M>
__device__ __forceinline__ void load_herm(const double2* src, double2 (&A)[M][M]) {
#pragma unroll
    for (int b = 0; b < M; ++b)
#pragma unroll
        for (int a = 0; a < M; ++a) A[a][b] = src[a + M * b];
#pragma unroll
    for (int a = 0; a < M; ++a) {
        A[a][a].y = 0.0;
#pragma unroll
        for (int b = a + 1; b < M; ++b) {
            const double2 v = make_double2(0.5 * (A[a][b].x + A[b][a].x), 0.5 * (A[a][b].y - A[b][a].y));
            A[a][b] = v;
            A[b][a] = make_double2(v.x, -v.y);
        }
    }
}

// one CTA per (group, subcarrier tile); thread = (f, user)
template <int M>
__global__ void __launch_bounds__(128) k_sinr_solve(Topo t, int FT, int Fc, int64_t f0, int64_t Ftot, double sigma,
                                                    const double2* __restrict__ GU, double* __restrict__ sinr,
                                                    double* __restrict__ signal, int* __restrict__ status) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int J = t.J, K = t.K, L = t.L, MM = M * M;
    const int users = t.users();
    double2* Pk = reinterpret_cast<double2*>(smem_raw);  // [FT][J][MM]
    int* pbad = reinterpret_cast<int*>(Pk + (size_t)FT * J * MM);  // [FT][J]
    const int64_t gidx = blockIdx.y;
    const int ft0 = blockIdx.x * FT;
    const int tid = threadIdx.x;
    const int f = tid / users, u = tid % users;
    const bool active = (f < FT) && (ft0 + f < Fc);
    const int i = u / K, j = u % K;
    double lam[M];
    int rank[M];
    double2 V[M][M];
    const double2* g = GU + (((gidx * Fc + ft0 + f) * users + u) * (int64_t)J) * MM;
    if (active) {
        double2 A[M][M];
        load_herm<M>(g, A);
        jacobi_herm<M>(A, V);
#pragma unroll
        for (int r = 0; r < M; ++r) lam[r] = A[r][r].x;
#pragma unroll
        for (int r = 0; r < M; ++r) {
            int rk = 0;
#pragma unroll
            for (int s2 = 0; s2 < M; ++s2) rk += (lam[s2] > lam[r] || (lam[s2] == lam[r] && s2 < r)) ? 1 : 0;
            rank[r] = rk;
        }
        if (j == 0) {  // partner projector P = U_L Lambda_L^{-1} U_L^H for the other cells' users
            double2* P = Pk + ((size_t)f * J + i) * MM;
            int bad = 0;
#pragma unroll
            for (int a = 0; a < M; ++a)
#pragma unroll
                for (int b = 0; b < M; ++b) {
                    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
                    for (int r = 0; r < M; ++r) {
                        if (rank[r] < L && lam[r] > 0.0) {
                            double2 v = make_double2(0, 0);
                            cfmac(v, V[a][r], V[b][r]);
                            const double il = 1.0 / lam[r];
                            acc.x += il * v.x;
                            acc.y += il * v.y;
                        }
                    }
                    P[a + M * b] = acc;
                }
#pragma unroll
            for (int r = 0; r < M; ++r) bad |= (rank[r] < L && !(lam[r] > 0.0));
            pbad[f * J + i] = bad;
        }
    }
    __syncthreads();
    if (!active) return;
    int st = 0;
    double2 Q[M][M];
    const double s2 = sigma * sigma;
#pragma unroll
    for (int a = 0; a < M; ++a)
#pragma unroll
        for (int b = 0; b < M; ++b) Q[a][b] = make_double2(a == b ? s2 : 0.0, 0.0);
#pragma unroll
    for (int r = 0; r < M; ++r) {
        if (rank[r] < L) {
            const double lr = fmax(lam[r], 0.0);
#pragma unroll
            for (int a = 0; a < M; ++a)
#pragma unroll
                for (int b = 0; b < M; ++b) {
                    double2 v = make_double2(0, 0);
                    cfmac(v, V[a][r], V[b][r]);
                    Q[a][b].x += lr * v.x;
                    Q[a][b].y += lr * v.y;
                }
        }
    }
    int s = 1;
    for (int k = 0; k < J; ++k) {
        if (k == i) continue;
        const double2* X = g + (int64_t)s * MM;
        const double2* P = Pk + ((size_t)f * J + k) * MM;
        if (pbad[f * J + k]) st = 5;
        double2 XP[M][M];
#pragma unroll
        for (int a = 0; a < M; ++a)
#pragma unroll
            for (int b = 0; b < M; ++b) {
                double2 acc = make_double2(0, 0);
#pragma unroll
                for (int c = 0; c < M; ++c) cfma(acc, X[a + M * c], P[c + M * b]);
                XP[a][b] = acc;
            }
#pragma unroll
        for (int a = 0; a < M; ++a)
#pragma unroll
            for (int b = 0; b < M; ++b) {
                double2 acc = Q[a][b];
#pragma unroll
                for (int c = 0; c < M; ++c) cfmac(acc, XP[a][c], X[b + M * c]);
                Q[a][b] = acc;
            }
        ++s;
    }
    bool finite = true;
#pragma unroll
    for (int a = 0; a < M; ++a)
#pragma unroll
        for (int b = 0; b < M; ++b) finite = finite && isfinite(Q[a][b].x) && isfinite(Q[a][b].y);
    bool pd = finite;
    double dmax = 0.0, dmin = 1e308;
#pragma unroll
    for (int c = 0; c < M; ++c) {
        double d = Q[c][c].x;
#pragma unroll
        for (int k2 = 0; k2 < c; ++k2) d -= Q[c][k2].x * Q[c][k2].x + Q[c][k2].y * Q[c][k2].y;
        pd = pd && (d > 0.0);
        const double inv = rsqrt(fmax(d, 1e-300));
        const double lcc = fmax(d, 1e-300) * inv;
        dmax = fmax(dmax, lcc);
        dmin = fmin(dmin, lcc);
        Q[c][c] = make_double2(lcc, inv);  // .y keeps 1/l_cc for the solves
#pragma unroll
        for (int r = c + 1; r < M; ++r) {
            double2 sacc = Q[r][c];
#pragma unroll
            for (int k2 = 0; k2 < c; ++k2) {
                sacc.x -= Q[r][k2].x * Q[c][k2].x + Q[r][k2].y * Q[c][k2].y;
                sacc.y -= Q[r][k2].y * Q[c][k2].x - Q[r][k2].x * Q[c][k2].y;
            }
            Q[r][c] = make_double2(sacc.x * inv, sacc.y * inv);
        }
    }
    if (!finite) st = 4;
    else if (!pd) st = 1;
    else if ((dmax / dmin) * (dmax / dmin) > 1e14) st = 2;
    const int64_t orow = (gidx * Ftot + f0 + ft0 + f) * users + u;
    double* so = sinr + orow * L;
    double* sg = signal + orow * L;
#pragma unroll
    for (int r = 0; r < M; ++r) {
        if (rank[r] >= L) continue;
        double gamma = 0.0;
        if (st != 1 && st != 2 && st != 4) {
            double2 y[M];
#pragma unroll
            for (int a = 0; a < M; ++a) {
                double2 acc = V[a][r];
#pragma unroll
                for (int k2 = 0; k2 < a; ++k2) {
                    acc.x -= Q[a][k2].x * y[k2].x - Q[a][k2].y * y[k2].y;
                    acc.y -= Q[a][k2].x * y[k2].y + Q[a][k2].y * y[k2].x;
                }
                y[a] = make_double2(acc.x * Q[a][a].y, acc.y * Q[a][a].y);
            }
            double nn = 0.0;
#pragma unroll
            for (int a = 0; a < M; ++a) nn += y[a].x * y[a].x + y[a].y * y[a].y;
            gamma = fmax(lam[r], 0.0) * nn;
        }
        const double sp = gamma * gamma;
        double den = gamma * (1.0 - gamma);
        if (den <= -1e-12 && st == 0) st = 3;
        den = fmax(den, 2.2250738585072014e-308);
        so[rank[r]] = sp / den;
        sg[rank[r]] = sp;
    }
    status[orow] = st;
}

template <class T, int M>
static cudaError_t launch_fused_m(const Topo& t, int ngroups, int Fc, int64_t f0, int64_t Ftot, double sigma,
                                  const void* Cd, const void* G, const double* tau, const double* freqs, int uniform,
                                  double df, const void* coeffs, double2* GU, double* sinr, double* signal,
                                  int* status, cudaStream_t st) {
    const size_t cs = sizeof(cplx_t<T>);
    const int users = t.users();
    const int mn = M * t.n;
    cudaError_t e = cudaSuccess;
    const char* eft = std::getenv("GWT_RG_FT");
    int gFT = 0;  // whole-group kernel tile (0 = does not fit)
    for (int cand : {8, 4, 2})
        if (!gFT && group_smem<T, M>(t, cand) <= (cand >= 4 ? 110 * 1024 : 200 * 1024)) gFT = cand;
    if (eft) gFT = std::atoi(eft) == 8 || std::atoi(eft) == 4 || std::atoi(eft) == 2 ? std::atoi(eft) : gFT;
    if (gFT && group_smem<T, M>(t, gFT) <= 220 * 1024) {
        auto rung = [&](auto ftc) {
            constexpr int FT = decltype(ftc)::value;
            const size_t sm = group_smem<T, M>(t, FT);
            e = cudaFuncSetAttribute(k_sinr_group<T, M, FT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            if (e != cudaSuccess) return;
            dim3 g((Fc + FT - 1) / FT, ngroups);
            k_sinr_group<T, M, FT><<<g, 256, sm, st>>>(t, Fc, f0, Ftot, (const cplx_t<T>*)Cd, (const cplx_t<T>*)G, tau,
                                                       freqs, (const cplx_t<T>*)coeffs, GU);
            e = cudaGetLastError();
        };
        if (gFT == 8) rung(std::integral_constant<int, 8>{});
        else if (gFT == 4) rung(std::integral_constant<int, 4>{});
        else rung(std::integral_constant<int, 2>{});
        if (e != cudaSuccess) return e;
    } else {
    // rebuild+Gram: FT subcarriers per CTA tile, a group of WG threads per user (named barriers).
    // GWT_RG_FT / GWT_RG_WG override the defaults (tuning).
    const int FTsel = eft ? std::atoi(eft) : 16;
    const char* ewg = std::getenv("GWT_RG_WG");
    int WG = ewg ? std::atoi(ewg) : (mn <= 128 ? 128 : 256);
    if (WG < 32 || 256 % WG) WG = 256;
    const int NG = 256 / WG;
    FusedShape fs;
    fs.B = std::min(users, 32);
    fs.fsplit = WG;
    auto run = [&](auto ftc) {
        constexpr int FT = decltype(ftc)::value;
        fs.FT = FT;
        const size_t tile = (size_t)mn * (FT + 1);
        const size_t sm1 = cs * ((size_t)t.J * tile + (size_t)NG * (2 * tile + (size_t)2 * FT * (t.P + t.p)));
        if (sm1 > 220 * 1024) { e = cudaErrorInvalidValue; return; }
        dim3 g1((Fc + FT - 1) / FT, (users + fs.B - 1) / fs.B, ngroups);
        e = cudaFuncSetAttribute(k_rebuild_gram<T, M, FT, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
        if (e != cudaSuccess) return;
        k_rebuild_gram<T, M, FT, 8><<<g1, 256, sm1, st>>>(t, fs, Fc, f0, Ftot, (const cplx_t<T>*)Cd,
                                                          (const cplx_t<T>*)G, tau, freqs, uniform, df,
                                                          (const cplx_t<T>*)coeffs, GU);
        e = cudaGetLastError();
    };
    if (FTsel == 8) run(std::integral_constant<int, 8>{});
    else run(std::integral_constant<int, 16>{});
    if (e != cudaSuccess) return e;
    }
    // solve: (users x FT2) threads per CTA, FT2 = 128 / users (>= 1)
    const int FT2 = std::max(1, 128 / users);
    const size_t sm2 = (size_t)FT2 * t.J * (16 * M * M + 4) + 16;
    dim3 g2((Fc + FT2 - 1) / FT2, ngroups);
    k_sinr_solve<M><<<g2, std::max(32, ((FT2 * users + 31) / 32) * 32), sm2, st>>>(t, FT2, Fc, f0, Ftot, sigma, GU,
                                                                                sinr, signal, status);
    return cudaGetLastError();
}

template <class T>
cudaError_t launch_sinr_fused(const Topo& t, int ngroups, int Fc, int64_t f0, int64_t Ftot, double sigma,
                              const void* Cd, const void* G, const double* tau, const double* freqs, int uniform,
                              double df, const void* coeffs, double2* GU, double* sinr, double* signal, int* status,
                              cudaStream_t st) {
    if (t.users() > 128) return cudaErrorInvalidValue;
    switch (t.m) {
#define GWT_FUSED_CASE(MM)                                                                                         \
    case MM:                                                                                                       \
        return launch_fused_m<T, MM>(t, ngroups, Fc, f0, Ftot, sigma, Cd, G, tau, freqs, uniform, df, coeffs, GU, \
                                     sinr, signal, status, st);
        GWT_FUSED_CASE(1) GWT_FUSED_CASE(2) GWT_FUSED_CASE(3) GWT_FUSED_CASE(4)
        GWT_FUSED_CASE(5) GWT_FUSED_CASE(6) GWT_FUSED_CASE(7) GWT_FUSED_CASE(8)
#undef GWT_FUSED_CASE
        default: return cudaErrorInvalidValue;
    }
}

template cudaError_t launch_sinr_fused<float>(const Topo&, int, int, int64_t, int64_t, double, const void*,
                                              const void*, const double*, const double*, int, double, const void*,
                                              double2*, double*, double*, int*, cudaStream_t);
template cudaError_t launch_sinr_fused<double>(const Topo&, int, int, int64_t, int64_t, double, const void*,
                                               const void*, const double*, const double*, int, double, const void*,
                                               double2*, double*, double*, int*, cudaStream_t);

// ---------------------------------------------------------------------------
// launchers

template <class T>
cudaError_t launch_rebuild(const Topo& t, int ngroups, int Fc, int64_t f0, int64_t Ftot, const void* Cd,
                           const void* G, const double* tau, const double* freqs, const void* coeffs, void* H,
                           cudaStream_t st) {
    using C = cplx_t<T>;
    constexpr int FT = 16;
    const char* rtc = std::getenv("GWT_REBUILD_TC");
    if (sizeof(T) == 4 && !coeffs && rtc && std::atoi(rtc) != 0) {
        // tensor-core rebuild (k_tc.cu, opt-in) when the shape fits; else the CUDA-core kernels below
        cudaError_t e = launch_rebuild_tc(t, ngroups, Fc, f0, Cd, G, tau, freqs, H, st);
        if (e != cudaErrorNotSupported) return e;
        cudaGetLastError();
    }
    if (sizeof(T) == 4 && !coeffs && rebuild_mm_fits(t) && !std::getenv("GWT_REBUILD_RB")) {
        cudaError_t e = launch_rebuild_mm(t, ngroups, Fc, f0, Cd, G, tau, freqs, H, st);
        if (e != cudaErrorNotSupported) return e;
        cudaGetLastError();
    }
    if (!coeffs && !std::getenv("GWT_REBUILD_V1")) {
        // subcarrier tile: 64 while the phasor tile (P x 64) stays <= 16 KB (C1/C2), else 32 (C3-C5:
        // P = 48/64, where FT = 64 halves the resident CTAs); GWT_REBUILD_FT overrides
        const char* ftv = std::getenv("GWT_REBUILD_FT");
        const int ft = ftv ? std::atoi(ftv) : (t.P * 64 * (int)sizeof(C) <= 16 * 1024 ? 64 : 32);
        cudaError_t e = (ft == 32)
                            ? launch_rebuild_rb<T, 32>(t, ngroups, Fc, f0, Cd, G, tau, freqs, H, st)
                            : launch_rebuild_rb<T, 64>(t, ngroups, Fc, f0, Cd, G, tau, freqs, H, st);
        if (e != cudaErrorNotSupported) return e;
        cudaGetLastError();
    }
    {
        constexpr int FTL = 32;
        const size_t sm = sizeof(C) * ((size_t)t.p * t.m * t.n + (size_t)t.p * t.P + (size_t)t.P * FTL + (size_t)t.p * FTL) +
                          8 * (size_t)t.P;
        if (!coeffs && sm <= 200 * 1024 && !std::getenv("GWT_REBUILD_TILED")) {
            // split the subcarriers so the grid covers >= ~8 CTAs per SM
            const int64_t base = (int64_t)ngroups * t.links();
            int nz = (int)std::max<int64_t>(1, std::min<int64_t>((148 * 8 + base - 1) / base, (Fc + 2 * FTL - 1) / (2 * FTL)));
            int frange = (Fc + nz - 1) / nz;
            frange = (frange + FTL - 1) / FTL * FTL;
            nz = (Fc + frange - 1) / frange;
            cudaError_t e = cudaFuncSetAttribute(k_rebuild_link<T, FTL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            if (e != cudaSuccess) return e;
            dim3 g2(t.links(), ngroups, nz);
            k_rebuild_link<T, FTL><<<g2, 128, sm, st>>>(t, Fc, f0, Ftot, frange, (const C*)Cd, (const C*)G, tau, freqs, (C*)H);
            return cudaGetLastError();
        }
    }
    dim3 grid((Fc + FT - 1) / FT, t.links(), ngroups);
    const size_t sm = sizeof(C) * (size_t)(t.P + t.p) * FT;
    if (sm > 48 * 1024)
        cudaFuncSetAttribute(k_rebuild<T, FT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_rebuild<T, FT><<<grid, 128, sm, st>>>(t, Fc, f0, Ftot, (const C*)Cd, (const C*)G, tau, freqs,
                                            (const C*)coeffs, (C*)H);
    return cudaGetLastError();
}

template <class T>
cudaError_t launch_pair_gram(const Topo& t, int scope, int S, int Fc, int ngroups, int64_t f0, int64_t Ftot,
                             const void* H, double2* PG, cudaStream_t st) {
    const int64_t items = (int64_t)ngroups * Fc * t.users();
    const int wpb = 4;
    const size_t smf = sizeof(double2) * (size_t)t.links() * t.m * t.n;
    if (sizeof(T) == 4 && scope == 1 && smf <= 48 * 1024 && t.m <= 8 && ((t.links() * t.m * t.n) % 2 == 0) &&
        std::getenv("GWT_PG_PIPE")) {
        const size_t sm = 2 * smf;  // two raw complex64 buffers + one binary64 buffer
        const int64_t nsl = (int64_t)ngroups * Fc;
        const int thr = (int)std::min<int64_t>(256, ((int64_t)t.users() * t.J * t.m * t.m + 31) / 32 * 32);
        int per_sm = 0;
        cudaError_t e = cudaSuccess;
        switch (t.m) {
#define GWT_PGP(MM)                                                                                               \
    case MM:                                                                                                      \
        e = cudaFuncSetAttribute(k_pair_gram_pipe<MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);     \
        if (e != cudaSuccess) return e;                                                                           \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pair_gram_pipe<MM>, thr, sm);                   \
        k_pair_gram_pipe<MM><<<(unsigned)std::min<int64_t>(nsl, 148 * std::max(per_sm, 1)), thr, sm, st>>>(       \
            t, Fc, f0, Ftot, nsl, (const float2*)H, PG);                                                          \
        return cudaGetLastError();
            GWT_PGP(1) GWT_PGP(2) GWT_PGP(3) GWT_PGP(4) GWT_PGP(5) GWT_PGP(6) GWT_PGP(7) GWT_PGP(8)
#undef GWT_PGP
        }
    }
    if (scope == 1 && smf <= 64 * 1024 && t.m <= 8 && !std::getenv("GWT_PG_STAGED")) {
        const int mn = t.m * t.n, LS = mn + ((4 - mn % 8) + 8) % 8;
        const size_t smp = sizeof(double2) * (size_t)t.links() * LS;
        const int thr = (int)std::min<int64_t>(256, ((int64_t)t.users() * t.J * t.m * t.m + 31) / 32 * 32);
        dim3 grid(Fc, ngroups);
        cudaError_t e = cudaSuccess;
        switch (t.m) {
#define GWT_PGF(MM)                                                                                              \
    case MM:                                                                                                     \
        e = cudaFuncSetAttribute(k_pair_gram_gf<T, MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smp);  \
        if (e != cudaSuccess) return e;                                                                          \
        k_pair_gram_gf<T, MM><<<grid, thr, smp, st>>>(t, Fc, f0, Ftot, LS, (const cplx_t<T>*)H, PG);             \
        return cudaGetLastError();
            GWT_PGF(1) GWT_PGF(2) GWT_PGF(3) GWT_PGF(4) GWT_PGF(5) GWT_PGF(6) GWT_PGF(7) GWT_PGF(8)
#undef GWT_PGF
        }
    }
    const size_t sm = sizeof(double2) * (size_t)wpb * (2 * t.J - 1) * t.m * t.n;
    if (scope == 1 && sm <= 96 * 1024 && !std::getenv("GWT_PG_UNSTAGED")) {
        cudaError_t e = cudaSuccess;
        switch (t.m) {
#define GWT_PGS(MM)                                                                                                  \
    case MM:                                                                                                         \
        e = cudaFuncSetAttribute(k_pair_gram_staged<T, MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);   \
        if (e != cudaSuccess) return e;                                                                              \
        k_pair_gram_staged<T, MM><<<(unsigned)((items + wpb - 1) / wpb), 32 * wpb, sm, st>>>(t, Fc, f0, Ftot, items, \
                                                                                            (const cplx_t<T>*)H, PG); \
        return cudaGetLastError();
            GWT_PGS(1) GWT_PGS(2) GWT_PGS(3) GWT_PGS(4) GWT_PGS(5) GWT_PGS(6) GWT_PGS(7) GWT_PGS(8)
#undef GWT_PGS
            default: break;
        }
    }
    k_pair_gram<T><<<(unsigned)((items + wpb - 1) / wpb), 32 * wpb, 0, st>>>(t, scope, S, Fc, f0, Ftot, items,
                                                                            (const cplx_t<T>*)H, PG);
    return cudaGetLastError();
}

template <int M>
static cudaError_t launch_small_m(const Topo& t, int scope, int S, int64_t items, double sigma, int fc, int64_t Ftot,
                                  int64_t f0, const double2* PG, double* EG, double* sinr, double* signal, int* status,
                                  cudaStream_t st) {
    const int users = t.users();
    if (users <= 128 && !std::getenv("GWT_SMALL_SPLIT")) {
        const int thr = (128 / users) * users;  // whole (group, subcarrier) slices per CTA
        const int Lp = (t.L + 1) & ~1;
        const size_t sm = (size_t)thr * (Lp + 2 * M * t.L) * 8;
        cudaError_t e = cudaFuncSetAttribute(k_small_fused<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
        k_small_fused<M><<<(unsigned)((items + thr - 1) / thr), thr, sm, st>>>(t, scope, S, items, sigma, fc, Ftot, f0,
                                                                                PG, sinr, signal, status);
        return cudaGetLastError();
    }
    const unsigned blocks = (unsigned)((items + 127) / 128);
    k_precoder_eig<M><<<blocks, 128, 0, st>>>(t, scope, S, items, PG, EG);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_mmse<M><<<blocks, 128, 0, st>>>(t, scope, S, items, sigma, fc, Ftot, f0, PG, EG, sinr, signal, status);
    return cudaGetLastError();
}

template <int M>
static cudaError_t launch_small_grp(const Topo& t, int scope, int S, int64_t items, double sigma, int fc,
                                    int64_t Ftot, int64_t f0, const double2* PG, double* sinr, double* signal,
                                    int* status, cudaStream_t st) {
    const int users = t.users();
    const int64_t nsl = items / users;
    const int spc = std::max(1, 128 / (users * 8));
    const size_t per_slice = (size_t)users * (64 * 16 * 2 + 8 * 8);
    const size_t sm = per_slice * spc;
    cudaError_t e = cudaFuncSetAttribute(k_small_grp<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k_small_grp<M><<<(unsigned)((nsl + spc - 1) / spc), users * 8 * spc, sm, st>>>(t, scope, S, nsl, spc, sigma, fc,
                                                                                   Ftot, f0, PG, sinr, signal, status);
    return cudaGetLastError();
}

cudaError_t launch_sinr_small(const Topo& t, int scope, int S, int64_t items, double sigma, int fc, int64_t Ftot,
                              int64_t f0, const double2* PG, double* EG, double* sinr, double* signal, int* status,
                              cudaStream_t st) {
    const char* grp = std::getenv("GWT_SMALL_GRP");  // 1: force the 8-lanes-per-user kernel, 0: never
    const bool use_grp = t.users() * 8 <= 256 && (grp ? std::atoi(grp) != 0 : t.m > 4);
    if (use_grp) {
        switch (t.m) {
            case 1: return launch_small_grp<1>(t, scope, S, items, sigma, fc, Ftot, f0, PG, sinr, signal, status, st);
            case 2: return launch_small_grp<2>(t, scope, S, items, sigma, fc, Ftot, f0, PG, sinr, signal, status, st);
            case 3: return launch_small_grp<3>(t, scope, S, items, sigma, fc, Ftot, f0, PG, sinr, signal, status, st);
            case 4: return launch_small_grp<4>(t, scope, S, items, sigma, fc, Ftot, f0, PG, sinr, signal, status, st);
            case 5: return launch_small_grp<5>(t, scope, S, items, sigma, fc, Ftot, f0, PG, sinr, signal, status, st);
            case 6: return launch_small_grp<6>(t, scope, S, items, sigma, fc, Ftot, f0, PG, sinr, signal, status, st);
            case 7: return launch_small_grp<7>(t, scope, S, items, sigma, fc, Ftot, f0, PG, sinr, signal, status, st);
            case 8: return launch_small_grp<8>(t, scope, S, items, sigma, fc, Ftot, f0, PG, sinr, signal, status, st);
            default: break;
        }
    }
    switch (t.m) {
        case 1: return launch_small_m<1>(t, scope, S, items, sigma, fc, Ftot, f0, PG, EG, sinr, signal, status, st);
        case 2: return launch_small_m<2>(t, scope, S, items, sigma, fc, Ftot, f0, PG, EG, sinr, signal, status, st);
        case 3: return launch_small_m<3>(t, scope, S, items, sigma, fc, Ftot, f0, PG, EG, sinr, signal, status, st);
        case 4: return launch_small_m<4>(t, scope, S, items, sigma, fc, Ftot, f0, PG, EG, sinr, signal, status, st);
        case 5: return launch_small_m<5>(t, scope, S, items, sigma, fc, Ftot, f0, PG, EG, sinr, signal, status, st);
        case 6: return launch_small_m<6>(t, scope, S, items, sigma, fc, Ftot, f0, PG, EG, sinr, signal, status, st);
        case 7: return launch_small_m<7>(t, scope, S, items, sigma, fc, Ftot, f0, PG, EG, sinr, signal, status, st);
        case 8: return launch_small_m<8>(t, scope, S, items, sigma, fc, Ftot, f0, PG, EG, sinr, signal, status, st);
        default: return cudaErrorInvalidValue;
    }
}

template cudaError_t launch_rebuild<float>(const Topo&, int, int, int64_t, int64_t, const void*, const void*,
                                           const double*, const double*, const void*, void*, cudaStream_t);
template cudaError_t launch_rebuild<double>(const Topo&, int, int, int64_t, int64_t, const void*, const void*,
                                            const double*, const double*, const void*, void*, cudaStream_t);
template cudaError_t launch_pair_gram<float>(const Topo&, int, int, int, int, int64_t, int64_t, const void*, double2*,
                                             cudaStream_t);
template cudaError_t launch_pair_gram<double>(const Topo&, int, int, int, int, int64_t, int64_t, const void*,
                                              double2*, cudaStream_t);

}  // namespace gwtk
