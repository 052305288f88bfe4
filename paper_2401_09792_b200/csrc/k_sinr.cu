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
    const char* gse = env_once("GWT_REBUILD_GSMEM");
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
            const double sc = frsqrt(fmax(lr, 1e-300));
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
        const double dc = fmax(d, 1e-300);
        const double inv = frsqrt(dc), lcc = dc * inv;  // 1 / L_cc rides in the diagonal's imaginary slot
        dmax = fmax(dmax, lcc);
        dmin = fmin(dmin, lcc);
        Q[c][c] = make_double2(lcc, inv);
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
    else if (dmax * dmax > 1e14 * (dmin * dmin)) st = 2;
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
                y[a] = make_double2(acc.x * Q[a][a].y, acc.y * Q[a][a].y);
            }
            double nn = 0.0;
#pragma unroll
            for (int a = 0; a < M; ++a) nn += y[a].x * y[a].x + y[a].y * y[a].y;
            gamma = lr * nn;  // g^H Q^{-1} g
        }
        const double sp = gamma * gamma;
        double den = gamma * (1.0 - gamma);  // w^H Q w - |w^H g|^2
        if (den <= -1e-12 && st == 0) st = 3 + (r << 8);  // code 3, first failing stream in bits 8+
        den = fmax(den, 2.2250738585072014e-308);
        so[r] = sp * frcp(den);
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
                const double rb = frsqrt(b2);
                phr = apq.x * rb;
                phi = apq.y * rb;
                const float tau = (float)((aqq.x - app.x) * (0.5 * rb));
                const float tf = copysignf(1.0f, tau) / (fabsf(tau) + sqrtf(fmaf(tau, tau, 1.0f)));
                const double tt = (double)tf;
                c = frsqrt(fma(tt, tt, 1.0));
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
    else if (dmax * dmax > 1e14 * (dmin * dmin)) st = 2;
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
        // code 3 carries the first failing stream (the lowest lane) in bits 8+
        const unsigned m3 = (__ballot_sync(0xffffffffu, st == 3) >> base) & 0xffu;
        if (valid && j == 0) status[orow] = ((st == 0 || st == 3) && m3) ? 3 + ((__ffs(m3) - 1) << 8) : st;
    }
}



// ---------------------------------------------------------------------------
// launchers

template <class T>
cudaError_t launch_rebuild(const Topo& t, int ngroups, int Fc, int64_t f0, int64_t Ftot, const void* Cd,
                           const void* G, const double* tau, const double* freqs, const void* coeffs, void* H,
                           cudaStream_t st) {
    using C = cplx_t<T>;
    constexpr int FT = 16;
    if (sizeof(T) == 4 && !coeffs && rebuild_mm_fits(t) && !env_once("GWT_REBUILD_RB")) {
        cudaError_t e = launch_rebuild_mm(t, ngroups, Fc, f0, Cd, G, tau, freqs, H, st);
        if (e != cudaErrorNotSupported) return e;
        cudaGetLastError();
    }
    if (!coeffs && !env_once("GWT_REBUILD_V1")) {
        // subcarrier tile: 64 while the phasor tile (P x 64) stays <= 16 KB (C1/C2), else 32 (C3-C5:
        // P = 48/64, where FT = 64 halves the resident CTAs); GWT_REBUILD_FT overrides
        const char* ftv = env_once("GWT_REBUILD_FT");
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
        if (!coeffs && sm <= 200 * 1024 && !env_once("GWT_REBUILD_TILED")) {
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
    if (scope == 1 && smf <= 64 * 1024 && t.m <= 8 && !env_once("GWT_PG_STAGED")) {
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
    if (scope == 1 && sm <= 96 * 1024 && !env_once("GWT_PG_UNSTAGED")) {
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
    if (users <= 128 && !env_once("GWT_SMALL_SPLIT")) {
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
    const char* grp = env_once("GWT_SMALL_GRP");  // 1: force the 8-lanes-per-user kernel, 0: never
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
