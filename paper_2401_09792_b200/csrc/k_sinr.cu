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
#include "kernels.cuh"

namespace gwtk {

// ---------------------------------------------------------------------------
// K1: rebuild H~(f) = sum_q G(:,:,q) * E[q][f],
//     E[q][f] = sum_r C(r,q) * conj(c_r(f)),  c_r(f) = exp(+j 2 pi f tau_r) or explicit.
// grid (ceil(Fc/FT), links, groups); one CTA per (link, subcarrier tile).
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
    for (int idx = threadIdx.x; idx < t.P * FT; idx += blockDim.x) {
        const int r = idx / FT, f = idx % FT;
        C v = czero<C>();
        if (f < nf) {
            const int64_t fa = f0 + ft0 + f;
            if (coeffs) {
                v = cconj(coeffs[(((int64_t)g * Ftot + fa) * links + l) * t.P + r]);
            } else {
                v = from_d2<C>(phasor_neg(freqs[fa], tau[gl * t.P + r]));
            }
        }
        ph[idx] = v;
    }
    __syncthreads();
    const C* Cl = Cd + gl * t.P * t.p;
    for (int idx = threadIdx.x; idx < t.p * FT; idx += blockDim.x) {
        const int q = idx / FT, f = idx % FT;
        C acc = czero<C>();
        for (int r = 0; r < t.P; ++r) cfma(acc, Cl[r + t.P * q], ph[r * FT + f]);
        E[idx] = acc;
    }
    __syncthreads();
    const int mn = t.m * t.n;
    const C* Gl = G + gl * mn * t.p;
    for (int row = threadIdx.x; row < mn; row += blockDim.x) {
        C acc[FT];
#pragma unroll
        for (int f = 0; f < FT; ++f) acc[f] = czero<C>();
        for (int q = 0; q < t.p; ++q) {
            const C gv = Gl[row + (int64_t)mn * q];
#pragma unroll
            for (int f = 0; f < FT; ++f) cfma(acc[f], gv, E[q * FT + f]);
        }
#pragma unroll
        for (int f = 0; f < FT; ++f)
            if (f < nf) H[(((int64_t)g * Fc + ft0 + f) * links + l) * mn + row] = acc[f];
    }
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
__global__ void __launch_bounds__(128) k_pair_gram(Topo t, int scope, int S, int Fc, int64_t items,
                                                   const cplx_t<T>* __restrict__ H, double2* __restrict__ PG) {
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
    for (int e = lane; e < total; e += 32) {
        const int s = e / (m * m);
        const int ab = e % (m * m);
        const int a = ab % m, b = ab / m;
        int k, l;
        scope_slot(t, scope, i, j, s, k, l);
        const C* h1 = Hgf + (int64_t)((k * t.J + i) * t.K + j) * mn;  // receive link (k,i,j)
        const C* h2 = Hgf + (int64_t)((k * t.J + k) * t.K + l) * mn;  // partner's serving link (k,k,l)
        double2 acc = make_double2(0.0, 0.0);
        for (int c = 0; c < n; ++c) cfmac(acc, to_d2(h1[a + m * c]), to_d2(h2[b + m * c]));
        PG[(item * S + s) * m * m + a + m * b] = acc;
    }
}

// ---------------------------------------------------------------------------
// Per-thread small Hermitian eigensolver (cyclic complex Jacobi, fp64), the
// rotation of the reference test oracle (proj/tests/support/oracles.hpp:31-97).
template <int M>
__device__ __forceinline__ void jacobi_herm(double2 (&A)[M][M], double2 (&V)[M][M]) {
#pragma unroll
    for (int r = 0; r < M; ++r)
#pragma unroll
        for (int c = 0; c < M; ++c) V[r][c] = make_double2(r == c ? 1.0 : 0.0, 0.0);
    for (int sweep = 0; sweep < 32; ++sweep) {
        double off = 0.0, dia = 0.0;
#pragma unroll
        for (int p = 0; p < M; ++p) {
            dia += A[p][p].x * A[p][p].x;
#pragma unroll
            for (int q = p + 1; q < M; ++q) off += A[p][q].x * A[p][q].x + A[p][q].y * A[p][q].y;
        }
        if (off <= 1e-34 * dia || off == 0.0) break;
#pragma unroll
        for (int p = 0; p < M; ++p)
#pragma unroll
            for (int q = p + 1; q < M; ++q) {
                const double b = hypot(A[p][q].x, A[p][q].y);
                if (b > 1e-300) {
                    const double phr = A[p][q].x / b, phi = A[p][q].y / b;  // phase = apq/|apq|
                    const double alpha = A[p][p].x, delta = A[q][q].x;
                    const double tau = (delta - alpha) / (2.0 * b);
                    const double tt = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                    const double c = 1.0 / sqrt(1.0 + tt * tt);
                    const double s = tt * c;
                    // U = [[c, s], [-s conj(ph), c conj(ph)]]
                    const double2 uqp = make_double2(-s * phr, s * phi);
                    const double2 uqq = make_double2(c * phr, -c * phi);
#pragma unroll
                    for (int r = 0; r < M; ++r) {  // A <- A U (columns p, q)
                        const double2 arp = A[r][p], arq = A[r][q];
                        double2 np = make_double2(c * arp.x, c * arp.y);
                        cfma(np, arq, uqp);
                        double2 nq = make_double2(s * arp.x, s * arp.y);
                        cfma(nq, arq, uqq);
                        A[r][p] = np;
                        A[r][q] = nq;
                    }
#pragma unroll
                    for (int cc = 0; cc < M; ++cc) {  // A <- U^H A (rows p, q)
                        const double2 apc = A[p][cc], aqc = A[q][cc];
                        double2 np = make_double2(c * apc.x, c * apc.y);
                        cfmaconj(np, uqp, aqc);
                        double2 nq = make_double2(s * apc.x, s * apc.y);
                        cfmaconj(nq, uqq, aqc);
                        A[p][cc] = np;
                        A[q][cc] = nq;
                    }
#pragma unroll
                    for (int r = 0; r < M; ++r) {  // V <- V U
                        const double2 vrp = V[r][p], vrq = V[r][q];
                        double2 np = make_double2(c * vrp.x, c * vrp.y);
                        cfma(np, vrq, uqp);
                        double2 nq = make_double2(s * vrp.x, s * vrp.y);
                        cfma(nq, vrq, uqq);
                        V[r][p] = np;
                        V[r][q] = nq;
                    }
                }
            }
    }
}

// ---------------------------------------------------------------------------
// K3a: precoder per (group, subcarrier, user): eig of the serving Gram ->
// top-L eigenpairs (descending). EG layout per item: lambda[L] (padded to even) then U[M][L]
// column-major (M x L), fp64.
template <int M>
__global__ void __launch_bounds__(128) k_precoder_eig(Topo t, int scope, int S, int64_t items,
                                                      const double2* __restrict__ PG, double* __restrict__ EG) {
    const int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= items) return;
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
    double* dst = EG + item * (int64_t)(Lp + 2 * M * L);
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

// ---------------------------------------------------------------------------
// K3b: covariance, Cholesky (with the reference's PD and condition checks),
// filter and per-stream SINR; one thread per (group, subcarrier, user).
template <int M>
__global__ void __launch_bounds__(128) k_mmse(Topo t, int scope, int S, int64_t items, double sigma, int fc,
                                              int64_t Ftot, int64_t f0, const double2* __restrict__ PG,
                                              const double* __restrict__ EG,
                                              double* __restrict__ sinr, double* __restrict__ signal,
                                              int* __restrict__ status) {
    const int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= items) return;
    const int L = t.L;
    const int users = t.users();
    const int u = (int)(item % users);
    const int64_t gf = item / users;
    const int i = u / t.K, j = u % t.K;
    const int Lp = (L + 1) & ~1;
    const int64_t eg_stride = Lp + 2 * M * L;
    const double* own = EG + item * eg_stride;
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
        const int64_t pidx = gf * users + (k * t.K + l);
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

// ---------------------------------------------------------------------------
// launchers

template <class T>
cudaError_t launch_rebuild(const Topo& t, int ngroups, int Fc, int64_t f0, int64_t Ftot, const void* Cd,
                           const void* G, const double* tau, const double* freqs, const void* coeffs, void* H,
                           cudaStream_t st) {
    using C = cplx_t<T>;
    constexpr int FT = 16;
    dim3 grid((Fc + FT - 1) / FT, t.links(), ngroups);
    const size_t sm = sizeof(C) * (size_t)(t.P + t.p) * FT;
    if (sm > 48 * 1024)
        cudaFuncSetAttribute(k_rebuild<T, FT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_rebuild<T, FT><<<grid, 128, sm, st>>>(t, Fc, f0, Ftot, (const C*)Cd, (const C*)G, tau, freqs,
                                            (const C*)coeffs, (C*)H);
    return cudaGetLastError();
}

template <class T>
cudaError_t launch_pair_gram(const Topo& t, int scope, int S, int Fc, int ngroups, const void* H, double2* PG,
                             cudaStream_t st) {
    const int64_t items = (int64_t)ngroups * Fc * t.users();
    const int wpb = 4;
    k_pair_gram<T><<<(unsigned)((items + wpb - 1) / wpb), 32 * wpb, 0, st>>>(t, scope, S, Fc, items,
                                                                            (const cplx_t<T>*)H, PG);
    return cudaGetLastError();
}

template <int M>
static cudaError_t launch_small_m(const Topo& t, int scope, int S, int64_t items, double sigma, int fc, int64_t Ftot,
                                  int64_t f0, const double2* PG, double* EG, double* sinr, double* signal, int* status,
                                  cudaStream_t st) {
    const unsigned blocks = (unsigned)((items + 127) / 128);
    k_precoder_eig<M><<<blocks, 128, 0, st>>>(t, scope, S, items, PG, EG);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_mmse<M><<<blocks, 128, 0, st>>>(t, scope, S, items, sigma, fc, Ftot, f0, PG, EG, sinr, signal, status);
    return cudaGetLastError();
}

cudaError_t launch_sinr_small(const Topo& t, int scope, int S, int64_t items, double sigma, int fc, int64_t Ftot,
                              int64_t f0, const double2* PG, double* EG, double* sinr, double* signal, int* status,
                              cudaStream_t st) {
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
template cudaError_t launch_pair_gram<float>(const Topo&, int, int, int, int, const void*, double2*, cudaStream_t);
template cudaError_t launch_pair_gram<double>(const Topo&, int, int, int, int, const void*, double2*, cudaStream_t);

}  // namespace gwtk
