// Stage S of the compressed-form SINR (paper_experiment scope), one kernel per
// subcarrier chunk after the rebuild K1 (H~ in HBM, [g][f][link][n][m]).
//
// Reference: proj/src/sinr.cpp:162-254 (precoder_compressed -> covariance_compressed
// -> woodbury_inverse_apply -> filter_compressed -> sinr_compressed) for every user
// of a ChannelSet at one coefficient grid, scope pairs of sinr.cpp:47-62.
//
// Reformulation (algebraically identical):
//  * serving Gram A = H~ H~^H (m x m, binary64 accumulation of the stored H~);
//    Hermitian eig A = U diag(lambda) U^H; the SVD precoder is V = H~^H U_L L^-1/2.
//  * precoders of the interfering scope users (k, 0) are formed explicitly,
//    V'_k = H~_kk0^H U'_L L'^-1/2 (n x L), once per (group, subcarrier), and every
//    interference term is Y = H~_kij V'_k (m x L) — products of stored-precision
//    values, the Gram of the anchor never enters (no kappa^2 amplification).
//  * Q = sigma^2 I + U_L L_L U_L^H (= A when L = m) + sum_k Y Y^H, Cholesky with the
//    reference's PD / condition / finiteness checks, gamma_r = lambda_r ||L^-1 u_r||^2,
//    SINR_r = gamma_r / (1 - gamma_r) (= s / (w^H Q w - s) of stream_sinrs).
//
// Mapping: a CTA holds SPC whole (group, subcarrier) slices; MP lanes per user
// (MP = 4 for m <= 4, 8 for m <= 8; rows >= m are zero padding), lane r owns row r.
//  eig: Householder tridiagonalisation (LAPACK zhetd2 / zlarfg conventions) on the
//  per-user shared-memory matrix, implicit QL with Wilkinson shift (tql2) on the real
//  tridiagonal — the scalar recurrence is carried by every lane of the user (static
//  register indexing, rotations predicated), each lane rotating its own row of Z —
//  then the back-transform with lane = eigenvector.
#include <cfloat>
#include <type_traits>

#include "kernels.cuh"

#ifndef GWT_QL_LANES
#define GWT_QL_LANES 4  // lanes per user in the packed QL phase (each rotates MP / GWT_QL_LANES rows of Z)
#endif

namespace gwtk {

namespace {

template <int MP> __device__ __forceinline__ unsigned seg_mask(int lane) {
    return MP == 32 ? 0xffffffffu : (((1u << MP) - 1u) << (lane & ~(MP - 1)));
}

template <int MP> __device__ __forceinline__ double seg_sum(double v) {
#pragma unroll
    for (int o = MP / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double2 dmul(double2 a, double2 b) { return cmul(a, b); }

// Implicit QL (tql2 with Wilkinson shift) on the real tridiagonal (d, e); this lane rotates RL rows of Z
// (rows row0 .. row0 + RL - 1). `valid` lanes only; every lane of the warp must call it (warp votes).
template <int MP, int RL>
__device__ __forceinline__ void ql_rows(double (&dg)[MP], double (&eo)[MP], double (&z)[RL][MP], bool valid) {
#pragma unroll
    for (int l = 0; l < MP - 1; ++l) {
        for (int iter = 0; iter < 40; ++iter) {
            int mm = MP - 1;
#pragma unroll
            for (int k = MP - 2; k >= l; --k) {
                const double dd = fabs(dg[k]) + fabs(dg[k + 1]);
                if (fabs(eo[k]) <= DBL_EPSILON * dd) mm = k;
            }
            const bool go = valid && mm != l;
            if (!__any_sync(0xffffffffu, go)) break;
            if (go) {
                double g = (dg[l + 1] - dg[l]) * (0.5 * frcp(eo[l]));
                const double t1 = fma(g, g, 1.0);
                double rr = t1 * frsqrt(t1);
                double dm = dg[MP - 1];
#pragma unroll
                for (int k = l + 1; k < MP - 1; ++k)
                    if (k == mm) dm = dg[k];
                g = dm - dg[l] + eo[l] * frcp(g + (g >= 0.0 ? rr : -rr));
                double s = 1.0, c = 1.0, p = 0.0;
                bool brk = false;
#pragma unroll
                for (int i = MP - 2; i >= l; --i) {
                    if (i < mm && !brk) {
                        const double f = s * eo[i], b = c * eo[i];
                        const double t2 = f * f + g * g;
                        const double inv = frsqrt(t2);
                        rr = t2 == 0.0 ? 0.0 : t2 * inv;
                        eo[i + 1] = rr;
                        if (t2 == 0.0) {
                            dg[i + 1] -= p;
#pragma unroll
                            for (int k = l; k < MP; ++k)
                                if (k == mm) eo[k] = 0.0;
                            brk = true;
                        } else {
                            s = f * inv;
                            c = g * inv;
                            g = dg[i + 1] - p;
                            rr = (dg[i] - g) * s + 2.0 * c * b;
                            p = s * rr;
                            dg[i + 1] = g + p;
                            g = c * rr - b;
#pragma unroll
                            for (int q = 0; q < RL; ++q) {
                                const double zf = z[q][i + 1];
                                z[q][i + 1] = s * z[q][i] + c * zf;
                                z[q][i] = c * z[q][i] - s * zf;
                            }
                        }
                    }
                }
                if (!brk) {
                    dg[l] -= p;
                    eo[l] = g;
#pragma unroll
                    for (int k = l + 1; k < MP; ++k)
                        if (k == mm) eo[k] = 0.0;
                }
            }
        }
    }
}

// shared-memory layout of one slice (all offsets in bytes, 16-byte aligned)
struct SliceLayout {
    int U, MP, L, n, J, tsz;  // tsz = sizeof(complex T)
    int a_off, z_off, u_off, lam_off, tau_off, v_off, tri_off, bytes;
    __host__ __device__ void init(int U_, int MP_, int L_, int n_, int J_, int tsz_) {
        U = U_; MP = MP_; L = L_; n = n_; J = J_; tsz = tsz_;
        int o = 0;
        a_off = o; o += U * MP * (MP + 1) * 16;            // A / Householder vectors / Cholesky factor
        z_off = o; o += U * MP * (MP + 1) * 8;             // Z rows (QL), then Y (m x L, T)
        const int ysz = U * MP * L * tsz;
        if (ysz > U * MP * (MP + 1) * 8) o = z_off + ((ysz + 15) & ~15);
        u_off = o; o += U * L * MP * 16;                   // eigenvectors of the kept streams
        lam_off = o; o += U * MP * 8;                      // eigenvalues by rank
        tau_off = o; o += U * MP * 16;                     // Householder scalars
        v_off = o; o += J * n * L * tsz;                   // anchor precoders V'_k [k][y][l]
        o = (o + 15) & ~15;
        tri_off = o;
        o += U * 2 * MP * 8;                               // tridiagonal (d, e) -> eigenvalues (packed QL phase)
        bytes = (o + 15) & ~15;
    }
};

}  // namespace

// PGM = false: H~ in HBM ([g][f][link][n][m]); the serving Gram and the interference products are formed
// here. PGM = true: the serving / pair Grams come precomputed in PG[item][user][J][m*m] (k_rgram.cu); the
// interference of cell k is Y = X_{u,k} W'_k with W'_k = U'_L Lambda'^{-1/2} of the anchor (k,0)
// (= H~_kij V'_k, the same product through the anchor's Gram eigenpairs), all in binary64.
template <class T, int MP, bool PGM, bool QLP>
__global__ void __launch_bounds__(256, 2) k_sinr_users(Topo t, int spc, int64_t nslices, int fc, int64_t Ftot,
                                                    int64_t f0, double sigma, const cplx_t<T>* __restrict__ H,
                                                    const double2* __restrict__ PG, double* __restrict__ sinr,
                                                    double* __restrict__ signal, int* __restrict__ status) {
    using C = typename std::conditional<PGM, double2, cplx_t<T>>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int U = t.users(), L = t.L, m = t.m, n = PGM ? MP : t.n, J = t.J, K = t.K, links = t.links();
    SliceLayout lay;
    lay.init(U, MP, L, n, J, (int)sizeof(C));
    const int tid = threadIdx.x, lane = tid & 31;
    const int r = tid % MP;                       // my row
    const int ug = tid / MP;                      // user slot in the CTA
    const int sl_local = ug / U, u = ug % U;
    const int64_t sl = (int64_t)blockIdx.x * spc + sl_local;
    const bool active = sl_local < spc && sl < nslices;
    const int64_t sl_c = active ? sl : 0;
    unsigned char* sbase = smem_raw + (size_t)sl_local * lay.bytes;  // threads past spc*U*MP own scratch slices
    double2* sA = reinterpret_cast<double2*>(sbase + lay.a_off) + u * MP * (MP + 1);
    double* sZ = reinterpret_cast<double*>(sbase + lay.z_off) + u * MP * (MP + 1);
    C* sY = reinterpret_cast<C*>(sbase + lay.z_off) + u * MP * L;
    double2* sU = reinterpret_cast<double2*>(sbase + lay.u_off);
    double* slam = reinterpret_cast<double*>(sbase + lay.lam_off);
    double2* stau = reinterpret_cast<double2*>(sbase + lay.tau_off) + u * MP;
    C* sV = reinterpret_cast<C*>(sbase + lay.v_off);
    const int i_cell = u / K, j_user = u % K;
    const int MM = m * m;
    // pair Grams of this (slice, user): slot 0 serving, then cells k != i ascending
    const double2* Pu = PG + (sl_c * U + u) * (int64_t)J * MM;
    if constexpr (PGM) {
        // ---------------- phase 1a (PG): serving Gram row r
#pragma unroll
        for (int c = 0; c < MP; ++c) {
            double2 a = (active && r < m && c < m) ? Pu[r + m * c] : make_double2(0.0, 0.0);
            if (c == r) a.y = 0.0;
            sA[r * (MP + 1) + c] = a;
        }
        __syncwarp();
    } else {
    // H~ of this slice: item (g, f-in-chunk) = sl, links contiguous
    const cplx_t<T>* Hs = H + (sl_c * links + (int64_t)(i_cell * J + i_cell) * K + j_user) * (int64_t)m * t.n;

    // ---------------- phase 1a: serving Gram (binary64), balanced cyclic entries per lane
    constexpr int ND = MP / 2 + 1;
    double2 acc[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) acc[d] = make_double2(0.0, 0.0);
    if (active) {
#pragma unroll 4
        for (int y = 0; y < t.n; ++y) {
            // the column is m contiguous entries shared by the user's lanes (L1 broadcast)
            const cplx_t<T>* col = Hs + (int64_t)y * m;
            const double2 hr = r < m ? to_d2(col[r]) : make_double2(0.0, 0.0);
#pragma unroll
            for (int d = 0; d < ND; ++d) {
                const int c = (r + d) & (MP - 1);
                const double2 hc = c < m ? to_d2(col[c]) : make_double2(0.0, 0.0);
                cfmac(acc[d], hr, hc);
            }
        }
    }
#pragma unroll
    for (int d = 0; d < ND; ++d) {
        const int c = (r + d) & (MP - 1);
        if (d < MP / 2 || r < MP / 2) {
            double2 v = acc[d];
            if (d == 0) v.y = 0.0;
            sA[r * (MP + 1) + c] = v;
            sA[c * (MP + 1) + r] = make_double2(v.x, -v.y);
        }
    }
    __syncwarp();
    }
    // keep my row of A when the serving term of Q is A itself (L == m)
    // (PG mode re-reads it from PG in phase 3 instead of keeping it live through the eig)
    double2 arow[PGM ? 1 : MP];
    if constexpr (!PGM) {
#pragma unroll
        for (int c = 0; c < MP; ++c) arow[c] = sA[r * (MP + 1) + c];
    }

    // ---------------- phase 1b: Householder tridiagonalisation (zhetd2, lower), lane r owns row r
    double dg[MP], eo[MP];  // tridiagonal (replicated in every lane of the user)
#pragma unroll
    for (int i = 0; i < MP - 1; ++i) {
        // column i below the diagonal: alpha = A[i+1][i], x = A[i+2..][i]
        const double2 alpha = sA[(i + 1) * (MP + 1) + i];
        const double2 xr = (r > i + 1) ? sA[r * (MP + 1) + i] : make_double2(0.0, 0.0);
        const double xn2 = seg_sum<MP>(xr.x * xr.x + xr.y * xr.y);
        double2 tau = make_double2(0.0, 0.0);
        double beta = alpha.x;
        double2 v = make_double2(r == i + 1 ? 1.0 : 0.0, 0.0);
        if (xn2 > 0.0 || alpha.y != 0.0) {
            // branch-free reciprocals / square roots (MUFU seed + Newton, ~1 ulp): the division and sqrt sequences
            // of libdevice sit on the serial chain of every reflector
            const double s2n = fmax(alpha.x * alpha.x + alpha.y * alpha.y + xn2, 1e-280);
            const double nrm = s2n * frsqrt(s2n);
            beta = alpha.x >= 0.0 ? -nrm : nrm;
            const double rb = frcp(beta);
            tau = make_double2((beta - alpha.x) * rb, -alpha.y * rb);
            // scale = 1 / (alpha - beta)
            const double2 am = make_double2(alpha.x - beta, alpha.y);
            const double den = frcp(am.x * am.x + am.y * am.y);
            const double2 sc = make_double2(am.x * den, -am.y * den);
            if (r > i + 1) v = dmul(xr, sc);
        }
        dg[i] = sA[i * (MP + 1) + i].x;
        eo[i] = beta;
        // store v in the column (rows > i+1) for the back-transform, tau aside
        if (r > i + 1) sA[r * (MP + 1) + i] = v;
        if (r == 0) stau[i] = tau;
        __syncwarp();
        if (tau.x != 0.0 || tau.y != 0.0) {
            // p = tau * A22 v   (rows > i)
            double2 pr = make_double2(0.0, 0.0);
            if (r > i) {
#pragma unroll
                for (int c = i + 1; c < MP; ++c) {
                    const double2 vc = (c == i + 1) ? make_double2(1.0, 0.0) : sA[c * (MP + 1) + i];
                    cfma(pr, sA[r * (MP + 1) + c], vc);
                }
                pr = dmul(tau, pr);
            }
            // K = -1/2 tau (p^H v)
            const double2 pv = make_double2(pr.x * v.x + pr.y * v.y, pr.x * v.y - pr.y * v.x);  // conj(p) v
            const double2 s = make_double2(seg_sum<MP>(pv.x), seg_sum<MP>(pv.y));
            const double2 kk = dmul(make_double2(-0.5 * tau.x, -0.5 * tau.y), s);
            double2 w = pr;
            cfma(w, kk, v);
            // broadcast v and w of rows > i through the (no longer needed) Z scratch
            double* sw = sZ;  // [MP] double2 for w, then v
            __syncwarp();
            reinterpret_cast<double2*>(sw)[r] = w;
            reinterpret_cast<double2*>(sw)[MP + r] = v;
            __syncwarp();
            if (r > i) {
#pragma unroll
                for (int c = i + 1; c < MP; ++c) {
                    const double2 wc = reinterpret_cast<double2*>(sw)[c];
                    const double2 vc = reinterpret_cast<double2*>(sw)[MP + c];
                    double2 a = sA[r * (MP + 1) + c];
                    // A -= v w^H + w v^H
                    a.x -= v.x * wc.x + v.y * wc.y + w.x * vc.x + w.y * vc.y;
                    a.y -= v.y * wc.x - v.x * wc.y + w.y * vc.x - w.x * vc.y;
                    sA[r * (MP + 1) + c] = a;
                }
            }
        }
        __syncwarp();
    }
    dg[MP - 1] = sA[(MP - 1) * (MP + 1) + MP - 1].x;
    eo[MP - 1] = 0.0;
    // the last step (i = MP-2) may leave a complex phase only through tau (|1 - tau| = 1): e is real.

    // ---------------- phase 1c: implicit QL (tql2) on (dg, eo).
    // QLP = true (packed, default): GWT_QL_LANES = 4 lanes per user, each rotating MP / 4 rows of Z, on the first
    // 4 U spc threads of the CTA behind two CTA barriers. QLP = false (warp-local): the recurrence replicated over the
    // user's MP lanes, lane r rotating row r of Z; no CTA barrier, but twice the binary64 warp instructions (fp64 pipe
    // 42 % busy). A warp advances its users in lockstep (every user of the warp converges on eigenvalue l before l + 1),
    // so fewer users per warp shorten the phase while more lanes per user replicate the recurrence. Measured per 64
    // groups (C4 / C3 solve): 1 lane 51.6 / 10.5 ms, 2 lanes 35.8 / -, 4 lanes 33.6 / 7.5, warp-local - / 7.6
    // (C4 warp-local against 2 packed lanes, before the fast reciprocals: 45.3 vs 42.6 ms, and 398 vs 337 ms on the
    // whole 512-group config).
    // GWT_QL_PACKED=0 selects the warp-local form.
    if constexpr (QLP) {
        double* stri = reinterpret_cast<double*>(sbase + lay.tri_off) + u * 2 * MP;
        if (r == 0) {
#pragma unroll
            for (int k = 0; k < MP; ++k) {
                stri[k] = dg[k];
                stri[MP + k] = eo[k];
            }
        }
        __syncthreads();
        constexpr int LQ = GWT_QL_LANES, RL = MP / LQ;
        const int nql = spc * U * LQ;
        if (tid < ((nql + 31) & ~31)) {
            const bool qv = tid < nql;
            const int qi = qv ? tid : 0;
            const int qs = qi / (U * LQ), qu = (qi / LQ) % U, qh = qi % LQ;
            unsigned char* qb = smem_raw + (size_t)qs * lay.bytes;
            double* qt = reinterpret_cast<double*>(qb + lay.tri_off) + qu * 2 * MP;
            double d[MP], e[MP];
#pragma unroll
            for (int k = 0; k < MP; ++k) {
                d[k] = qt[k];
                e[k] = qt[MP + k];
            }
            double zq[RL][MP];
#pragma unroll
            for (int q = 0; q < RL; ++q)
#pragma unroll
                for (int c = 0; c < MP; ++c) zq[q][c] = c == qh * RL + q ? 1.0 : 0.0;
            ql_rows<MP, RL>(d, e, zq, qv);
            __syncwarp();
            if (qv) {
                double* zs = reinterpret_cast<double*>(qb + lay.z_off) + qu * MP * (MP + 1);
#pragma unroll
                for (int q = 0; q < RL; ++q)
#pragma unroll
                    for (int c = 0; c < MP; ++c) zs[(qh * RL + q) * (MP + 1) + c] = zq[q][c];
                if (qh == 0)
#pragma unroll
                    for (int k = 0; k < MP; ++k) qt[k] = d[k];
            }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < MP; ++k) dg[k] = stri[k];
    } else {
        double zr[1][MP];
#pragma unroll
        for (int c = 0; c < MP; ++c) zr[0][c] = c == r ? 1.0 : 0.0;
        ql_rows<MP, 1>(dg, eo, zr, active);
        __syncwarp();
#pragma unroll
        for (int c = 0; c < MP; ++c) sZ[r * (MP + 1) + c] = zr[0][c];
        __syncwarp();
    }
    // ---------------- phase 1d: back-transform, lane j = eigenvector j: u = H_0 ... H_{MP-2} z_j
    double2 uv[MP];
#pragma unroll
    for (int a = 0; a < MP; ++a) uv[a] = make_double2(sZ[a * (MP + 1) + r], 0.0);
#pragma unroll
    for (int i = MP - 2; i >= 0; --i) {
        const double2 tau = stau[i];
        if (tau.x != 0.0 || tau.y != 0.0) {
            // s = v^H u ; u -= tau v s
            double2 s = uv[i + 1];
#pragma unroll
            for (int a = i + 2; a < MP; ++a) cfmaconj(s, sA[a * (MP + 1) + i], uv[a]);
            const double2 ts = dmul(tau, s);
            uv[i + 1].x -= ts.x;
            uv[i + 1].y -= ts.y;
#pragma unroll
            for (int a = i + 2; a < MP; ++a) {
                const double2 va = sA[a * (MP + 1) + i];
                uv[a].x -= va.x * ts.x - va.y * ts.y;
                uv[a].y -= va.x * ts.y + va.y * ts.x;
            }
        }
    }
    // PG mode: the pair Gram of the first interfering cell is copied asynchronously into the user's (now free)
    // Householder area, entry (row, b) at b (MP + 1) + row, so its global-memory latency passes behind the ranking,
    // the CTA barriers and the anchor precoders without holding registers (at its use in phase 3 the plain loads
    // were 14 % of the kernel's stall samples)
    if constexpr (PGM) {
        __syncwarp();  // every lane of the user is done with the Householder vectors
        if (J > 1 && active && r < m) {
#pragma unroll
            for (int b = 0; b < MP; ++b)
                if (b < m) {
                    const unsigned dst = (unsigned)__cvta_generic_to_shared(sA + b * (MP + 1) + r);
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(Pu + MM + r + m * b) : "memory");
                }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    // rank (descending, lower index first on ties) over the real rows; keep the top L
    {
        const double lam = dg[0];
        double lj = dg[0];
#pragma unroll
        for (int k = 1; k < MP; ++k)
            if (k == r) lj = dg[k];
        int rank = 0;
#pragma unroll
        for (int k = 0; k < MP; ++k) rank += (dg[k] > lj || (dg[k] == lj && k < r)) ? 1 : 0;
        (void)lam;
        __syncwarp();
        if (rank < L) {
            slam[u * MP + rank] = fmax(lj, 0.0);
#pragma unroll
            for (int a = 0; a < MP; ++a) sU[(u * L + rank) * MP + a] = uv[a];
            if constexpr (PGM) {
                // the anchor (k, 0) publishes W'_k = U'_L Lambda'^{-1/2} (m x L) itself: no separate phase, one CTA
                // barrier less
                if (j_user == 0) {
                    const double sc = lj > 0.0 ? frsqrt(fmax(lj, 1e-300)) : 0.0;
#pragma unroll
                    for (int a = 0; a < MP; ++a) sV[(i_cell * MP + a) * L + rank] = make_double2(uv[a].x * sc, uv[a].y * sc);
                }
            }
        }
    }
    __syncthreads();

    // ---------------- phase 2 (H~ mode): anchor precoders V'_k = H~_kk0^H U'_L L'^-1/2 (all threads of the CTA);
    // PG mode uses W'_k = U'_L L'^-1/2 (m x L), written by the anchors' own lanes above
    if constexpr (!PGM) {
        const int per = J * n;
        for (int e = tid; e < spc * per; e += blockDim.x) {
            const int s2 = e / per, rem = e % per, k = rem / n, y = rem % n;
            const int64_t sl2 = (int64_t)blockIdx.x * spc + s2;
            if (sl2 >= nslices) continue;
            unsigned char* sb2 = smem_raw + (size_t)s2 * lay.bytes;
            const double2* U2 = reinterpret_cast<const double2*>(sb2 + lay.u_off) + (k * K) * L * MP;
            const double* l2 = reinterpret_cast<const double*>(sb2 + lay.lam_off) + (k * K) * MP;
            C* V2 = reinterpret_cast<C*>(sb2 + lay.v_off) + (k * n + y) * L;
            const cplx_t<T>* col = H + (sl2 * links + (int64_t)(k * J + k) * K) * (int64_t)m * t.n + (int64_t)y * m;
            double2 h[MP];
#pragma unroll
            for (int a = 0; a < MP; ++a) h[a] = a < m ? to_d2(col[a]) : make_double2(0.0, 0.0);
            for (int l = 0; l < L; ++l) {
                const double lam = l2[l];
                double2 s = make_double2(0.0, 0.0);
#pragma unroll
                for (int a = 0; a < MP; ++a) cfmaconj(s, h[a], U2[l * MP + a]);
                const double sc = lam > 0.0 ? frsqrt(fmax(lam, 1e-300)) : 0.0;
                V2[l] = from_d2<C>(make_double2(s.x * sc, s.y * sc));
            }
        }
        __syncthreads();
    }

    // ---------------- phase 3: covariance, Cholesky, per-stream SINR
    int st = 0;
    const double s2 = sigma * sigma;
    double2 q[MP];
    if (L == m) {
#pragma unroll
        for (int c = 0; c < MP; ++c) {
            if constexpr (PGM) {
                double2 a = (active && r < m && c < m) ? Pu[r + m * c] : make_double2(0.0, 0.0);
                if (c == r) a.y = 0.0;
                q[c] = a;
            } else {
                q[c] = arow[c];
            }
        }
    } else {
#pragma unroll
        for (int c = 0; c < MP; ++c) q[c] = make_double2(0.0, 0.0);
        for (int rk = 0; rk < L; ++rk) {
            const double lr = slam[u * MP + rk];
            const double2* ur = sU + (u * L + rk) * MP;
            const double2 ua = ur[r];
#pragma unroll
            for (int c = 0; c < MP; ++c) {
                double2 v = make_double2(0.0, 0.0);
                cfmac(v, ua, ur[c]);
                q[c].x += lr * v.x;
                q[c].y += lr * v.y;
            }
        }
    }
    q[0].x += (r == 0) ? s2 : 0.0;
#pragma unroll
    for (int c = 1; c < MP; ++c)
        if (c == r) q[c].x += s2;
    // interference of every other cell's scope user (k, 0): Y = H~_kij V'_k
    for (int k = 0; k < J; ++k) {
        if (k == i_cell) continue;
        const double* lk = slam + (k * K) * MP;
        for (int l = 0; l < L; ++l)
            if (!(lk[l] > 0.0)) st = st ? st : 5;
        const C* Vk = sV + (size_t)k * n * L;
        C yrow[MP];  // my row of Y (L <= MP entries)
#pragma unroll
        for (int l = 0; l < MP; ++l) yrow[l] = czero<C>();
        if constexpr (PGM) {
            const int slot = 1 + (k < i_cell ? k : k - 1);
            const double2* Xg = Pu + (int64_t)slot * MM;  // slot of cell k
            if (slot == 1) {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
                __syncwarp();
            }
            if (active && r < m) {
#pragma unroll
                for (int b = 0; b < MP; ++b) {
                    if (b < m) {
                        const double2 xv = slot == 1 ? sA[b * (MP + 1) + r] : Xg[r + m * b];
                        const double2* wb = Vk + (size_t)b * L;
#pragma unroll
                        for (int l = 0; l < MP; ++l)
                            if (l < L) cfma(yrow[l], xv, wb[l]);
                    }
                }
            }
        } else {
        const cplx_t<T>* Hx = H + (sl_c * links + (int64_t)(k * J + i_cell) * K + j_user) * (int64_t)m * t.n;
        if (active && r < m) {
#pragma unroll 2
            for (int y = 0; y < t.n; ++y) {
                const C hv = Hx[(int64_t)y * m + r];
                const C* vr = Vk + (size_t)y * L;
                if (sizeof(C) == 8 && L == MP) {  // 16-byte broadcast loads of V'_k[y][:]
#pragma unroll
                    for (int l = 0; l < MP; l += 2) {
                        const float4 v4 = *reinterpret_cast<const float4*>(vr + l);
                        cfma(yrow[l], hv, mk((decltype(hv.x))v4.x, (decltype(hv.x))v4.y));
                        cfma(yrow[l + 1], hv, mk((decltype(hv.x))v4.z, (decltype(hv.x))v4.w));
                    }
                } else {
#pragma unroll
                    for (int l = 0; l < MP; ++l)
                        if (l < L) cfma(yrow[l], hv, vr[l]);
                }
            }
        }
        }
        __syncwarp();
#pragma unroll
        for (int l = 0; l < MP; ++l)
            if (l < L) sY[r * L + l] = yrow[l];
        __syncwarp();
        // Q[r][c] += sum_l Y[r][l] conj(Y[c][l])
#pragma unroll
        for (int c = 0; c < MP; ++c) {
#pragma unroll
            for (int l = 0; l < MP; ++l)
                if (l < L) cfmac(q[c], to_d2(yrow[l]), to_d2(sY[c * L + l]));
        }
        __syncwarp();
    }
    // non-finite check (check_finite(q, "woodbury_inverse_apply"))
    bool fin = true;
#pragma unroll
    for (int c = 0; c < MP; ++c) fin = fin && isfinite(q[c].x) && isfinite(q[c].y);
    const bool finite = __all_sync(seg_mask<MP>(lane), fin);
    // right-looking Cholesky (Eigen::LLT: d_k = Q_kk - sum |L_kj|^2 > 0), lane = row; columns of L
    // published through shared memory (the A region is free now)
    double2* sLf = sA;  // [row][col], stride MP+1
    bool pd = finite;
    double dmax = 0.0, dmin = 1e308;
#pragma unroll
    for (int kc = 0; kc < MP; ++kc) {
        if (kc < m) {
            const double dkk = __shfl_sync(0xffffffffu, q[kc].x, (lane & ~(MP - 1)) + kc);
            pd = pd && (dkk > 0.0);
            const double dk = fmax(dkk, 1e-300);
            const double rl = frsqrt(dk), lkk = dk * rl;  // 1 / L_kk rides in the (otherwise zero) imaginary slot
            dmax = fmax(dmax, lkk);
            dmin = fmin(dmin, lkk);
            double2 lrk;
            if (r == kc) lrk = make_double2(lkk, rl);
            else lrk = make_double2(q[kc].x * rl, q[kc].y * rl);
            if (r >= kc) sLf[r * (MP + 1) + kc] = lrk;
            __syncwarp();
            if (r > kc && r < m) {
#pragma unroll
                for (int c = kc + 1; c < MP; ++c) {
                    if (c <= r) {  // Q[r][c] -= L[r][kc] conj(L[c][kc])
                        const double2 lc = sLf[c * (MP + 1) + kc];
                        q[c].x -= lrk.x * lc.x + lrk.y * lc.y;
                        q[c].y -= lrk.y * lc.x - lrk.x * lc.y;
                    }
                }
            }
            __syncwarp();
        }
    }
    if (!finite) st = 4;
    else if (!pd) st = 1;
    else if (dmax * dmax > 1e14 * (dmin * dmin)) st = 2;  // (dmax / dmin)^2 > 1e14 without the divisions
    int64_t g, fl;
    if (sl_c < (int64_t(1) << 31)) {  // 32-bit division when the slice index allows it
        g = (uint32_t)sl_c / (uint32_t)fc;
        fl = (uint32_t)sl_c % (uint32_t)fc;
    } else {
        g = sl_c / fc;
        fl = sl_c % fc;
    }
    const int64_t orow = (g * Ftot + f0 + fl) * U + u;
    int st3 = 0;
    if (active && r < L) {
        double gamma = 0.0;
        const double lr = slam[u * MP + r];
        if (st != 1 && st != 2 && st != 4) {
            const double2* ur = sU + (u * L + r) * MP;
            double2 yv[MP];
            double nn = 0.0;
#pragma unroll
            for (int a = 0; a < MP; ++a) {
                if (a < m) {
                    double2 acc2 = ur[a];
#pragma unroll
                    for (int k2 = 0; k2 < a; ++k2) {
                        double2 pr = make_double2(0.0, 0.0);
                        cfma(pr, sLf[a * (MP + 1) + k2], yv[k2]);
                        acc2.x -= pr.x;
                        acc2.y -= pr.y;
                    }
                    const double rla = sLf[a * (MP + 1) + a].y;  // 1 / L_aa
                    yv[a] = make_double2(acc2.x * rla, acc2.y * rla);
                    nn += yv[a].x * yv[a].x + yv[a].y * yv[a].y;
                } else {
                    yv[a] = make_double2(0.0, 0.0);
                }
            }
            gamma = lr * nn;
        }
        const double sp = gamma * gamma;
        double den = gamma * (1.0 - gamma);
        if (den <= -1e-12 && st == 0) st3 = 3;
        den = fmax(den, 2.2250738585072014e-308);
        sinr[orow * L + r] = sp * frcp(den);
        signal[orow * L + r] = sp;
    }
    // code 3 carries the first failing stream (the user's lowest lane) in bits 8+
    const unsigned m3 = (__ballot_sync(0xffffffffu, st3 == 3) & seg_mask<MP>(lane)) >> (lane & ~(MP - 1));
    if (active && r == 0) status[orow] = (st == 0 && m3) ? 3 + ((__ffs(m3) - 1) << 8) : st;
}

bool sinr_users_fits(const Topo& t, size_t csize) {
    const int MP = t.m <= 4 ? 4 : 8;
    if (t.m > 8 || t.L > t.m || t.users() * MP > 256) return false;
    SliceLayout lay;
    lay.init(t.users(), MP, t.L, t.n, t.J, (int)csize);
    return lay.bytes <= 200 * 1024;
}

template <class T, int MP, bool PGM, bool QLP>
static cudaError_t launch_users_qlp(const Topo& t, int64_t nslices, int fc, int64_t Ftot, int64_t f0, double sigma,
                                   const void* H, const double2* PG, double* sinr, double* signal, int* status,
                                   cudaStream_t st) {
    SliceLayout lay;
    lay.init(t.users(), MP, t.L, PGM ? MP : t.n, t.J, PGM ? 16 : (int)sizeof(cplx_t<T>));
    const int per = t.users() * MP;
    int spc = std::max(1, 256 / per);
    while (spc > 1 && (size_t)(spc + 1) * lay.bytes > 200 * 1024) --spc;
    const int threads = ((spc * per + 31) / 32) * 32;
    const size_t smem = (size_t)((threads + per - 1) / per) * lay.bytes;
    cudaError_t e =
        cudaFuncSetAttribute(k_sinr_users<T, MP, PGM, QLP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t blocks = (nslices + spc - 1) / spc;
    k_sinr_users<T, MP, PGM, QLP><<<(unsigned)blocks, threads, smem, st>>>(t, spc, nslices, fc, Ftot, f0, sigma,
                                                                           (const cplx_t<T>*)H, PG, sinr, signal, status);
    return cudaGetLastError();
}

template <class T, int MP, bool PGM>
static cudaError_t launch_users_mp(const Topo& t, int64_t nslices, int fc, int64_t Ftot, int64_t f0, double sigma,
                                   const void* H, const double2* PG, double* sinr, double* signal, int* status,
                                   cudaStream_t st) {
    if constexpr (PGM && MP == 8) {
        static const int force = [] {
            const char* v = env_once("GWT_QL_PACKED");
            return v ? std::atoi(v) : -1;
        }();
        const bool packed = force != 0;  // see phase 1c
        if (packed) return launch_users_qlp<T, MP, PGM, true>(t, nslices, fc, Ftot, f0, sigma, H, PG, sinr, signal, status, st);
    }
    return launch_users_qlp<T, MP, PGM, false>(t, nslices, fc, Ftot, f0, sigma, H, PG, sinr, signal, status, st);
}

template <class T>
cudaError_t launch_sinr_users(const Topo& t, int64_t nslices, int fc, int64_t Ftot, int64_t f0, double sigma,
                              const void* H, double* sinr, double* signal, int* status, cudaStream_t st) {
    if (!sinr_users_fits(t, sizeof(cplx_t<T>))) return cudaErrorNotSupported;
    return t.m <= 4 ? launch_users_mp<T, 4, false>(t, nslices, fc, Ftot, f0, sigma, H, nullptr, sinr, signal, status, st)
                    : launch_users_mp<T, 8, false>(t, nslices, fc, Ftot, f0, sigma, H, nullptr, sinr, signal, status, st);
}

bool sinr_users_pg_fits(const Topo& t) {
    const int MP = t.m <= 4 ? 4 : 8;
    if (t.m > 8 || t.L > t.m || t.users() * MP > 256) return false;
    SliceLayout lay;
    lay.init(t.users(), MP, t.L, MP, t.J, 16);
    return lay.bytes <= 200 * 1024;
}

cudaError_t launch_sinr_users_pg(const Topo& t, int64_t nslices, int fc, int64_t Ftot, int64_t f0, double sigma,
                                 const double2* PG, double* sinr, double* signal, int* status, cudaStream_t st) {
    if (!sinr_users_pg_fits(t)) return cudaErrorNotSupported;
    return t.m <= 4 ? launch_users_mp<double, 4, true>(t, nslices, fc, Ftot, f0, sigma, nullptr, PG, sinr, signal, status, st)
                    : launch_users_mp<double, 8, true>(t, nslices, fc, Ftot, f0, sigma, nullptr, PG, sinr, signal, status, st);
}

template cudaError_t launch_sinr_users<float>(const Topo&, int64_t, int, int64_t, int64_t, double, const void*, double*,
                                              double*, int*, cudaStream_t);
template cudaError_t launch_sinr_users<double>(const Topo&, int64_t, int, int64_t, int64_t, double, const void*,
                                               double*, double*, int*, cudaStream_t);

}  // namespace gwtk
