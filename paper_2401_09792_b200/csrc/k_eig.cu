// Batched Hermitian eigensolver for the Tucker factor updates, sm_100a.
//
// Reference: leading_eigenvectors (proj/src/linalg.cpp:27-45) -> Eigen
// SelfAdjointEigenSolver (Householder tridiagonalisation + implicit QR),
// reversed to descending order, then phase_normalize_columns (:11-25).
//
// B200 mapping: one CTA (256 threads) per matrix, binary64 throughout (the Gram
// may be c64; its eigenvectors are computed in fp64 and rounded once).
//  1. Householder reduction to Hermitian tridiagonal: each step is a CTA-wide
//     block reduction + a coalesced Hermitian mat-vec + a rank-2 update of the
//     trailing block; the matrix lives in shared memory when n <= 64, else in a
//     global workspace (L1/L2 resident).
//  2. Diagonal phase similarity to a real symmetric tridiagonal T.
//  3. Only the wanted top-`count` eigenpairs of T: one thread per eigenvalue,
//     bisection on Sturm counts, then inverse iteration with a partially pivoted
//     tridiagonal LU (LAPACK dgtsv-style elimination); eigenvalues closer than
//     1e-3 ||T|| form clusters whose vectors are orthogonalised (modified
//     Gram-Schmidt) inside the iteration, one cluster member per round.
//  4. Back-transform through the stored reflectors, phase normalisation
//     (largest-|.| entry real >= 0, lowest index on ties).
#include <cstdlib>
#include <cstring>

#include "kernels.cuh"
#include "small_linalg.cuh"

namespace gwtk {

constexpr int kEigThreads = 256;
#ifdef GWT_PHASE_TIMERS
__device__ long long g_eig_phase[8];
#define GWT_CLK(v) const long long v = clock64()
#define GWT_TICK(v) v = clock64()
#else
#define GWT_CLK(v)
#define GWT_TICK(v)
#endif
constexpr int kSmemMaxD = 64;

__device__ __forceinline__ double block_sum(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x < 32) {
        s = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) red[32] = s;
    }
    __syncthreads();
    return red[32];
}

// number of eigenvalues of T (d, e2 = e^2) strictly below x
__device__ __forceinline__ int sturm_count(int D, const double* d, const double* e2, double x, double pivmin) {
    int cnt = 0;
    double q = d[0] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
    for (int i = 1; i < D; ++i) {
        q = d[i] - x - e2[i - 1] / q;
        if (fabs(q) < pivmin) q = -pivmin;
        cnt += q < 0.0;
    }
    return cnt;
}

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// fast binary64 reciprocal for Sturm counts (only signs matter; one Newton step on a fp32 seed)
__device__ __forceinline__ double fast_rcp(double q) {
    const double a = fabs(q);
    if (a > 1e-30 && a < 1e30) {
        const double r0 = (double)__frcp_rn((float)q);
        return r0 * (2.0 - q * r0);
    }
    return 1.0 / q;
}

__device__ __forceinline__ int sturm_count_fast(int D, const double* d, const double* e2, double x, double pivmin) {
    int cnt = 0;
    double q = d[0] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
    for (int i = 1; i < D; ++i) {
        q = d[i] - x - e2[i - 1] * fast_rcp(q);
        if (fabs(q) < pivmin) q = -pivmin;
        cnt += q < 0.0;
    }
    return cnt;
}

// fp32 Sturm count on a scaled tridiagonal: bisection only has to deliver an inverse-iteration
// shift (~1e-7 relative); the reported eigenvalue is the binary64 Rayleigh quotient.
// Division-free form: the count of sign changes of the leading-minor sequence
// p_i = (d_i - x) p_{i-1} - e_{i-1}^2 p_{i-2} (p_0 = 1) equals the count of negative pivots
// q_i = p_i / p_{i-1}, so the serial chain is one FFMA per row (the e^2 p_{i-2} product is off the
// chain) instead of a reciprocal + multiply + add; the pair (p_{i-1}, p_i) is rescaled by a power
// of two every 8 rows (|d - x| <= 2 on the normalised T keeps 8 rows far from overflow). An exact
// zero p_i (+0) counts like the q = -pivmin convention: the sign change moves to the next row.
// Used for the fp32-storage (c64) solvers; the c128 solvers keep the pivot recurrence below, whose
// count is monotone in x (Kahan), so their fp32 shifts resolve small eigenvalues reproducibly.
__device__ __forceinline__ int sturm_count_p32(int D, const float* d, const float* e2s, float x) {
    // e2s is the SHIFTED squared off-diagonal (e2s[0] = 0, e2s[i] = e_{i-1}^2, written so by the fp32
    // callers) and d, e2s are 16-byte aligned: p_{i+1} = (d_i - x) p_i - e2s[i] p_{i-1}, p_0 = 1,
    // p_{-1} = 0; blocks of 8 rows read both arrays with 16-byte loads
    float pm = 0.0f, p = 1.0f;
    int cnt = 0;
    int i = 0;
    for (; i + 8 <= D; i += 8) {
        const float4 da = *reinterpret_cast<const float4*>(d + i), db = *reinterpret_cast<const float4*>(d + i + 4);
        const float4 ea = *reinterpret_cast<const float4*>(e2s + i), eb = *reinterpret_cast<const float4*>(e2s + i + 4);
        const float dv[8] = {da.x, da.y, da.z, da.w, db.x, db.y, db.z, db.w};
        const float ev[8] = {ea.x, ea.y, ea.z, ea.w, eb.x, eb.y, eb.z, eb.w};
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float pn = fmaf(dv[u] - x, p, -ev[u] * pm);
            cnt += (int)((__float_as_uint(pn) ^ __float_as_uint(p)) >> 31);
            pm = p;
            p = pn;
        }
        const float mx = fmaxf(fabsf(p), fabsf(pm));
        const float sc = __int_as_float(0x7f000000 - (__float_as_int(mx) & 0x7f800000));  // ~1/mx, power of 2
        p *= sc;
        pm *= sc;
    }
    for (; i < D; ++i) {
        const float pn = fmaf(d[i] - x, p, -e2s[i] * pm);
        cnt += (int)((__float_as_uint(pn) ^ __float_as_uint(p)) >> 31);
        pm = p;
        p = pn;
    }
    return cnt;
}

// inverse-iteration arithmetic in the storage precision: fp32 uses the fast reciprocal (the LU of
// T - lambda I only has to be backward stable; the eigenvalue is the binary64 Rayleigh quotient)
__device__ __forceinline__ float ii_div(float a, float b) { return __fdividef(a, b); }
// binary64: MUFU-seeded reciprocal (~1 ulp) instead of the division sequence; the seed flushes subnormal inputs, so a
// (never observed) subnormal divisor is clamped to the smallest magnitude the callers' own `tiny` guards use
__device__ __forceinline__ double ii_div(double a, double b) {
    const double bb = fabs(b) < 1e-290 ? copysign(1e-290, b) : b;
    return a * frcp(bb);
}

__device__ __forceinline__ int sturm_count_f32(int D, const float* d, const float* e2, float x, float pivmin) {
    int cnt = 0;
    float q = d[0] - x;
    if (fabsf(q) < pivmin) q = -pivmin;
    cnt += q < 0.0f;
    for (int i = 1; i < D; ++i) {
        q = d[i] - x - __fdividef(e2[i - 1], q);
        if (fabsf(q) < pivmin) q = -pivmin;
        cnt += q < 0.0f;
    }
    return cnt;
}
// binary64 Sturm count on the unnormalised tridiagonal (e2[i] couples rows i, i+1); MUFU-seeded reciprocal
// with two Newton steps in place of the division (the count stays backward stable)
__device__ __forceinline__ int sturm_count_f64(int D, const double* d, const double* e2, double x) {
    const double pivmin = 1e-290;
    int cnt = 0;
    double q = d[0] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
    for (int i = 1; i < D; ++i) {
        double y;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q));
        y = fma(y, fma(-q, y, 1.0), y);
        y = fma(y, fma(-q, y, 1.0), y);
        q = d[i] - x - e2[i - 1] * y;
        if (fabs(q) < pivmin) q = -pivmin;
        cnt += q < 0.0;
    }
    return cnt;
}

template <class R>
__device__ __forceinline__ int sturm_count_r(int D, const float* d, const float* e2, float x) {
    if constexpr (sizeof(R) == 4) return sturm_count_p32(D, d, e2, x);
    else return sturm_count_f32(D, d, e2, x, 1e-30f);
}

#ifndef GWT_FP32_SOLVES
#define GWT_FP32_SOLVES 2  // inverse-iteration solves for fp32 storage (eig_warp.cuh / eig_cta.cuh)
#endif
#include "eig_warp.cuh"
#include "eig_cta.cuh"
#include "eig_big.cuh"

// in: [batch][D][D] Hermitian (column-major; lower triangle read),
// out: [batch][count][D] top eigenvectors, evals (nullable): [batch][count].
// ws_a: [batch][D][D] double2 (used when D > 64), ws_z: [batch][count][6*D] double, ws_x: [batch][count][D] double2
template <class T>
__global__ void __launch_bounds__(kEigThreads) k_heev_topk(int D, int count, const cplx_t<T>* __restrict__ in,
                                                           cplx_t<T>* __restrict__ out, double* __restrict__ evals,
                                                           double2* __restrict__ ws_a, double* __restrict__ ws_z,
                                                           double2* __restrict__ ws_x, int* __restrict__ fail) {
    using C = cplx_t<T>;
    extern __shared__ __align__(16) unsigned char smem_dyn[];
    __shared__ double2 sv[256];   // Householder vector of the current step
    __shared__ double2 sp[256];   // p / w
    __shared__ double2 salpha[256];
    __shared__ double stau[256];
    __shared__ double sd[256], se2[256], sl[256];
    __shared__ double2 sdelta[256];
    __shared__ double red[33];
    __shared__ int scl[256];   // cluster id per wanted eigenvalue, -> round index
    __shared__ int sround[2];
    const int64_t b = blockIdx.x;
    const int tid = threadIdx.x;
    double2* A = D <= kSmemMaxD ? reinterpret_cast<double2*>(smem_dyn) : ws_a + b * (int64_t)D * D;
    const C* H = in + b * (int64_t)D * D;
    for (int idx = tid; idx < D * D; idx += kEigThreads) {
        const int i = idx % D, j = idx / D;
        if (i >= j) {
            double2 v = to_d2(H[idx]);
            if (i == j) v.y = 0.0;
            A[i + D * j] = v;
            A[j + D * i] = make_double2(v.x, -v.y);
        }
    }
    __syncthreads();
    GWT_CLK(t_ph0);
    // 1. Householder tridiagonalisation: 4 CTA barriers per reflector (warp 0 does the scalar work)
    __shared__ double sK;
    for (int k = 0; k + 2 < D; ++k) {
        const int len = D - k - 1;
        double2* col = A + (k + 1) + D * k;
        if (tid < 32) {
            double tl = 0.0;
            for (int r = 1 + tid; r < len; r += 32) tl += col[r].x * col[r].x + col[r].y * col[r].y;
            for (int o = 16; o > 0; o >>= 1) tl += __shfl_xor_sync(0xffffffffu, tl, o);
            if (tid == 0) {
                const double2 x0 = col[0];
                if (tl == 0.0) {
                    stau[k] = 0.0;
                    salpha[k] = x0;
                } else {
                    const double ax0 = hypot(x0.x, x0.y);
                    const double xnorm = sqrt(tl + ax0 * ax0);
                    const double2 ph = ax0 > 0.0 ? make_double2(x0.x / ax0, x0.y / ax0) : make_double2(1.0, 0.0);
                    const double2 al = make_double2(-ph.x * xnorm, -ph.y * xnorm);
                    const double2 v0 = make_double2(x0.x - al.x, x0.y - al.y);
                    col[0] = v0;  // the reflector overwrites column k below the diagonal
                    stau[k] = 2.0 / (tl + v0.x * v0.x + v0.y * v0.y);
                    salpha[k] = al;
                }
            }
        }
        __syncthreads();
        const double tau = stau[k];
        if (tau == 0.0) continue;  // uniform: column already reduced
        for (int r = tid; r < len; r += kEigThreads) sv[r] = col[r];
        {
            // p = tau A22 v: SPLIT threads per row (lanes of one warp), partial dots + shuffle reduction
            const int split = len <= 32 ? 8 : (len <= 64 ? 4 : (len <= 128 ? 2 : 1));
            const int rows_per_pass = kEigThreads / split;
            const int sub = tid % split;
            for (int r0 = 0; r0 < len; r0 += rows_per_pass) {
                const int r = r0 + tid / split;
                double2 acc = make_double2(0, 0);
                if (r < len) {
                    const double2* arow = A + (k + 1 + r) + D * (k + 1);
                    for (int c = sub; c < len; c += split) cfma(acc, arow[D * c], col[c]);
                }
                for (int o = split / 2; o > 0; o >>= 1) {
                    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
                    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
                }
                if (r < len && sub == 0) sp[r] = make_double2(acc.x * tau, acc.y * tau);
            }
        }
        __syncthreads();
        if (tid < 32) {  // K = tau/2 v^H p (real for Hermitian A22)
            double part = 0.0;
            for (int r = tid; r < len; r += 32) part += sv[r].x * sp[r].x + sv[r].y * sp[r].y;
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            if (tid == 0) sK = 0.5 * tau * part;
        }
        __syncthreads();
        const double kk = sK;
        // A22 -= v w^H + w v^H with w = p - K v formed on the fly
        for (int idx = tid; idx < len * len; idx += kEigThreads) {
            const int r = idx % len, c = idx / len;
            double2 a = A[(k + 1 + r) + D * (k + 1 + c)];
            const double2 vr = sv[r], vc = sv[c];
            const double2 wr = make_double2(sp[r].x - kk * vr.x, sp[r].y - kk * vr.y);
            const double2 wc = make_double2(sp[c].x - kk * vc.x, sp[c].y - kk * vc.y);
            a.x -= vr.x * wc.x + vr.y * wc.y + wr.x * vc.x + wr.y * vc.y;
            a.y -= vr.y * wc.x - vr.x * wc.y + wr.y * vc.x - wr.x * vc.y;
            A[(k + 1 + r) + D * (k + 1 + c)] = a;
        }
        __syncthreads();
    }
    GWT_CLK(t_ph1);
    // 2. real symmetric tridiagonal (d, e) via the phase similarity
    for (int r = tid; r < D; r += kEigThreads) sd[r] = A[r + D * r].x;
    __syncthreads();
    if (tid == 0) {
        double2 dl = make_double2(1.0, 0.0);
        sdelta[0] = dl;
        for (int i = 0; i + 1 < D; ++i) {
            const double2 sub = (i + 2 < D) ? salpha[i] : A[(i + 1) + D * i];
            const double mag = hypot(sub.x, sub.y);
            sl[i] = mag;
            se2[i] = mag * mag;
            if (mag > 0.0) dl = cmul(dl, make_double2(sub.x / mag, sub.y / mag));
            sdelta[i + 1] = dl;
        }
        sl[D - 1] = 0.0;
        se2[D - 1] = 0.0;
    }
    __syncthreads();
    // Gershgorin bounds and scale
    double lo_p = 1e308, hi_p = -1e308, nrm_p = 0.0;
    for (int i = tid; i < D; i += kEigThreads) {
        const double r = (i > 0 ? sl[i - 1] : 0.0) + sl[i];
        lo_p = fmin(lo_p, sd[i] - r);
        hi_p = fmax(hi_p, sd[i] + r);
        nrm_p = fmax(nrm_p, fabs(sd[i]) + r);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo_p = fmin(lo_p, __shfl_xor_sync(0xffffffffu, lo_p, o));
        hi_p = fmax(hi_p, __shfl_xor_sync(0xffffffffu, hi_p, o));
        nrm_p = fmax(nrm_p, __shfl_xor_sync(0xffffffffu, nrm_p, o));
    }
    __syncthreads();
    if ((tid & 31) == 0) {
        red[tid / 32] = lo_p;
        red[8 + tid / 32] = hi_p;
        red[16 + tid / 32] = nrm_p;
    }
    __syncthreads();
    double glo = 1e308, ghi = -1e308, tnorm = 0.0;
    for (int w = 0; w < kEigThreads / 32; ++w) {
        glo = fmin(glo, red[w]);
        ghi = fmax(ghi, red[8 + w]);
        tnorm = fmax(tnorm, red[16 + w]);
    }
    const double eps = 2.220446049250313e-16;
    const double pivmin = fmax(1e-290, eps * eps * fmax(tnorm, 1e-290));
    glo -= 2.0 * eps * tnorm + pivmin;
    ghi += 2.0 * eps * tnorm + pivmin;
    // 3a. bisection (fp32, on T / ||T||): thread t -> t-th largest eigenvalue (ascending index D-1-t)
    __shared__ float fd[256], fe2[256];
    const double inv_n = tnorm > 0.0 ? 1.0 / tnorm : 1.0;
    for (int i = tid; i < D; i += kEigThreads) {
        fd[i] = (float)(sd[i] * inv_n);
        fe2[i] = (float)(se2[i] * inv_n * inv_n);
    }
    __syncthreads();
    double lam = 0.0;
    if (tid < count) {
        const int want = D - 1 - tid;
        const float pivf = 1e-30f;
        float lo = (float)(glo * inv_n) - 1e-6f, hi = (float)(ghi * inv_n) + 1e-6f;
        for (int it = 0; it < 64; ++it) {
            const float mid = 0.5f * (lo + hi);
            if (hi - lo <= 2e-7f * fmaxf(fmaxf(fabsf(lo), fabsf(hi)), 1e-3f) || mid <= lo || mid >= hi) break;
            if (sturm_count_f32(D, fd, fe2, mid, pivf) <= want) lo = mid;
            else hi = mid;
        }
        lam = 0.5 * ((double)lo + (double)hi) * tnorm;
        sp[tid] = make_double2(lam, 0.0);  // stash for cluster detection
    }
    __syncthreads();
    GWT_CLK(t_ph2);
    // clusters among the wanted eigenvalues (descending order): rounds = position inside the cluster
    if (tid == 0) {
        const double ctol = 1e-3 * fmax(tnorm, 1e-300);
        int pos = 0, maxr = 0;
        for (int t = 0; t < count; ++t) {
            pos = (t > 0 && fabs(sp[t - 1].x - sp[t].x) <= ctol) ? pos + 1 : 0;
            scl[t] = pos;
            maxr = max(maxr, pos);
        }
        sround[0] = maxr + 1;
    }
    __syncthreads();
    // 3b. inverse iteration; LU + iterate in the global workspace, thread (eigenvalue) fastest (coalesced)
    double* Zw = (D <= kSmemMaxD && count * 6 * D * 8 <= 96 * 1024)
                     ? reinterpret_cast<double*>(smem_dyn + (size_t)D * D * sizeof(double2))
                     : ws_z + b * (int64_t)count * 6 * D;
    double2* X = ws_x + b * (int64_t)count * D;  // [count][D]; real part = z during the iteration
    const int t = tid;
#define ZW(arr, i) Zw[((int64_t)(arr) * D + (i)) * count + t]
    const double tiny = fmax(eps * tnorm, 1e-290);
    if (t < count) {
        for (int i = 0; i < D; ++i) {
            ZW(0, i) = sd[i] - lam;
            ZW(1, i) = sl[i];
            ZW(2, i) = 0.0;
        }
        for (int i = 0; i + 1 < D; ++i) {
            const double sub = sl[i];
            double di = ZW(0, i);
            if (fabs(di) >= fabs(sub)) {
                if (di == 0.0) di = tiny;
                const double mult = sub / di;
                ZW(0, i) = di;
                ZW(3, i) = mult;
                ZW(4, i) = 0.0;
                ZW(0, i + 1) -= mult * ZW(1, i);
            } else {
                const double mult = di / sub;
                ZW(3, i) = mult;
                ZW(4, i) = 1.0;
                ZW(0, i) = sub;
                const double tmp = ZW(0, i + 1);
                ZW(0, i + 1) = ZW(1, i) - mult * tmp;
                if (i + 2 < D) {
                    ZW(2, i) = ZW(1, i + 1);
                    ZW(1, i + 1) = -mult * ZW(2, i);
                }
                ZW(1, i) = tmp;
            }
        }
        for (int i = 0; i < D; ++i) {
            const double di = ZW(0, i);
            if (fabs(di) < tiny) ZW(0, i) = di < 0 ? -tiny : tiny;
            ZW(5, i) = 1.0 + 0.25 * __sinf(0.7f * i + 1.3f * t);
        }
    }
    const int rounds = sround[0];
    for (int rd = 0; rd < rounds; ++rd) {
        if (t < count && scl[t] == rd) {
            for (int it = 0; it < 4; ++it) {
                for (int s = t - rd; s < t; ++s) {
                    const double2* zs = X + (int64_t)s * D;
                    double dot = 0.0;
                    for (int i = 0; i < D; ++i) dot += zs[i].x * ZW(5, i);
                    for (int i = 0; i < D; ++i) ZW(5, i) -= dot * zs[i].x;
                }
                double nn = 0.0;
                for (int i = 0; i < D; ++i) nn += ZW(5, i) * ZW(5, i);
                const double inv = nn > 0.0 ? rsqrt(nn) : 1.0;
                for (int i = 0; i < D; ++i) ZW(5, i) *= inv;
                if (it == 3) break;
                for (int i = 0; i + 1 < D; ++i) {
                    if (ZW(4, i) != 0.0) {
                        const double t0 = ZW(5, i);
                        ZW(5, i) = ZW(5, i + 1);
                        ZW(5, i + 1) = t0 - ZW(3, i) * ZW(5, i + 1);
                    } else {
                        ZW(5, i + 1) -= ZW(3, i) * ZW(5, i);
                    }
                }
                ZW(5, D - 1) /= ZW(0, D - 1);
                if (D >= 2) ZW(5, D - 2) = (ZW(5, D - 2) - ZW(1, D - 2) * ZW(5, D - 1)) / ZW(0, D - 2);
                for (int i = D - 3; i >= 0; --i)
                    ZW(5, i) = (ZW(5, i) - ZW(1, i) * ZW(5, i + 1) - ZW(2, i) * ZW(5, i + 2)) / ZW(0, i);
                double mx = 0.0;
                for (int i = 0; i < D; ++i) mx = fmax(mx, fabs(ZW(5, i)));
                if (!(mx > 0.0) || !isfinite(mx)) {
                    if (fail) atomicExch(fail, 1);
                    break;
                }
                const double sc = 1.0 / mx;
                for (int i = 0; i < D; ++i) ZW(5, i) *= sc;
            }
            // Rayleigh quotient z^T T z for the reported eigenvalue
            double rq = 0.0;
            for (int i = 0; i < D; ++i) {
                double tz = sd[i] * ZW(5, i);
                if (i > 0) tz += sl[i - 1] * ZW(5, i - 1);
                if (i + 1 < D) tz += sl[i] * ZW(5, i + 1);
                rq += ZW(5, i) * tz;
            }
            sp[t] = make_double2(rq, 0.0);
            double2* zt = X + (int64_t)t * D;
            for (int i = 0; i < D; ++i) zt[i] = make_double2(ZW(5, i), 0.0);
        }
        __syncthreads();
    }
#undef ZW
    GWT_CLK(t_ph3);
    if (evals)
        for (int c = tid; c < count; c += kEigThreads) evals[b * count + c] = sp[c].x;
    // eigenvectors of A: X <- Q diag(delta) z
    for (int idx = tid; idx < count * D; idx += kEigThreads) {
        const int r = idx % D;
        const double z = X[idx].x;
        X[idx] = make_double2(sdelta[r].x * z, sdelta[r].y * z);
    }
    __syncthreads();
    const int warp = tid / 32, lane = tid % 32;
    for (int k = D - 3; k >= 0; --k) {
        const double tau = stau[k];
        if (tau != 0.0) {
            const int len = D - k - 1;
            for (int c = warp; c < count; c += kEigThreads / 32) {
                double2* xc = X + (int64_t)c * D + k + 1;
                double2 dot = make_double2(0, 0);
                for (int r = lane; r < len; r += 32) cfmaconj(dot, A[(k + 1 + r) + D * k], xc[r]);
                for (int o = 16; o > 0; o >>= 1) {
                    dot.x += __shfl_xor_sync(0xffffffffu, dot.x, o);
                    dot.y += __shfl_xor_sync(0xffffffffu, dot.y, o);
                }
                dot.x *= tau;
                dot.y *= tau;
                for (int r = lane; r < len; r += 32) {
                    const double2 v = A[(k + 1 + r) + D * k];
                    double2 xv = xc[r];
                    const double2 pr = cmul(v, dot);
                    xv.x -= pr.x;
                    xv.y -= pr.y;
                    xc[r] = xv;
                }
            }
        }
        __syncthreads();
    }
    // phase normalisation + store
    C* ob = out + b * (int64_t)count * D;
    for (int c = warp; c < count; c += kEigThreads / 32) {
        const double2* xc = X + (int64_t)c * D;
        double best = -1.0;
        int bi = 0;
        for (int r = lane; r < D; r += 32) {
            const double mag = hypot(xc[r].x, xc[r].y);
            if (mag > best) { best = mag; bi = r; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ob2 = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ob2 > best || (ob2 == best && oi < bi)) { best = ob2; bi = oi; }
        }
        double2 fac = make_double2(1.0, 0.0);
        if (best > 0.0) fac = make_double2(xc[bi].x / best, -xc[bi].y / best);
        for (int r = lane; r < D; r += 32) ob[(int64_t)c * D + r] = from_d2<C>(cmul(xc[r], fac));
    }
#ifdef GWT_PHASE_TIMERS
    if (b == 0 && tid == 0) {
        long long t_ph4 = clock64();
        g_eig_phase[0] = t_ph1 - t_ph0;
        g_eig_phase[1] = t_ph2 - t_ph1;
        g_eig_phase[2] = t_ph3 - t_ph2;
        g_eig_phase[3] = t_ph4 - t_ph3;
    }
#endif
}

#ifdef GWT_PHASE_TIMERS
extern "C" int gwt_debug_eig_phases(long long* out4) {
    return (int)cudaMemcpyFromSymbol(out4, g_eig_phase, 8 * sizeof(long long));
}
#endif

// ---------------------------------------------------------------------------
// Warp-per-matrix variant for D <= 64: the same algorithm, warp-synchronous
// (no CTA barriers), W matrices per CTA, each warp's matrix in shared memory.

template <class T>
__global__ void __launch_bounds__(256) k_heev_warp(int D, int count, int64_t batch, int W,
                                                   const cplx_t<T>* __restrict__ in, cplx_t<T>* __restrict__ out,
                                                   double* __restrict__ evals, double* __restrict__ ws_z,
                                                   double2* __restrict__ ws_x, int* __restrict__ fail) {
    using C = cplx_t<T>;
    extern __shared__ __align__(16) unsigned char smem_dyn[];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t b = (int64_t)blockIdx.x * W + warp;
    if (b >= batch) return;
    const size_t per = ((size_t)D * D * 16 + (size_t)D * (16 + 16 + 16 + 8 + 8 + 8 + 8 + 4) + 15) & ~size_t(15);
    unsigned char* base = smem_dyn + warp * per;
    double2* A = reinterpret_cast<double2*>(base);
    double2* pv = A + D * D;        // p / w
    double2* alpha = pv + D;
    double2* delta = alpha + D;
    double* tau = reinterpret_cast<double*>(delta + D);
    double* sd = tau + D;
    double* se = sd + D;
    double* se2 = se + D;
    int* scl = reinterpret_cast<int*>(se2 + D);
    const C* H = in + b * (int64_t)D * D;
    for (int idx = lane; idx < D * D; idx += 32) {
        const int i = idx % D, j = idx / D;
        if (i >= j) {
            double2 v = to_d2(H[idx]);
            if (i == j) v.y = 0.0;
            A[i + D * j] = v;
            A[j + D * i] = make_double2(v.x, -v.y);
        }
    }
    __syncwarp();
    GWT_CLK(t_ph0);
    for (int k = 0; k + 2 < D; ++k) {
        const int len = D - k - 1;
        double2* col = A + (k + 1) + D * k;  // x = A[k+1.., k]; becomes the reflector v
        double tl = 0.0;
        for (int r = 1 + lane; r < len; r += 32) tl += col[r].x * col[r].x + col[r].y * col[r].y;
        const double tail2 = warp_sum(tl);
        if (tail2 == 0.0) {
            if (lane == 0) {
                tau[k] = 0.0;
                alpha[k] = col[0];
            }
            __syncwarp();
            continue;
        }
        if (lane == 0) {
            const double2 x0 = col[0];
            const double ax0 = hypot(x0.x, x0.y);
            const double xnorm = sqrt(tail2 + ax0 * ax0);
            const double2 ph = ax0 > 0.0 ? make_double2(x0.x / ax0, x0.y / ax0) : make_double2(1.0, 0.0);
            const double2 al = make_double2(-ph.x * xnorm, -ph.y * xnorm);
            const double2 v0 = make_double2(x0.x - al.x, x0.y - al.y);
            col[0] = v0;
            tau[k] = 2.0 / (tail2 + v0.x * v0.x + v0.y * v0.y);
            alpha[k] = al;
        }
        __syncwarp();
        const double tk = tau[k];
        double2* A22 = A + (k + 1) + D * (k + 1);
        for (int r = lane; r < len; r += 32) {
            double2 a0 = make_double2(0, 0), a1 = make_double2(0, 0);
            int c = 0;
            for (; c + 1 < len; c += 2) {
                cfma(a0, A22[r + D * c], col[c]);
                cfma(a1, A22[r + D * (c + 1)], col[c + 1]);
            }
            if (c < len) cfma(a0, A22[r + D * c], col[c]);
            pv[r] = make_double2((a0.x + a1.x) * tk, (a0.y + a1.y) * tk);
        }
        __syncwarp();
        double part = 0.0;
        for (int r = lane; r < len; r += 32) part += col[r].x * pv[r].x + col[r].y * pv[r].y;
        const double kk = 0.5 * tk * warp_sum(part);
        for (int r = lane; r < len; r += 32) pv[r] = make_double2(pv[r].x - kk * col[r].x, pv[r].y - kk * col[r].y);
        __syncwarp();
        for (int idx = lane; idx < len * len; idx += 32) {
            const int r = idx % len, c = idx / len;
            double2 a = A22[r + D * c];
            const double2 vr = col[r], wr = pv[r], vc = col[c], wc = pv[c];
            a.x -= vr.x * wc.x + vr.y * wc.y + wr.x * vc.x + wr.y * vc.y;
            a.y -= vr.y * wc.x - vr.x * wc.y + wr.y * vc.x - wr.x * vc.y;
            A22[r + D * c] = a;
        }
        __syncwarp();
    }
    GWT_CLK(t_ph1);
    for (int r = lane; r < D; r += 32) sd[r] = A[r + D * r].x;
    if (lane == 0) {
        double2 dl = make_double2(1.0, 0.0);
        delta[0] = dl;
        for (int i = 0; i + 1 < D; ++i) {
            const double2 sub = (i + 2 < D) ? alpha[i] : A[(i + 1) + D * i];
            const double mag = hypot(sub.x, sub.y);
            se[i] = mag;
            se2[i] = mag * mag;
            if (mag > 0.0) dl = cmul(dl, make_double2(sub.x / mag, sub.y / mag));
            delta[i + 1] = dl;
        }
        se[D - 1] = 0.0;
        se2[D - 1] = 0.0;
    }
    __syncwarp();
    double lo_p = 1e308, hi_p = -1e308, nrm_p = 0.0;
    for (int i = lane; i < D; i += 32) {
        const double r = (i > 0 ? se[i - 1] : 0.0) + se[i];
        lo_p = fmin(lo_p, sd[i] - r);
        hi_p = fmax(hi_p, sd[i] + r);
        nrm_p = fmax(nrm_p, fabs(sd[i]) + r);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo_p = fmin(lo_p, __shfl_xor_sync(0xffffffffu, lo_p, o));
        hi_p = fmax(hi_p, __shfl_xor_sync(0xffffffffu, hi_p, o));
        nrm_p = fmax(nrm_p, __shfl_xor_sync(0xffffffffu, nrm_p, o));
    }
    const double eps = 2.220446049250313e-16;
    const double tnorm = nrm_p;
    const double pivmin = fmax(1e-290, eps * eps * fmax(tnorm, 1e-290));
    const double glo = lo_p - 2.0 * eps * tnorm - pivmin, ghi = hi_p + 2.0 * eps * tnorm + pivmin;
    double* lamv = reinterpret_cast<double*>(pv);  // reuse p/w storage for the wanted eigenvalues
    float* fd = reinterpret_cast<float*>(alpha);      // alpha (no longer needed) -> fp32 copies of T/||T||
    float* fe2 = fd + D;
    const double inv_n = tnorm > 0.0 ? 1.0 / tnorm : 1.0;
    __syncwarp();
    for (int i = lane; i < D; i += 32) {
        fd[i] = (float)(sd[i] * inv_n);
        fe2[i] = (float)(se2[i] * inv_n * inv_n);
    }
    __syncwarp();
    for (int t = lane; t < count; t += 32) {
        const int want = D - 1 - t;
        float lo = (float)(glo * inv_n) - 1e-6f, hi = (float)(ghi * inv_n) + 1e-6f;
        for (int it = 0; it < 64; ++it) {
            const float mid = 0.5f * (lo + hi);
            if (hi - lo <= 2e-7f * fmaxf(fmaxf(fabsf(lo), fabsf(hi)), 1e-3f) || mid <= lo || mid >= hi) break;
            if (sturm_count_f32(D, fd, fe2, mid, 1e-30f) <= want) lo = mid;
            else hi = mid;
        }
        lamv[t] = 0.5 * ((double)lo + (double)hi) * tnorm;
    }
    __syncwarp();
    int rounds = 1;
    if (lane == 0) {
        const double ctol = 1e-3 * fmax(tnorm, 1e-300);
        int pos = 0, maxr = 0;
        for (int t = 0; t < count; ++t) {
            pos = (t > 0 && fabs(lamv[t - 1] - lamv[t]) <= ctol) ? pos + 1 : 0;
            scl[t] = pos;
            maxr = max(maxr, pos);
        }
        rounds = maxr + 1;
    }
    rounds = __shfl_sync(0xffffffffu, rounds, 0);
    __syncwarp();
    GWT_CLK(t_ph2);
    // per-matrix workspaces, lane (eigenvalue) fastest so every warp access is coalesced:
    //   Zw[arr][i][t] (arr: 0 dd, 1 du, 2 du2, 3 ml, 4 sw, 5 x),  X[i][t] eigenvector t
    double* Zw = ws_z + b * (int64_t)count * 6 * D;
    double2* X = ws_x + b * (int64_t)count * D;
#define ZW(arr, i) Zw[((int64_t)(arr) * D + (i)) * count + t]
#define XV(i, c) X[(int64_t)(i) * count + (c)]
    const double tiny = fmax(eps * tnorm, 1e-290);
    for (int rd = 0; rd < rounds; ++rd) {
        for (int t = lane; t < count; t += 32) {
            if (scl[t] != rd) continue;
            const double lam = lamv[t];
            for (int i = 0; i < D; ++i) {
                ZW(0, i) = sd[i] - lam;
                ZW(1, i) = se[i];
                ZW(2, i) = 0.0;
            }
            for (int i = 0; i + 1 < D; ++i) {
                const double sub = se[i];
                double di = ZW(0, i);
                if (fabs(di) >= fabs(sub)) {
                    if (di == 0.0) di = tiny;
                    const double mult = sub / di;
                    ZW(0, i) = di;
                    ZW(3, i) = mult;
                    ZW(4, i) = 0.0;
                    ZW(0, i + 1) -= mult * ZW(1, i);
                } else {
                    const double mult = di / sub;
                    ZW(3, i) = mult;
                    ZW(4, i) = 1.0;
                    ZW(0, i) = sub;
                    const double tmp = ZW(0, i + 1);
                    ZW(0, i + 1) = ZW(1, i) - mult * tmp;
                    if (i + 2 < D) {
                        ZW(2, i) = ZW(1, i + 1);
                        ZW(1, i + 1) = -mult * ZW(2, i);
                    }
                    ZW(1, i) = tmp;
                }
            }
            for (int i = 0; i < D; ++i) {
                const double di = ZW(0, i);
                if (fabs(di) < tiny) ZW(0, i) = di < 0 ? -tiny : tiny;
                ZW(5, i) = 1.0 + 0.25 * __sinf(0.7f * i + 1.3f * t);
            }
            for (int it = 0; it < 4; ++it) {
                for (int s = t - rd; s < t; ++s) {
                    double dot = 0.0;
                    for (int i = 0; i < D; ++i) dot += XV(i, s).x * ZW(5, i);
                    for (int i = 0; i < D; ++i) ZW(5, i) -= dot * XV(i, s).x;
                }
                double nn = 0.0;
                for (int i = 0; i < D; ++i) nn += ZW(5, i) * ZW(5, i);
                const double inv = nn > 0.0 ? rsqrt(nn) : 1.0;
                for (int i = 0; i < D; ++i) ZW(5, i) *= inv;
                if (it == 3) break;
                for (int i = 0; i + 1 < D; ++i) {
                    if (ZW(4, i) != 0.0) {
                        const double t0 = ZW(5, i);
                        ZW(5, i) = ZW(5, i + 1);
                        ZW(5, i + 1) = t0 - ZW(3, i) * ZW(5, i + 1);
                    } else {
                        ZW(5, i + 1) -= ZW(3, i) * ZW(5, i);
                    }
                }
                ZW(5, D - 1) /= ZW(0, D - 1);
                if (D >= 2) ZW(5, D - 2) = (ZW(5, D - 2) - ZW(1, D - 2) * ZW(5, D - 1)) / ZW(0, D - 2);
                for (int i = D - 3; i >= 0; --i)
                    ZW(5, i) = (ZW(5, i) - ZW(1, i) * ZW(5, i + 1) - ZW(2, i) * ZW(5, i + 2)) / ZW(0, i);
                double mx = 0.0;
                for (int i = 0; i < D; ++i) mx = fmax(mx, fabs(ZW(5, i)));
                if (!(mx > 0.0) || !isfinite(mx)) {
                    if (fail) atomicExch(fail, 1);
                    break;
                }
                const double sc = 1.0 / mx;
                for (int i = 0; i < D; ++i) ZW(5, i) *= sc;
            }
            for (int i = 0; i < D; ++i) XV(i, t) = make_double2(ZW(5, i), 0.0);
            double rq = 0.0;  // Rayleigh quotient for the reported eigenvalue
            for (int i = 0; i < D; ++i) {
                double tz = sd[i] * ZW(5, i);
                if (i > 0) tz += se[i - 1] * ZW(5, i - 1);
                if (i + 1 < D) tz += se[i] * ZW(5, i + 1);
                rq += ZW(5, i) * tz;
            }
            lamv[t] = rq;
        }
        __syncwarp();
    }
    GWT_CLK(t_ph3);
    if (evals)
        for (int c = lane; c < count; c += 32) evals[b * count + c] = lamv[c];
    // back-transform: lane = column; x <- H_0 ... H_{D-3} diag(delta) z
    C* ob = out + b * (int64_t)count * D;
    for (int c = lane; c < count; c += 32) {
        for (int r = 0; r < D; ++r) {
            const double z = XV(r, c).x;
            XV(r, c) = make_double2(delta[r].x * z, delta[r].y * z);
        }
        for (int k = D - 3; k >= 0; --k) {
            const double tk = tau[k];
            if (tk == 0.0) continue;
            const double2* v = A + (k + 1) + D * k;
            const int len = D - k - 1;
            double2 d0 = make_double2(0, 0), d1 = make_double2(0, 0);
            int r = 0;
            for (; r + 1 < len; r += 2) {
                cfmaconj(d0, v[r], XV(k + 1 + r, c));
                cfmaconj(d1, v[r + 1], XV(k + 2 + r, c));
            }
            if (r < len) cfmaconj(d0, v[r], XV(k + 1 + r, c));
            const double2 dot = make_double2((d0.x + d1.x) * tk, (d0.y + d1.y) * tk);
            for (int rr = 0; rr < len; ++rr) {
                const double2 pr = cmul(v[rr], dot);
                double2 xv = XV(k + 1 + rr, c);
                xv.x -= pr.x;
                xv.y -= pr.y;
                XV(k + 1 + rr, c) = xv;
            }
        }
        double best = -1.0;
        int bi = 0;
        for (int r = 0; r < D; ++r) {
            const double2 xv = XV(r, c);
            const double mag = xv.x * xv.x + xv.y * xv.y;
            if (mag > best) { best = mag; bi = r; }
        }
        double2 fac = make_double2(1.0, 0.0);
        if (best > 0.0) {
            const double2 xb = XV(bi, c);
            const double im = rsqrt(best);
            fac = make_double2(xb.x * im, -xb.y * im);
        }
        for (int r = 0; r < D; ++r) ob[(int64_t)c * D + r] = from_d2<C>(cmul(XV(r, c), fac));
    }
#ifdef GWT_PHASE_TIMERS
    if (b == 0 && lane == 0) {
        const long long t_ph4 = clock64();
        g_eig_phase[0] = t_ph1 - t_ph0;
        g_eig_phase[1] = t_ph2 - t_ph1;
        g_eig_phase[2] = t_ph3 - t_ph2;
        g_eig_phase[3] = t_ph4 - t_ph3;
    }
#endif
#undef ZW
#undef XV
}

// ---------------------------------------------------------------------------
// Parallel cyclic Jacobi for 8 < D <= 64: one CTA per matrix, A and V in shared
// memory (binary64). Each round applies D/2 disjoint plane rotations (round-robin
// "circle" pairing) with the rotation of the reference test oracle
// (proj/tests/support/oracles.hpp:31-97): the rotations are computed by D/2 threads,
// then all 2x2 blocks of A and all row pairs of V are updated in parallel.
template <class T>
__global__ void __launch_bounds__(256) k_heev_jacobi(int D, int count, const cplx_t<T>* __restrict__ in,
                                                     cplx_t<T>* __restrict__ out, double* __restrict__ evals,
                                                     int* __restrict__ fail) {
    using C = cplx_t<T>;
    extern __shared__ __align__(16) unsigned char smem_dyn[];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int D2 = (D + 1) & ~1, NP = D2 / 2;
    const int LDA = D + 1;  // padded stride
    double2* A = reinterpret_cast<double2*>(smem_dyn);  // A[r + LDA*c]
    double2* V = A + (size_t)D * LDA;                   // V[r + LDA*c]
    double2* Upq = V + (size_t)D * LDA;                 // per pair: [0]=(c,0) [1]=s [2]=uqp [3]=uqq
    int* pp = reinterpret_cast<int*>(Upq + 4 * 32);     // pair -> p
    int* pq = pp + 32;                                  // pair -> q
    __shared__ double red[33];
    __shared__ int sel[64];
    const int64_t b = blockIdx.x;
    const C* H = in + b * (int64_t)D * D;
    for (int idx = tid; idx < D * D; idx += nt) {
        const int i = idx % D, j = idx / D;
        if (i >= j) {
            double2 v = to_d2(H[idx]);
            if (i == j) v.y = 0.0;
            A[i + LDA * j] = v;
            A[j + LDA * i] = make_double2(v.x, -v.y);
        }
        V[i + LDA * j] = make_double2(i == j ? 1.0 : 0.0, 0.0);
    }
    __syncthreads();
    int sweep = 0;
    for (; sweep < 40; ++sweep) {
        double off = 0.0, dia = 0.0;
        for (int idx = tid; idx < D * D; idx += nt) {
            const int i = idx % D, j = idx / D;
            const double2 a = A[i + LDA * j];
            if (i < j) off += a.x * a.x + a.y * a.y;
            else if (i == j) dia += a.x * a.x;
        }
        off = block_sum(off, red);
        dia = block_sum(dia, red);
        if (off <= 1e-30 * dia || off == 0.0) break;
        for (int r = 0; r < D2 - 1; ++r) {
            if (tid < NP) {
                const int i = tid;
                int a = i == 0 ? D2 - 1 : (r + i) % (D2 - 1);
                int bq = (r + D2 - 1 - i) % (D2 - 1);
                const int p = min(a, bq), q = max(a, bq);
                pp[i] = p;
                pq[i] = q;
                double c = 1.0, s = 0.0, phr = 1.0, phi = 0.0;
                if (q < D) {
                    const double2 apq = A[p + LDA * q];
                    const double b2 = apq.x * apq.x + apq.y * apq.y;
                    if (b2 > 1e-300) {
                        const double rb = rsqrt(b2);
                        phr = apq.x * rb;
                        phi = apq.y * rb;
                        const double tau = (A[q + LDA * q].x - A[p + LDA * p].x) * (0.5 * rb);
                        const double tt = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        c = rsqrt(1.0 + tt * tt);
                        s = tt * c;
                    }
                }
                Upq[4 * i + 0] = make_double2(c, 0.0);
                Upq[4 * i + 1] = make_double2(s, 0.0);
                Upq[4 * i + 2] = make_double2(-s * phr, s * phi);  // -s conj(ph)
                Upq[4 * i + 3] = make_double2(c * phr, -c * phi);  //  c conj(ph)
            }
            __syncthreads();
            // A <- U^H A U on every 2x2 block (pair i rows, pair j cols); V <- V U
            for (int idx = tid; idx < NP * NP; idx += nt) {
                const int i = idx % NP, j = idx / NP;
                const int p = pp[i], q = pq[i], p2 = pp[j], q2 = pq[j];
                const bool qi = q < D, qj = q2 < D;
                const double2 ui0 = Upq[4 * i], ui1 = Upq[4 * i + 1], ui2 = Upq[4 * i + 2], ui3 = Upq[4 * i + 3];
                const double2 uj0 = Upq[4 * j], uj1 = Upq[4 * j + 1], uj2 = Upq[4 * j + 2], uj3 = Upq[4 * j + 3];
                const double2 zero = make_double2(0.0, 0.0);
                const double2 a00 = A[p + LDA * p2];
                const double2 a01 = qj ? A[p + LDA * q2] : zero;
                const double2 a10 = qi ? A[q + LDA * p2] : zero;
                const double2 a11 = (qi && qj) ? A[q + LDA * q2] : zero;
                // B = A U_j (columns p2, q2)
                double2 b00 = cmul(a00, uj0), b01 = cmul(a00, uj1), b10 = cmul(a10, uj0), b11 = cmul(a10, uj1);
                cfma(b00, a01, uj2);
                cfma(b01, a01, uj3);
                cfma(b10, a11, uj2);
                cfma(b11, a11, uj3);
                // A' = U_i^H B
                double2 n00 = cmul(cconj(ui0), b00), n01 = cmul(cconj(ui0), b01);
                double2 n10 = cmul(cconj(ui1), b00), n11 = cmul(cconj(ui1), b01);
                cfmaconj(n00, ui2, b10);
                cfmaconj(n01, ui2, b11);
                cfmaconj(n10, ui3, b10);
                cfmaconj(n11, ui3, b11);
                A[p + LDA * p2] = n00;
                if (qj) A[p + LDA * q2] = n01;
                if (qi) A[q + LDA * p2] = n10;
                if (qi && qj) A[q + LDA * q2] = n11;
            }
            for (int idx = tid; idx < D * NP; idx += nt) {
                const int row = idx % D, j = idx / D;
                const int p2 = pp[j], q2 = pq[j];
                if (q2 >= D) continue;
                const double2 uj0 = Upq[4 * j], uj1 = Upq[4 * j + 1], uj2 = Upq[4 * j + 2], uj3 = Upq[4 * j + 3];
                const double2 vp = V[row + LDA * p2], vq = V[row + LDA * q2];
                double2 np = cmul(vp, uj0), nq = cmul(vp, uj1);
                cfma(np, vq, uj2);
                cfma(nq, vq, uj3);
                V[row + LDA * p2] = np;
                V[row + LDA * q2] = nq;
            }
            __syncthreads();
        }
    }
    if (sweep >= 40 && tid == 0 && fail) atomicExch(fail, 1);
    // select top-count (descending, lowest index first on ties)
    for (int r = tid; r < D; r += nt) {
        const double v = A[r + LDA * r].x;
        int rk = 0;
        for (int s2 = 0; s2 < D; ++s2) {
            const double w = A[s2 + LDA * s2].x;
            rk += (w > v || (w == v && s2 < r)) ? 1 : 0;
        }
        if (rk < count) sel[rk] = r;
    }
    __syncthreads();
    if (evals)
        for (int c = tid; c < count; c += nt) evals[b * count + c] = A[sel[c] + LDA * sel[c]].x;
    const int warp = tid / 32, lane = tid % 32;
    C* ob = out + b * (int64_t)count * D;
    for (int c = warp; c < count; c += nt / 32) {
        const double2* vc = V + LDA * sel[c];
        double best = -1.0;
        int bi = 0;
        for (int r = lane; r < D; r += 32) {
            const double mag = vc[r].x * vc[r].x + vc[r].y * vc[r].y;
            if (mag > best) { best = mag; bi = r; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ob2 = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ob2 > best || (ob2 == best && oi < bi)) { best = ob2; bi = oi; }
        }
        double2 fac = make_double2(1.0, 0.0);
        if (best > 0.0) {
            const double im = rsqrt(best);
            fac = make_double2(vc[bi].x * im, -vc[bi].y * im);
        }
        for (int r = lane; r < D; r += 32) ob[(int64_t)c * D + r] = from_d2<C>(cmul(vc[r], fac));
    }
}

// ---------------------------------------------------------------------------
// D <= 8: one thread per matrix, cyclic Jacobi in registers (jacobi_herm).
template <class T, int M>
__global__ void __launch_bounds__(128) k_heev_small(int count, int64_t batch, const cplx_t<T>* __restrict__ in,
                                                    cplx_t<T>* __restrict__ out, double* __restrict__ evals) {
    using C = cplx_t<T>;
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    const C* H = in + b * M * M;
    double2 A[M][M], V[M][M];
#pragma unroll
    for (int j = 0; j < M; ++j)
#pragma unroll
        for (int i = 0; i < M; ++i)
            if (i >= j) {
                double2 v = to_d2(H[i + M * j]);
                if (i == j) v.y = 0.0;
                A[i][j] = v;
                A[j][i] = make_double2(v.x, -v.y);
            }
    jacobi_herm<M>(A, V);
    double lam[M];
#pragma unroll
    for (int r = 0; r < M; ++r) lam[r] = A[r][r].x;
    C* ob = out + b * (int64_t)count * M;
#pragma unroll
    for (int r = 0; r < M; ++r) {
        int rk = 0;
#pragma unroll
        for (int s = 0; s < M; ++s) rk += (lam[s] > lam[r] || (lam[s] == lam[r] && s < r)) ? 1 : 0;
        if (rk < count) {
            double best = -1.0;
            int bi = 0;
#pragma unroll
            for (int a = 0; a < M; ++a) {
                const double mag = V[a][r].x * V[a][r].x + V[a][r].y * V[a][r].y;
                if (mag > best) { best = mag; bi = a; }
            }
            double2 vb = V[0][r];
#pragma unroll
            for (int a = 0; a < M; ++a)
                if (a == bi) vb = V[a][r];
            double2 fac = make_double2(1.0, 0.0);
            if (best > 0.0) {
                const double im = rsqrt(best);
                fac = make_double2(vb.x * im, -vb.y * im);
            }
#pragma unroll
            for (int a = 0; a < M; ++a) ob[(int64_t)rk * M + a] = from_d2<C>(cmul(V[a][r], fac));
            if (evals) evals[b * count + rk] = lam[r];
        }
    }
}

template <class T>
cudaError_t launch_heev_topk(int D, int count, int64_t batch, const void* in, void* out, double* evals, double2* ws_a,
                             double* ws_z, double2* ws_x, int* fail, cudaStream_t st) {
    if (D > 256 || D < 1 || count < 1 || count > D) return cudaErrorInvalidValue;
    const char* mode = env_once("GWT_EIG_MODE");  // tuning override: "warp", "cta"
    const bool force_warp = mode && std::strcmp(mode, "warp") == 0, force_cta = mode && std::strcmp(mode, "cta") == 0;
    const bool legacy_warp = mode && std::strcmp(mode, "warp_old") == 0;
    if (!force_warp && !force_cta && D <= 8) {
        const unsigned blocks = (unsigned)((batch + 127) / 128);
        switch (D) {
#define GWT_SMALL(MM) \
    case MM: k_heev_small<T, MM><<<blocks, 128, 0, st>>>(count, batch, (const cplx_t<T>*)in, (cplx_t<T>*)out, evals); break;
            GWT_SMALL(1) GWT_SMALL(2) GWT_SMALL(3) GWT_SMALL(4) GWT_SMALL(5) GWT_SMALL(6) GWT_SMALL(7) GWT_SMALL(8)
#undef GWT_SMALL
        }
        return cudaGetLastError();
    }
    const char* jmode = env_once("GWT_EIG_JACOBI");
    if (jmode && D <= kSmemMaxD) {
        // parallel cyclic Jacobi, one CTA per matrix (kept for comparison; slower than Householder on B200)
        const size_t sm = sizeof(double2) * ((size_t)2 * D * (D + 1) + 4 * 32) + sizeof(int) * 64;
        cudaError_t e = cudaFuncSetAttribute(k_heev_jacobi<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
        const int threads = D <= 16 ? 64 : (D <= 32 ? 128 : 256);
        k_heev_jacobi<T><<<(unsigned)batch, threads, sm, st>>>(D, count, (const cplx_t<T>*)in, (cplx_t<T>*)out, evals,
                                                              fail);
        return cudaGetLastError();
    }
    const bool cta32 = mode && std::strcmp(mode, "cta32") == 0;
    if (cta32 && D <= 32) {
        const EigCtaLayout L = eig_cta_layout(D, count, sizeof(T));
        cudaError_t e = cudaFuncSetAttribute(k_heev_cr<T, 32, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)L.total);
        if (e != cudaSuccess) return e;
        k_heev_cr<T, 32, 128><<<(unsigned)batch, 128, L.total, st>>>(D, count, (const cplx_t<T>*)in, (cplx_t<T>*)out,
                                                                      evals, fail);
        return cudaGetLastError();
    }
    if (!force_cta && !force_warp && !legacy_warp && D <= 32) {
        // warp per matrix in the storage precision, registers + shared memory only (eig_warp.cuh)
        const EigWarpLayout L = eig_warp_layout(D, count, sizeof(T));
        int W = 4;
        while (W > 1 && W * L.total > 100 * 1024) W /= 2;
        const size_t sm = L.total * W;
        const unsigned blocks = (unsigned)((batch + W - 1) / W);
        cudaError_t e;
        if (D <= 16) {
            e = cudaFuncSetAttribute(k_heev_wr<T, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            if (e != cudaSuccess) return e;
            k_heev_wr<T, 16><<<blocks, 32 * W, sm, st>>>(D, count, batch, W, (const cplx_t<T>*)in, (cplx_t<T>*)out,
                                                          evals, fail);
        } else {
            e = cudaFuncSetAttribute(k_heev_wr<T, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            if (e != cudaSuccess) return e;
            k_heev_wr<T, 32><<<blocks, 32 * W, sm, st>>>(D, count, batch, W, (const cplx_t<T>*)in, (cplx_t<T>*)out,
                                                          evals, fail);
        }
        return cudaGetLastError();
    }
    if (!force_cta && !force_warp && !legacy_warp && D > 32 && count <= 64 && (sizeof(T) == 4 ? D <= 128 : D <= 64)) {
        // CTA per matrix in the storage precision, matrix in shared memory (eig_cta.cuh)
        const EigCtaLayout L = eig_cta_layout(D, count, sizeof(T));
        if (L.total <= 227 * 1024) {
            const size_t sm = L.total;
            cudaError_t e;
            if (D <= 64 && sizeof(T) == 4 && batch <= 64) {
                // small batch (C2 tx Grams): latency-bound, register-resident Householder
                e = cudaFuncSetAttribute(k_heev_cr<T, 64, 256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sm);
                if (e != cudaSuccess) return e;
                k_heev_cr<T, 64, 256, true><<<(unsigned)batch, 256, sm, st>>>(D, count, (const cplx_t<T>*)in,
                                                                              (cplx_t<T>*)out, evals, fail);
            } else if (D <= 64) {
                e = cudaFuncSetAttribute(k_heev_cr<T, 64, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                if (e != cudaSuccess) return e;
                // binary64 D <= 64 (the delay Grams): 2 CTAs per SM when the layout fits (<= 113 KB each)
                e = cudaFuncSetAttribute(k_heev_cr<T, 64, 256>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
                if (e != cudaSuccess) return e;
                k_heev_cr<T, 64, 256><<<(unsigned)batch, 256, sm, st>>>(D, count, (const cplx_t<T>*)in, (cplx_t<T>*)out,
                                                                  evals, fail);
            } else {
                e = cudaFuncSetAttribute(k_heev_cr<T, 128, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                if (e != cudaSuccess) return e;
                k_heev_cr<T, 128, 256><<<(unsigned)batch, 256, sm, st>>>(D, count, (const cplx_t<T>*)in, (cplx_t<T>*)out,
                                                                   evals, fail);
            }
            return cudaGetLastError();
        }
    }
    const bool cr_fits = D <= 128 && count <= 64 && eig_cta_layout(D, count, sizeof(T)).total <= 227 * 1024;
    if (sizeof(T) == 4 && !force_cta && !force_warp && !legacy_warp && D > 64 && D <= 256 && count <= 128 &&
        eig_big_smem(D, count) <= 227 * 1024 && !(D <= 128 && cr_fits)) {
        // fp32, matrix in the (L2-resident) global workspace (eig_big.cuh)
        const size_t sm = eig_big_smem(D, count);
        cudaError_t e = cudaFuncSetAttribute(k_heev_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
        // joint-orthogonalisation threshold of the inverse iterations (relative to ||T||)
        static const double big_ctol = [] {
            const char* v = env_once("GWT_EIG_BIG_CTOL");
            return v ? std::atof(v) : 1e-4;
        }();
        k_heev_big<<<(unsigned)batch, kBigNT, sm, st>>>(D, count, big_ctol, (const float2*)in, (float2*)out, evals,
                                                        reinterpret_cast<float2*>(ws_a), reinterpret_cast<float*>(ws_z),
                                                        fail);
        return cudaGetLastError();
    }
    if (!force_cta && (force_warp || legacy_warp ? D <= kSmemMaxD : D <= 32)) {
        // warp per matrix (Householder + bisection + inverse iteration); W matrices per CTA
        const size_t per = ((size_t)D * D * 16 + (size_t)D * (16 + 16 + 16 + 8 + 8 + 8 + 8 + 4) + 15) & ~size_t(15);
        const int W = (int)std::max<size_t>(1, std::min<size_t>(8, (200 * 1024) / per));
        const size_t sm = per * W;
        cudaError_t e = cudaFuncSetAttribute(k_heev_warp<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
        k_heev_warp<T><<<(unsigned)((batch + W - 1) / W), 32 * W, sm, st>>>(D, count, batch, W, (const cplx_t<T>*)in,
                                                                          (cplx_t<T>*)out, evals, ws_z, ws_x, fail);
        return cudaGetLastError();
    }
    // D > 32 (or forced): CTA per matrix, Householder + bisection + inverse iteration; A in smem when D <= 64
    const size_t smA = D <= kSmemMaxD ? sizeof(double2) * D * D +
                                            ((size_t)count * 6 * D * 8 <= 96 * 1024 ? (size_t)count * 6 * D * 8 : 0)
                                      : 0;
    if (smA > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_heev_topk<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smA);
        if (e != cudaSuccess) return e;
    }
    k_heev_topk<T><<<(unsigned)batch, kEigThreads, smA, st>>>(D, count, (const cplx_t<T>*)in, (cplx_t<T>*)out, evals,
                                                             ws_a, ws_z, ws_x, fail);
    return cudaGetLastError();
}

// workspace doubles needed per matrix: A (D > 64 only) as double2, LU+vector 6*D per wanted pair
size_t heev_ws_a_elems(int D) { return (size_t)D * D; }
size_t heev_ws_z_elems(int D, int count) { return (size_t)count * 6 * D; }

template cudaError_t launch_heev_topk<float>(int, int, int64_t, const void*, void*, double*, double2*, double*,
                                             double2*, int*, cudaStream_t);
template cudaError_t launch_heev_topk<double>(int, int, int64_t, const void*, void*, double*, double2*, double*,
                                              double2*, int*, cudaStream_t);

}  // namespace gwtk
