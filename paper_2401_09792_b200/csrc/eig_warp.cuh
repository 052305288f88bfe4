// Warp-per-matrix Hermitian top-k eigensolver for 8 < D <= 32, in the storage precision R
// (float for c64 Grams, double for c128). Included by k_eig.cu.
//
// Same algorithm and conventions as k_heev_topk (reference: leading_eigenvectors,
// proj/src/linalg.cpp:27-45, Eigen SelfAdjointEigenSolver reversed + phase_normalize_columns
// :11-25), restructured so that nothing on a serial chain touches global memory:
//  1. Householder tridiagonalisation, lane r owns row r of the shared-memory matrix; the
//     reflector v and w = p - K v are broadcast from shared memory (one wavefront each), the
//     matrix rows are read/written conflict-free, loads batched ahead of stores.
//  2. fp32 multisection on Sturm counts of T/||T||: S = 32/count lanes per wanted eigenvalue
//     evaluate S interior points per round (interval shrinks (S+1)x per round).
//  3. Inverse iteration (pivoted tridiagonal LU, LAPACK dlagtf-style; 3 solves), one lane per
//     eigenvalue, the iterate in registers and the LU factors in shared memory; eigenvalues
//     within 1e-3 ||T|| form clusters orthogonalised (MGS) inside the iteration round by round.
//  4. Back-transform through the reflectors with the vector in registers (reflector entries are
//     warp-broadcast reads), phase normalisation (largest |.| entry real >= 0, lowest index).
#pragma once
// (included inside namespace gwtk, after sturm_count_f32 and the phase-timer macros)

struct EigWarpLayout {
    size_t oA, ov, ow, otau, osub, odl, od, oe, oe2, ofd, ofe2, olam, oscl, odd, odu, oml, oxr, total;
};

__host__ __device__ inline EigWarpLayout eig_warp_layout(int D, int count, int rs) {
    EigWarpLayout L;
    size_t o = 0;
    const size_t cs = 2 * (size_t)rs;
#define GWT_TAKE(field, bytes)          \
    L.field = o;                        \
    o = (o + (bytes) + 15) & ~size_t(15);
    GWT_TAKE(oA, (size_t)D * D * cs)
    GWT_TAKE(ov, ((D + 31) / 32 * 32) * cs)  // a full warp's worth: hh_reg32 reads v/w pairs up to column 31
    GWT_TAKE(ow, ((D + 31) / 32 * 32) * cs)
    GWT_TAKE(otau, D * (size_t)rs)
    GWT_TAKE(osub, D * cs)
    GWT_TAKE(odl, D * cs)
    GWT_TAKE(od, D * (size_t)rs)
    GWT_TAKE(oe, D * (size_t)rs)
    GWT_TAKE(oe2, D * (size_t)rs)
    GWT_TAKE(ofd, D * 4)
    GWT_TAKE(ofe2, D * 4)
    GWT_TAKE(olam, count * 8)
    GWT_TAKE(oscl, count * 4)
    GWT_TAKE(odd, (size_t)D * count * rs)
    GWT_TAKE(odu, (size_t)D * count * rs)
    GWT_TAKE(oml, (size_t)D * count * rs)
    GWT_TAKE(oxr, (size_t)D * count * rs)
#undef GWT_TAKE
    L.total = o;
    return L;
}

template <class R>
__device__ __forceinline__ R warp_sum_r(R v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float2 shfl_c(float2 v, int src) {
    return make_float2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}
__device__ __forceinline__ double2 shfl_c(double2 v, int src) {
    return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// Householder reflector of x = (x0, tail) with ||tail||^2 = t2 (t2 > 0): alpha = -phase(x0) ||x||,
// v0 = x0 - alpha, tau = 2 / ||v||^2. fp32: one rsqrt + one reciprocal on the step's critical path.
__device__ __forceinline__ void reflector(float2 x0, float t2, float2& al, float2& v0, float& tk) {
    const float s2 = x0.x * x0.x + x0.y * x0.y;
    const float xn = sqrtf(t2 + s2);
    if (s2 > 0.f) {
        const float f = xn * rsqrtf(s2);  // ||x|| / |x0|
        al = make_float2(-x0.x * f, -x0.y * f);
        v0 = make_float2(x0.x * (1.f + f), x0.y * (1.f + f));
        tk = __frcp_rn(0.5f * (t2 + s2 * (1.f + f) * (1.f + f)));
    } else {
        al = make_float2(-xn, 0.f);
        v0 = make_float2(xn, 0.f);
        tk = __frcp_rn(0.5f * (t2 + xn * xn));
    }
}
__device__ __forceinline__ void reflector(double2 x0, double t2, double2& al, double2& v0, double& tk) {
    const double ax0 = hypot(x0.x, x0.y);
    const double xnorm = sqrt(t2 + ax0 * ax0);
    const double2 ph = ax0 > 0.0 ? make_double2(x0.x / ax0, x0.y / ax0) : make_double2(1.0, 0.0);
    al = make_double2(-ph.x * xnorm, -ph.y * xnorm);
    v0 = make_double2(x0.x - al.x, x0.y - al.y);
    tk = 2.0 / (t2 + v0.x * v0.x + v0.y * v0.y);
}

// Register-resident Householder for fp32 storage and 16 < D <= 32 (phase 1 of k_heev_wr): lane r
// keeps row r of the matrix in registers, so a reflector step costs two broadcast 16-byte shared
// loads per column pair (v and w) instead of a shared-memory read-modify-write of the whole trailing
// matrix (the old form was shared-pipe bound with ~12 warps per SM). v_c = w_c = 0 for c <= k, so
// the mat-vec and the rank-2 update run unpredicated over a static column range [CB, 32): the k
// loop is split into 4 blocks of 8 steps, each starting at column CB = 8 b.
template <int CB>
__device__ __forceinline__ void hh_reg_block(int k0, int k1, int D, int r, float2 (&a)[32], float2& x, float2* A,
                                             float2* vv, float2* ww, float* tau, float2* sub) {
    for (int k = k0; k < k1 && k + 2 < D; ++k) {
        const bool act = r > k && r < D;
        const float t2 = warp_sum_r<float>((r > k + 1 && r < D) ? x.x * x.x + x.y * x.y : 0.f);
        const float2 x0 = shfl_c(x, k + 1);
        if (t2 == 0.f) {  // warp-uniform: column already reduced
            if (r == 0) {
                tau[k] = 0.f;
                sub[k] = x0;
            }
#pragma unroll
            for (int c = CB; c < 32; ++c)
                if (c == k + 1) x = a[c];
            continue;
        }
        float2 al, v0;
        float tk;
        reflector(x0, t2, al, v0, tk);
        const float2 v = act ? (r == k + 1 ? v0 : x) : make_float2(0.f, 0.f);
        if (act) A[r + D * k] = v;  // reflector column k (read by the back-transform)
        if (r == 0) {
            tau[k] = tk;
            sub[k] = al;
        }
        vv[r] = v;
        __syncwarp();
        float2 p0 = make_float2(0.f, 0.f), p1 = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = CB; c < 32; c += 2) {
            const float4 vc = *reinterpret_cast<const float4*>(vv + c);
            cfma(p0, a[c], make_float2(vc.x, vc.y));
            cfma(p1, a[c + 1], make_float2(vc.z, vc.w));
        }
        const float2 p = make_float2(tk * (p0.x + p1.x), tk * (p0.y + p1.y));
        const float kk = 0.5f * tk * warp_sum_r<float>(act ? v.x * p.x + v.y * p.y : 0.f);
        const float2 w = act ? make_float2(p.x - kk * v.x, p.y - kk * v.y) : make_float2(0.f, 0.f);
        ww[r] = w;
        __syncwarp();
#pragma unroll
        for (int c = CB; c < 32; c += 2) {
            const float4 vc = *reinterpret_cast<const float4*>(vv + c);
            const float4 wc = *reinterpret_cast<const float4*>(ww + c);
            // a[r][c] -= v_r conj(w_c) + w_r conj(v_c)
            a[c].x -= v.x * wc.x + v.y * wc.y + w.x * vc.x + w.y * vc.y;
            a[c].y -= v.y * wc.x - v.x * wc.y + w.y * vc.x - w.x * vc.y;
            a[c + 1].x -= v.x * wc.z + v.y * wc.w + w.x * vc.z + w.y * vc.w;
            a[c + 1].y -= v.y * wc.z - v.x * wc.w + w.y * vc.z - w.x * vc.w;
        }
#pragma unroll
        for (int c = CB; c < 32; ++c)
            if (c == k + 1) x = a[c];
        __syncwarp();  // v/w of this step consumed before the next step rewrites them
    }
}

__device__ __forceinline__ void hh_reg32(int D, int r, float2* A, float2* vv, float2* ww, float* tau, float2* sub) {
    float2 a[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) a[c] = (r < D && c < D) ? A[r + D * c] : make_float2(0.f, 0.f);
    float2 x = a[0];
    hh_reg_block<0>(0, 8, D, r, a, x, A, vv, ww, tau, sub);
    hh_reg_block<8>(8, 16, D, r, a, x, A, vv, ww, tau, sub);
    hh_reg_block<16>(16, 24, D, r, a, x, A, vv, ww, tau, sub);
    hh_reg_block<24>(24, 32, D, r, a, x, A, vv, ww, tau, sub);
    // diagonal and the last subdiagonal entry back to shared memory (phase 2 reads them there)
    float2 dg = make_float2(0.f, 0.f), ls = make_float2(0.f, 0.f);
#pragma unroll
    for (int c = 0; c < 32; ++c) {
        if (c == r) dg = a[c];
        if (c == D - 2) ls = a[c];
    }
    if (r < D) A[r + D * r] = dg;
    if (r == D - 1 && D >= 2) A[(D - 1) + D * (D - 2)] = ls;
    __syncwarp();
}

template <class R, int DM>
__global__ void __launch_bounds__(128) k_heev_wr(int D, int count, int64_t batch, int W,
                                                 const cplx_t<R>* __restrict__ in, cplx_t<R>* __restrict__ out,
                                                 double* __restrict__ evals, int* __restrict__ fail) {
    using C = cplx_t<R>;
    extern __shared__ __align__(16) unsigned char smem_dyn[];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t b = (int64_t)blockIdx.x * W + warp;
    if (b >= batch) return;
    const EigWarpLayout L = eig_warp_layout(D, count, sizeof(R));
    unsigned char* base = smem_dyn + warp * L.total;
    C* A = reinterpret_cast<C*>(base + L.oA);
    C* vv = reinterpret_cast<C*>(base + L.ov);
    C* ww = reinterpret_cast<C*>(base + L.ow);
    R* tau = reinterpret_cast<R*>(base + L.otau);
    C* sub = reinterpret_cast<C*>(base + L.osub);
    C* dlt = reinterpret_cast<C*>(base + L.odl);
    R* sd = reinterpret_cast<R*>(base + L.od);
    R* se = reinterpret_cast<R*>(base + L.oe);
    R* se2 = reinterpret_cast<R*>(base + L.oe2);
    float* fd = reinterpret_cast<float*>(base + L.ofd);
    float* fe2 = reinterpret_cast<float*>(base + L.ofe2);
    double* lamv = reinterpret_cast<double*>(base + L.olam);
    int* scl = reinterpret_cast<int*>(base + L.oscl);
    R* DDv = reinterpret_cast<R*>(base + L.odd);
    R* DUv = reinterpret_cast<R*>(base + L.odu);
    R* MLv = reinterpret_cast<R*>(base + L.oml);
    R* XR = reinterpret_cast<R*>(base + L.oxr);
    const C* H = in + b * (int64_t)D * D;
    for (int idx = lane; idx < D * D; idx += 32) {
        const int i = idx % D, j = idx / D;
        if (i >= j) {
            C v = H[idx];
            if (i == j) v.y = R(0);
            A[i + D * j] = v;
            A[j + D * i] = mk(v.x, -v.y);
        }
    }
    __syncwarp();
    GWT_CLK(t_ph0);
    const int r = lane;
    // 1. Householder: A22 <- H A22 H, reflector of step k stored in column k below the diagonal
    bool hh_done = false;
    if constexpr (sizeof(R) == 4 && DM == 32) {
        hh_reg32(D, r, reinterpret_cast<float2*>(A), reinterpret_cast<float2*>(vv), reinterpret_cast<float2*>(ww),
                 reinterpret_cast<float*>(tau), reinterpret_cast<float2*>(sub));
        hh_done = true;
    }
    for (int k = 0; !hh_done && k + 2 < D; ++k) {
        const bool act = r > k && r < D;
        C x = czero<C>();
        if (act) x = A[r + D * k];
        const R t2 = warp_sum_r<R>((r > k + 1 && r < D) ? x.x * x.x + x.y * x.y : R(0));
        const C x0 = shfl_c(x, k + 1);
        if (t2 == R(0)) {  // warp-uniform: column already reduced
            if (lane == 0) {
                tau[k] = R(0);
                sub[k] = x0;
            }
            __syncwarp();
            continue;
        }
        const R ax0 = hypot(x0.x, x0.y);
        const R xnorm = sqrt(t2 + ax0 * ax0);
        const C ph = ax0 > R(0) ? mk(x0.x / ax0, x0.y / ax0) : mk(R(1), R(0));
        const C al = mk(-ph.x * xnorm, -ph.y * xnorm);
        const C v0 = mk(x0.x - al.x, x0.y - al.y);
        const R tk = R(2) / (t2 + v0.x * v0.x + v0.y * v0.y);
        const C v = act ? (r == k + 1 ? v0 : x) : czero<C>();
        if (act) vv[r] = v;
        if (r == k + 1) A[r + D * k] = v0;
        if (lane == 0) {
            tau[k] = tk;
            sub[k] = al;
        }
        __syncwarp();
        // p = tk * A22 v (row r)
        C p0 = czero<C>(), p1 = czero<C>();
        if (act) {
            const C* arow = A + r;
            int c = k + 1;
            for (; c + 3 < D; c += 4) {
                const C a0 = arow[D * c], a1 = arow[D * (c + 1)], a2 = arow[D * (c + 2)], a3 = arow[D * (c + 3)];
                const C b0 = vv[c], b1 = vv[c + 1], b2 = vv[c + 2], b3 = vv[c + 3];
                cfma(p0, a0, b0);
                cfma(p1, a1, b1);
                cfma(p0, a2, b2);
                cfma(p1, a3, b3);
            }
            for (; c < D; ++c) cfma(p0, arow[D * c], vv[c]);
        }
        const C p = mk(tk * (p0.x + p1.x), tk * (p0.y + p1.y));
        const R kk = R(0.5) * tk * warp_sum_r<R>(act ? v.x * p.x + v.y * p.y : R(0));
        const C w = mk(p.x - kk * v.x, p.y - kk * v.y);
        if (act) ww[r] = w;
        __syncwarp();
        // A22 -= v w^H + w v^H (row r; loads of a 4-column batch issued before its stores)
        if (act) {
            C* arow = A + r;
            int c = k + 1;
            for (; c + 3 < D; c += 4) {
                C a[4], vc[4], wc[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    a[u] = arow[D * (c + u)];
                    vc[u] = vv[c + u];
                    wc[u] = ww[c + u];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    a[u].x -= v.x * wc[u].x + v.y * wc[u].y + w.x * vc[u].x + w.y * vc[u].y;
                    a[u].y -= v.y * wc[u].x - v.x * wc[u].y + w.y * vc[u].x - w.x * vc[u].y;
                    arow[D * (c + u)] = a[u];
                }
            }
            for (; c < D; ++c) {
                C a = arow[D * c];
                const C vc = vv[c], wc = ww[c];
                a.x -= v.x * wc.x + v.y * wc.y + w.x * vc.x + w.y * vc.y;
                a.y -= v.y * wc.x - v.x * wc.y + w.y * vc.x - w.x * vc.y;
                arow[D * c] = a;
            }
        }
        __syncwarp();
    }
    GWT_CLK(t_ph1);
    // 2. real symmetric tridiagonal via the diagonal phase similarity
    for (int i = lane; i < D; i += 32) sd[i] = A[i + D * i].x;
    if (lane == 0) {
        C dl = mk(R(1), R(0));
        dlt[0] = dl;
        for (int i = 0; i + 1 < D; ++i) {
            const C s = (i + 2 < D) ? sub[i] : A[(i + 1) + D * i];
            const R mag = hypot(s.x, s.y);
            se[i] = mag;
            se2[i] = mag * mag;
            if (mag > R(0)) dl = cmul(dl, mk(s.x / mag, s.y / mag));
            dlt[i + 1] = dl;
        }
        se[D - 1] = R(0);
        se2[D - 1] = R(0);
    }
    __syncwarp();
    double lo_p = 1e308, hi_p = -1e308, nrm_p = 0.0;
    for (int i = lane; i < D; i += 32) {
        const double rr = (double)(i > 0 ? se[i - 1] : R(0)) + (double)se[i];
        lo_p = fmin(lo_p, (double)sd[i] - rr);
        hi_p = fmax(hi_p, (double)sd[i] + rr);
        nrm_p = fmax(nrm_p, fabs((double)sd[i]) + rr);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo_p = fmin(lo_p, __shfl_xor_sync(0xffffffffu, lo_p, o));
        hi_p = fmax(hi_p, __shfl_xor_sync(0xffffffffu, hi_p, o));
        nrm_p = fmax(nrm_p, __shfl_xor_sync(0xffffffffu, nrm_p, o));
    }
    const double eps = sizeof(R) == 4 ? 1.1920928955078125e-07 : 2.220446049250313e-16;
    const double tnorm = nrm_p;
    const double glo = lo_p - 2.0 * eps * tnorm, ghi = hi_p + 2.0 * eps * tnorm;
    const double inv_n = tnorm > 0.0 ? 1.0 / tnorm : 1.0;
    for (int i = lane; i < D; i += 32) {
        fd[i] = (float)((double)sd[i] * inv_n);
        // fp32 storage: shifted (fe2[i] = e_{i-1}^2) for sturm_count_p32; binary64: as is
        if constexpr (sizeof(R) == 4) fe2[i] = i > 0 ? (float)((double)se2[i - 1] * inv_n * inv_n) : 0.f;
        else fe2[i] = (float)((double)se2[i] * inv_n * inv_n);
    }
    __syncwarp();
    // 3a. multisection: S lanes per wanted eigenvalue (t-th largest = ascending index D-1-t)
    {
        const int S = count <= 8 ? 4 : (count <= 10 ? 3 : (count <= 16 ? 2 : 1));
        const int t = lane / S, s = lane % S;
        const int want = D - 1 - t;
        float lo = (float)(glo * inv_n) - 1e-6f, hi = (float)(ghi * inv_n) + 1e-6f;
        bool done = t >= count;
        for (int it = 0; it < 96; ++it) {
            if (!done && hi - lo <= 2e-7f * fmaxf(fmaxf(fabsf(lo), fabsf(hi)), 1e-3f)) done = true;
            if (__all_sync(0xffffffffu, done)) break;
            const float step = (hi - lo) / (float)(S + 1);
            const float pt = lo + (float)(s + 1) * step;
            const bool le = !done && sturm_count_r<R>(D, fd, fe2, pt) <= want;
            const unsigned bits = __ballot_sync(0xffffffffu, le);
            if (!done) {
                const int j = __popc((bits >> (t * S)) & ((1u << S) - 1u));
                const float nlo = j > 0 ? lo + (float)j * step : lo;
                const float nhi = j < S ? lo + (float)(j + 1) * step : hi;
                if (!(nlo >= lo && nhi <= hi && nlo < nhi) || (nlo == lo && nhi == hi)) done = true;
                else {
                    lo = nlo;
                    hi = nhi;
                }
            }
        }
        if (t < count && s == 0) lamv[t] = 0.5 * ((double)lo + (double)hi) * tnorm;
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
    // 3b. inverse iteration, lane t = eigenvalue t; LU factors [i][t] in shared memory
    const int t = lane;
#define LU_(arr, i) arr[(i) * count + t]
    const R tiny = (R)fmax(eps * tnorm, sizeof(R) == 4 ? 1e-30 : 1e-290);
    // solves from the fp32 bisection shift (~2e-7 rel): 2 reach fp32 accuracy, 3 binary64
    constexpr int kSolves = sizeof(R) == 4 ? GWT_FP32_SOLVES : 3;
    R x[DM];
#pragma unroll
    for (int i = 0; i < DM; ++i) x[i] = R(0);
    for (int rd = 0; rd < rounds; ++rd) {
        if (t < count && scl[t] == rd) {
            const R lam = (R)lamv[t];
            unsigned sw = 0u;
            R dcur = sd[0] - lam, ucur = se[0];
            for (int i = 0; i + 1 < D; ++i) {
                const R sb = se[i], dn = sd[i + 1] - lam, en = (i + 2 < D) ? se[i + 1] : R(0);
                // branch-free partial pivoting (lanes pivot differently; if/else serialised both paths)
                const bool piv = !(fabs(dcur) >= fabs(sb));
                const R di = piv ? sb : (dcur == R(0) ? tiny : dcur);
                const R mult = ii_div(piv ? dcur : sb, di);
                if (piv) sw |= 1u << i;
                LU_(DDv, i) = di;
                LU_(DUv, i) = piv ? dn : ucur;
                const R ndc = piv ? ucur - mult * dn : dn - mult * ucur;
                ucur = piv ? -mult * en : en;
                dcur = ndc;
                LU_(MLv, i) = mult;
            }
            LU_(DDv, D - 1) = dcur;
            for (int i = 0; i < D; ++i) {  // reciprocal pivots (tiny-guarded)
                R di = LU_(DDv, i);
                if (fabs(di) < tiny) di = di < R(0) ? -tiny : tiny;
                LU_(DDv, i) = ii_div(R(1), di);
            }
#pragma unroll
            for (int i = 0; i < DM; ++i) x[i] = i < D ? R(1) + R(0.25) * (R)__sinf(0.7f * i + 1.3f * t) : R(0);
            for (int it = 0; it <= kSolves; ++it) {
                for (int s = t - rd; s < t; ++s) {
                    R dot = R(0);
#pragma unroll
                    for (int i = 0; i < DM; ++i)
                        if (i < D) dot += XR[i * count + s] * x[i];
#pragma unroll
                    for (int i = 0; i < DM; ++i)
                        if (i < D) x[i] -= dot * XR[i * count + s];
                }
                R nn = R(0);
#pragma unroll
                for (int i = 0; i < DM; ++i) nn += x[i] * x[i];
                const R inv = nn > R(0) ? R(1) / sqrt(nn) : R(1);
#pragma unroll
                for (int i = 0; i < DM; ++i) x[i] *= inv;
                if (it == kSolves) break;
                // forward: apply the row interchanges and multipliers
#pragma unroll
                for (int i = 0; i + 1 < DM; ++i) {
                    if (i + 1 < D) {
                        const R ml = LU_(MLv, i);
                        if ((sw >> i) & 1u) {
                            const R t0 = x[i];
                            x[i] = x[i + 1];
                            x[i + 1] = t0 - ml * x[i + 1];
                        } else {
                            x[i + 1] -= ml * x[i];
                        }
                    }
                }
                // back substitution with U (superdiagonals du, du2 = swapped ? e[i+1] : 0)
#pragma unroll
                for (int i = DM - 1; i >= 0; --i) {
                    if (i < D) {
                        R acc = x[i];
                        if (i + 1 < DM && i + 1 < D) acc -= LU_(DUv, i) * x[i + 1];
                        if (i + 2 < DM && i + 2 < D && ((sw >> i) & 1u)) acc -= se[i + 1] * x[i + 2];
                        x[i] = acc * LU_(DDv, i);
                    }
                }
                R mx = R(0);
#pragma unroll
                for (int i = 0; i < DM; ++i) mx = fmax(mx, fabs(x[i]));
                if (!(mx > R(0)) || !isfinite(mx)) {
                    if (fail) atomicExch(fail, 1);
                    break;
                }
                const R sc = ii_div(R(1), mx);
#pragma unroll
                for (int i = 0; i < DM; ++i) x[i] *= sc;
            }
#pragma unroll
            for (int i = 0; i < DM; ++i)
                if (i < D) XR[i * count + t] = x[i];
            double rq = 0.0;  // Rayleigh quotient z^T T z (reported eigenvalue)
#pragma unroll
            for (int i = 0; i < DM; ++i) {
                if (i < D) {
                    double tz = (double)sd[i] * x[i];
                    if (i > 0) tz += (double)se[i - 1] * x[i - 1];
                    if (i + 1 < DM && i + 1 < D) tz += (double)se[i] * x[i + 1];
                    rq += (double)x[i] * tz;
                }
            }
            lamv[t] = rq;
        }
        __syncwarp();
    }
#undef LU_
    GWT_CLK(t_ph3);
    // 4. back-transform y = H_0 ... H_{D-3} diag(delta) z. count <= 16: 2 lanes per eigenvector (rows
    // i = h mod 2, z read from XR, dots combined by one shuffle); else lane = eigenvector.
    if (count <= 16) {
        constexpr int RPT = DM / 2;
        const int tv = lane >> 1, h = lane & 1;
        const bool on = tv < count;
        if (on && h == 0 && evals) evals[b * count + tv] = lamv[tv];
        C y[RPT];
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
            const int i = h + 2 * u;
            y[u] = czero<C>();
            if (on && i < D) {
                const R z = XR[i * count + tv];
                const C dl = dlt[i];
                y[u] = mk(dl.x * z, dl.y * z);
            }
        }
        for (int k = D - 3; k >= 0; --k) {
            const R tk = tau[k];
            if (tk == R(0)) continue;
            C dot = czero<C>();
#pragma unroll
            for (int u = 0; u < RPT; ++u) {
                const int i = h + 2 * u;
                if (i > k && i < D) cfmaconj(dot, A[i + D * k], y[u]);
            }
            dot.x += __shfl_xor_sync(0xffffffffu, dot.x, 1);
            dot.y += __shfl_xor_sync(0xffffffffu, dot.y, 1);
            dot = mk(dot.x * tk, dot.y * tk);
#pragma unroll
            for (int u = 0; u < RPT; ++u) {
                const int i = h + 2 * u;
                if (i > k && i < D) {
                    const C pr = cmul(A[i + D * k], dot);
                    y[u].x -= pr.x;
                    y[u].y -= pr.y;
                }
            }
        }
        R best = R(-1);
        int bi = 0;
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
            const int i = h + 2 * u;
            const R mag = y[u].x * y[u].x + y[u].y * y[u].y;
            if (i < D && mag > best) {
                best = mag;
                bi = i;
            }
        }
        {
            const R ob2 = __shfl_xor_sync(0xffffffffu, best, 1);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, 1);
            if (ob2 > best || (ob2 == best && oi < bi)) {
                best = ob2;
                bi = oi;
            }
        }
        C yb = czero<C>();
#pragma unroll
        for (int u = 0; u < RPT; ++u)
            if (h + 2 * u == bi) yb = y[u];
        yb = shfl_c(yb, (lane & ~1) | (bi & 1));
        if (on) {
            C fac = mk(R(1), R(0));
            if (best > R(0)) {
                const R im = R(1) / sqrt(best);
                fac = mk(yb.x * im, -yb.y * im);
            }
            C* ob = out + (b * count + tv) * (int64_t)D;
#pragma unroll
            for (int u = 0; u < RPT; ++u) {
                const int i = h + 2 * u;
                if (i < D) ob[i] = cmul(y[u], fac);
            }
        }
    } else if (t < count) {
        if (evals) evals[b * count + t] = lamv[t];
        C y[DM];
#pragma unroll
        for (int i = 0; i < DM; ++i) {
            y[i] = czero<C>();
            if (i < D) {
                const C dl = dlt[i];
                y[i] = mk(dl.x * x[i], dl.y * x[i]);
            }
        }
        for (int k = D - 3; k >= 0; --k) {
            const R tk = tau[k];
            if (tk == R(0)) continue;
            C dot = czero<C>();
#pragma unroll
            for (int i = 0; i < DM; ++i)
                if (i > k && i < D) cfmaconj(dot, A[i + D * k], y[i]);
            dot = mk(dot.x * tk, dot.y * tk);
#pragma unroll
            for (int i = 0; i < DM; ++i) {
                if (i > k && i < D) {
                    const C pr = cmul(A[i + D * k], dot);
                    y[i].x -= pr.x;
                    y[i].y -= pr.y;
                }
            }
        }
        R best = R(-1);
        C yb = czero<C>();
#pragma unroll
        for (int i = 0; i < DM; ++i) {
            const R mag = y[i].x * y[i].x + y[i].y * y[i].y;
            if (i < D && mag > best) {
                best = mag;
                yb = y[i];
            }
        }
        C fac = mk(R(1), R(0));
        if (best > R(0)) {
            const R im = R(1) / sqrt(best);
            fac = mk(yb.x * im, -yb.y * im);
        }
        C* ob = out + (b * count + t) * (int64_t)D;
#pragma unroll
        for (int i = 0; i < DM; ++i)
            if (i < D) ob[i] = cmul(y[i], fac);
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
}

