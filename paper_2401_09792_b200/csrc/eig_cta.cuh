// CTA-per-matrix Hermitian top-k eigensolver for 32 < D <= DM (DM = 64 or 128), in the storage
// precision R, matrix resident in shared memory. Included by k_eig.cu (inside namespace gwtk).
//
// Same algorithm and conventions as k_heev_wr / k_heev_topk (reference leading_eigenvectors,
// proj/src/linalg.cpp:27-45 + phase_normalize_columns :11-25):
//  1. Householder tridiagonalisation with Q = 256/DM adjacent threads per row (columns split
//     mod Q, combined by shuffles), 2 CTA barriers per reflector, every thread forms the
//     reflector scalars itself (no single-thread serial section).
//  2. fp32 multisection on Sturm counts (S = 1..8 lanes per wanted eigenvalue).
//  3. Inverse iteration, one thread per eigenvalue, iterate in registers, LU in shared memory.
//  4. Back-transform with 4 threads per eigenvector (rows split mod 4, shuffle-reduced dots).
#pragma once

struct EigCtaLayout {
    size_t oA, ov, ow, otau, osub, odl, od, oe, oe2, ofd, ofe2, olam, oscl, ored, odd, odu, oml, oxr, total;
    int lda;
};

__host__ __device__ inline EigCtaLayout eig_cta_layout(int D, int count, int rs) {
    EigCtaLayout L;
    // float2 with 4 threads per row (D <= 64): column stride = 16 banks -> 2 wavefronts per warp access
    L.lda = (rs == 4 && D <= 64) ? D + 8 : D;
    size_t o = 0;
    const size_t cs = 2 * (size_t)rs;
#define GWT_TAKE(field, bytes)          \
    L.field = o;                        \
    o = (o + (bytes) + 15) & ~size_t(15);
    GWT_TAKE(oA, (size_t)L.lda * D * cs)
    GWT_TAKE(ov, D * cs)
    GWT_TAKE(ow, D * cs)
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
    GWT_TAKE(ored, 4 * 8 * 8)
    GWT_TAKE(odd, (size_t)D * count * rs)
    L.odu = o;  // no stored U superdiagonal: recomputed in the back substitution (k_heev_cr)
    GWT_TAKE(oml, (size_t)D * count * rs)
    GWT_TAKE(oxr, (size_t)D * count * rs)
#undef GWT_TAKE
    L.total = o;
    return L;
}

// sum over the lanes q == 0 of each Q-lane row group (values of the other lanes must be 0 or equal
// across the group's lanes are ignored by construction): log2(32/Q) shuffle levels, result in lane 0
template <int Q, class R>
__device__ __forceinline__ R rows_sum(R v) {
#pragma unroll
    for (int o = Q; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// back-transform y = H_0 ... H_{D-3} diag(delta) z with QB threads per eigenvector (rows i = qb mod QB),
// phase normalisation, store (shared by k_heev_cr's two thread-per-vector configurations)
template <class R, int DM, int QB>
__device__ __forceinline__ void cta_backtransform(int D, int count, int LD, int64_t b, const cplx_t<R>* A,
                                                  const R* XR, const cplx_t<R>* dlt, const R* tau, const double* lamv,
                                                  double* evals, cplx_t<R>* out) {
    using C = cplx_t<R>;
    const int tid = threadIdx.x, lane = tid % 32;
{
        constexpr int RPT = DM / QB;
        const int t = tid / QB, qb = tid % QB;
        const bool on = t < count;  // count <= 64 (host-checked)
        if (on && qb == 0 && evals) evals[b * count + t] = lamv[t];
        C y[RPT];
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
            const int i = qb + QB * u;
            y[u] = czero<C>();
            if (on && i < D) {
                const R z = XR[i * count + t];
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
                const int i = qb + QB * u;
                if (i > k && i < D) cfmaconj(dot, A[i + LD * k], y[u]);
            }
#pragma unroll
            for (int o = 1; o < QB; o <<= 1) {
                dot.x += __shfl_xor_sync(0xffffffffu, dot.x, o);
                dot.y += __shfl_xor_sync(0xffffffffu, dot.y, o);
            }
            dot = mk(dot.x * tk, dot.y * tk);
#pragma unroll
            for (int u = 0; u < RPT; ++u) {
                const int i = qb + QB * u;
                if (i > k && i < D) {
                    const C pr = cmul(A[i + LD * k], dot);
                    y[u].x -= pr.x;
                    y[u].y -= pr.y;
                }
            }
        }
        R best = R(-1);
        int bi = 0;
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
            const int i = qb + QB * u;
            const R mag = y[u].x * y[u].x + y[u].y * y[u].y;
            if (i < D && mag > best) {
                best = mag;
                bi = i;
            }
        }
#pragma unroll
        for (int o = 1; o < QB; o <<= 1) {
            const R ob2 = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ob2 > best || (ob2 == best && oi < bi)) {
                best = ob2;
                bi = oi;
            }
        }
        // the owner of row bi broadcasts y[bi]
        C yb = czero<C>();
#pragma unroll
        for (int u = 0; u < RPT; ++u)
            if (qb + QB * u == bi) yb = y[u];
        const int owner = (lane & ~(QB - 1)) | (bi % QB);
        yb = shfl_c(yb, owner);
        if (on) {
            C fac = mk(R(1), R(0));
            if (best > R(0)) {
                const R im = R(1) / sqrt(best);
                fac = mk(yb.x * im, -yb.y * im);
            }
            C* ob = out + (b * count + t) * (int64_t)D;
#pragma unroll
            for (int u = 0; u < RPT; ++u) {
                const int i = qb + QB * u;
                if (i < D) ob[i] = cmul(y[u], fac);
            }
        }
    }
}

// Register-resident Householder for fp32 storage, 32 < D <= 64, 256 threads (phase 1 of k_heev_cr
// with HREG, used for small batches where the per-matrix latency is the critical path: C2's tx
// Grams, 193k -> 177k cycles; its 134 registers cost occupancy on the large delay batches of C3/C5):
// thread (r, q) keeps A[r][q + 4u] (u < 16) in registers. The shared-memory matrix only receives
// the column that becomes the next reflector (written by its owners during the update) plus the
// diagonal at the end, so a step reads the reflector column and p by broadcast instead of
// reading and writing the whole trailing matrix (the old form was shared-pipe bound).
__device__ __forceinline__ void hh_cta_reg64(int D, int LD, float2* A, float2* pp, float* tau, float2* sub,
                                             float* rt2, float* rkp) {
    constexpr int Q = 4, NW = 8, U = 16;
    const int tid = threadIdx.x, lane = tid % 32, wid = tid / 32;
    const int r = tid / Q, q = tid % Q;
    float2 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int c = q + Q * u;
        a[u] = (r < D && c < D) ? A[r + LD * c] : make_float2(0.f, 0.f);
    }
    {
        float part = 0.f;
        if (q == 0 && r > 1 && r < D) {
            const float2 x = A[r];
            part = x.x * x.x + x.y * x.y;
        }
        part = rows_sum<Q>(part);
        if (lane == 0) rt2[wid] = part;
    }
    for (int k = 0; k + 2 < D; ++k) {
        const bool act = r > k && r < D;
        __syncthreads();  // [A] column k and its norm partials are in shared memory
        float t2 = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) t2 += rt2[w];
        const float2* colk = A + LD * k;
        const float2 x0 = colk[k + 1];
        const int kn = k + 1, qn = kn % Q, un = kn / Q;  // owner of column k+1
        if (t2 == 0.f) {  // uniform: column already reduced
            if (tid == 0) {
                tau[k] = 0.f;
                sub[k] = x0;
            }
            __syncthreads();  // rt2 reads done
            float2 xn = make_float2(0.f, 0.f);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (u == un) xn = a[u];
            float part = 0.f;
            if (q == qn && r < D) {
                A[r + LD * kn] = xn;
                if (r > kn + 1) part = xn.x * xn.x + xn.y * xn.y;
            }
            part = __shfl_sync(0xffffffffu, rows_sum<Q>(part), qn);  // the owner lanes hold the partials
            if (lane == 0) rt2[wid] = part;
            continue;
        }
        float2 al, v0;
        float tk;
        reflector(x0, t2, al, v0, tk);
        const float2 v = act ? (r == k + 1 ? v0 : colk[r]) : make_float2(0.f, 0.f);
        float2 vc[U];
        float2 p0 = make_float2(0.f, 0.f), p1 = make_float2(0.f, 0.f);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int c = q + Q * u;
            // unconditional load (c < 64 stays inside the shared matrix: LD*(D-3) + 63 < LD*D), then
            // selects: the predicated load compiled to per-column branches (ncu: branch_resolving stalls)
            const float2 ck = colk[c];
            vc[u] = (c > k && c < D) ? (c == k + 1 ? v0 : ck) : make_float2(0.f, 0.f);
            if (u & 1) cfma(p1, a[u], vc[u]);
            else cfma(p0, a[u], vc[u]);
        }
        float2 p = make_float2(p0.x + p1.x, p0.y + p1.y);
#pragma unroll
        for (int o = 1; o < Q; o <<= 1) {
            p.x += __shfl_xor_sync(0xffffffffu, p.x, o);
            p.y += __shfl_xor_sync(0xffffffffu, p.y, o);
        }
        p = make_float2(p.x * tk, p.y * tk);
        float kp = (q == 0 && act) ? v.x * p.x + v.y * p.y : 0.f;
        kp = rows_sum<Q>(kp);
        if (lane == 0) rkp[wid] = kp;
        if (act && q == 0) pp[r] = p;
        __syncthreads();  // [B]
        float ks = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) ks += rkp[w];
        const float kk = 0.5f * tk * ks;
        const float2 w = act ? make_float2(p.x - kk * v.x, p.y - kk * v.y) : make_float2(0.f, 0.f);
        if (tid == 0) {
            tau[k] = tk;
            sub[k] = al;
        }
        float2 xn = make_float2(0.f, 0.f);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int c = q + Q * u;
            const float2 pc = pp[c];  // unconditional (inside the shared-memory layout), masked below
            const float2 wc = (c > k && c < D) ? make_float2(pc.x - kk * vc[u].x, pc.y - kk * vc[u].y)
                                                : make_float2(0.f, 0.f);
            // a[r][c] -= v_r conj(w_c) + w_r conj(v_c)
            a[u].x -= v.x * wc.x + v.y * wc.y + w.x * vc[u].x + w.y * vc[u].y;
            a[u].y -= v.y * wc.x - v.x * wc.y + w.y * vc[u].x - w.x * vc[u].y;
            if (u == un) xn = a[u];
        }
        float part = 0.f;
        if (q == qn && r < D) {  // next column to shared memory (next reflector) + its norm partials
            A[r + LD * kn] = xn;
            if (r > kn + 1) part = xn.x * xn.x + xn.y * xn.y;
        }
        if (r == k + 1 && q == 0) A[r + LD * k] = v0;  // store the reflector (x0 no longer read)
        part = __shfl_sync(0xffffffffu, rows_sum<Q>(part), qn);  // the owner lanes hold the partials
        if (lane == 0) rt2[wid] = part;  // rt2 of step k was consumed before [B]
    }
    // diagonal back to shared memory (phase 2 reads it there)
    float2 dg = make_float2(0.f, 0.f);
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (q + Q * u == r) dg = a[u];
    if (r < D && (r % Q) == q) A[r + LD * r] = dg;
    __syncthreads();
}

template <class R, int DM, int NT, bool HREG = false>
__global__ void __launch_bounds__(NT, (sizeof(R) == 8 && DM == 64) ? 2 : 256 / NT) k_heev_cr(int D, int count, const cplx_t<R>* __restrict__ in,
                                                          cplx_t<R>* __restrict__ out, double* __restrict__ evals,
                                                          int* __restrict__ fail) {
    using C = cplx_t<R>;
    constexpr int Q = NT / DM, NW = NT / 32;
    extern __shared__ __align__(16) unsigned char smem_dyn[];
    const int tid = threadIdx.x, lane = tid % 32, wid = tid / 32;
    const int64_t b = blockIdx.x;
    const EigCtaLayout L = eig_cta_layout(D, count, sizeof(R));
    const int LD = L.lda;
    unsigned char* base = smem_dyn;
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
    double* red = reinterpret_cast<double*>(base + L.ored);  // [4 slots][NW]
    R* DDv = reinterpret_cast<R*>(base + L.odd);
    R* MLv = reinterpret_cast<R*>(base + L.oml);
    R* XR = reinterpret_cast<R*>(base + L.oxr);
    const C* H = in + b * (int64_t)D * D;
    for (int idx = tid; idx < D * D; idx += NT) {
        const int i = idx % D, j = idx / D;
        if (i >= j) {
            C v = H[idx];
            if (i == j) v.y = R(0);
            A[i + LD * j] = v;
            A[j + LD * i] = mk(v.x, -v.y);
        }
    }
    __syncthreads();
    GWT_CLK(t_ph0);
    const int r = tid / Q, q = tid % Q;
    // 1. Householder, two CTA barriers per reflector:
    //   [A] column-k norm partials visible -> every thread forms (alpha, tau, v0); p = tau A22 v
    //       reading v straight from column k (v0 substituted for row k+1); publish p and v^H p partials
    //   [B] K = tau/2 v^H p; A22 -= v w^H + w v^H with w = p - K v; the updated column k+1
    //       yields the next step's norm partials (published before the next [A]).
    R* rt2 = reinterpret_cast<R*>(red);       // [NW] norm partials of the current column
    R* rkp = rt2 + NW;                        // [NW] v^H p partials
    C* pp = vv;              // p of the current step
    bool hh_done = false;
    if constexpr (HREG && sizeof(R) == 4 && DM == 64 && NT == 256) {
        hh_cta_reg64(D, LD, reinterpret_cast<float2*>(A), reinterpret_cast<float2*>(pp), reinterpret_cast<float*>(tau),
                     reinterpret_cast<float2*>(sub), reinterpret_cast<float*>(rt2), reinterpret_cast<float*>(rkp));
        hh_done = true;
    }
    if (!hh_done) {
        R part = R(0);
        if (q == 0 && r > 1 && r < D) {
            const C a = A[r];
            part = a.x * a.x + a.y * a.y;
        }
        part = rows_sum<Q>(part);
        if (lane == 0) rt2[wid] = part;
    }
    for (int k = 0; !hh_done && k + 2 < D; ++k) {
        const bool act = r > k && r < D;
        __syncthreads();  // [A]
        R t2 = R(0);
#pragma unroll
        for (int w = 0; w < NW; ++w) t2 += rt2[w];
        const C x0 = A[(k + 1) + LD * k];
        const C* colk = A + LD * k;
        if (t2 == R(0)) {  // uniform: column already reduced; next column's partials
            if (tid == 0) {
                tau[k] = R(0);
                sub[k] = x0;
            }
            __syncthreads();  // all reads of rt2 done before it is rewritten
            R part = R(0);
            if (q == 0 && r > k + 2 && r < D) {
                const C a = A[r + LD * (k + 1)];
                part = a.x * a.x + a.y * a.y;
            }
            part = rows_sum<Q>(part);
            if (lane == 0) rt2[wid] = part;
            continue;
        }
        C al, v0;
        R tk;
        reflector(x0, t2, al, v0, tk);
        const C v = act ? (r == k + 1 ? v0 : colk[r]) : czero<C>();
        C p0 = czero<C>(), p1 = czero<C>();
        if (act) {
            // columns c = k+1+q, +Q, ...; 4-column batches with all loads issued first
            const C* arow = A + r;
            int c = k + 1 + q;
            for (; c + 3 * Q < D; c += 4 * Q) {
                C a[4], b[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    a[u] = arow[LD * (c + u * Q)];
                    b[u] = colk[c + u * Q];
                }
                if (c == k + 1) b[0] = v0;  // the reflector's first entry is v0, not the stored x0
                cfma(p0, a[0], b[0]);
                cfma(p1, a[1], b[1]);
                cfma(p0, a[2], b[2]);
                cfma(p1, a[3], b[3]);
            }
            for (; c < D; c += Q) cfma(p0, arow[LD * c], c == k + 1 ? v0 : colk[c]);
        }
        C p = mk(p0.x + p1.x, p0.y + p1.y);
#pragma unroll
        for (int o = 1; o < Q; o <<= 1) {
            p.x += __shfl_xor_sync(0xffffffffu, p.x, o);
            p.y += __shfl_xor_sync(0xffffffffu, p.y, o);
        }
        p = mk(p.x * tk, p.y * tk);
        R kp = (q == 0 && act) ? v.x * p.x + v.y * p.y : R(0);
        kp = rows_sum<Q>(kp);
        if (lane == 0) rkp[wid] = kp;
        if (act && q == 0) pp[r] = p;
        __syncthreads();  // [B]
        R ks = R(0);
#pragma unroll
        for (int w = 0; w < NW; ++w) ks += rkp[w];
        const R kk = R(0.5) * tk * ks;
        const C w = mk(p.x - kk * v.x, p.y - kk * v.y);
        if (tid == 0) {
            tau[k] = tk;
            sub[k] = al;
        }
        R part = R(0);
        if (act) {
            // a[r][c] -= v_r conj(w_c) + w_r conj(v_c),  w_c = p_c - K v_c
            C* arow = A + r;
            int c = k + 1 + q;
            for (; c + 3 * Q < D; c += 4 * Q) {
                C a[4], vc[4], pc[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    a[u] = arow[LD * (c + u * Q)];
                    vc[u] = colk[c + u * Q];
                    pc[u] = pp[c + u * Q];
                }
                if (c == k + 1) vc[0] = v0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const C wc = mk(pc[u].x - kk * vc[u].x, pc[u].y - kk * vc[u].y);
                    a[u].x -= v.x * wc.x + v.y * wc.y + w.x * vc[u].x + w.y * vc[u].y;
                    a[u].y -= v.y * wc.x - v.x * wc.y + w.y * vc[u].x - w.x * vc[u].y;
                    arow[LD * (c + u * Q)] = a[u];
                }
                if (c == k + 1 && r > k + 2) part = a[0].x * a[0].x + a[0].y * a[0].y;
            }
            for (; c < D; c += Q) {
                const C vc = c == k + 1 ? v0 : colk[c];
                const C pc = pp[c];
                const C wc = mk(pc.x - kk * vc.x, pc.y - kk * vc.y);
                C a = arow[LD * c];
                a.x -= v.x * wc.x + v.y * wc.y + w.x * vc.x + w.y * vc.y;
                a.y -= v.y * wc.x - v.x * wc.y + w.y * vc.x - w.x * vc.y;
                arow[LD * c] = a;
                if (c == k + 1 && r > k + 2) part = a.x * a.x + a.y * a.y;
            }
            if (r == k + 1 && q == 0) A[r + LD * k] = v0;  // store the reflector (x0 no longer read)
        }
        part = rows_sum<Q>(part);
        if (lane == 0) rt2[wid] = part;  // rt2 of step k was consumed before [B]
    }
    __syncthreads();
    GWT_CLK(t_ph1);
    // 2. real symmetric tridiagonal via the diagonal phase similarity
    for (int i = tid; i < D; i += NT) sd[i] = A[i + LD * i].x;
    if (tid == 0) {
        C dl = mk(R(1), R(0));
        dlt[0] = dl;
        for (int i = 0; i + 1 < D; ++i) {
            const C s = (i + 2 < D) ? sub[i] : A[(i + 1) + LD * i];
            const R mag = hypot(s.x, s.y);
            se[i] = mag;
            se2[i] = mag * mag;
            if (mag > R(0)) dl = cmul(dl, mk(s.x / mag, s.y / mag));
            dlt[i + 1] = dl;
        }
        se[D - 1] = R(0);
        se2[D - 1] = R(0);
    }
    __syncthreads();
    double lo_p = 1e308, hi_p = -1e308, nrm_p = 0.0;
    for (int i = tid; i < D; i += NT) {
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
    if (lane == 0) {
        red[wid] = lo_p;
        red[NW + wid] = hi_p;
        red[2 * NW + wid] = nrm_p;
    }
    __syncthreads();
    double glo = 1e308, ghi = -1e308, tnorm = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        glo = fmin(glo, red[w]);
        ghi = fmax(ghi, red[NW + w]);
        tnorm = fmax(tnorm, red[2 * NW + w]);
    }
    const double eps = sizeof(R) == 4 ? 1.1920928955078125e-07 : 2.220446049250313e-16;
    glo -= 2.0 * eps * tnorm;
    ghi += 2.0 * eps * tnorm;
    const double inv_n = tnorm > 0.0 ? 1.0 / tnorm : 1.0;
    for (int i = tid; i < D; i += NT) {
        fd[i] = (float)((double)sd[i] * inv_n);
        // fp32 storage: shifted (fe2[i] = e_{i-1}^2) for sturm_count_p32; binary64: as is
        if constexpr (sizeof(R) == 4) fe2[i] = i > 0 ? (float)((double)se2[i - 1] * inv_n * inv_n) : 0.f;
        else fe2[i] = (float)((double)se2[i] * inv_n * inv_n);
    }
    __syncthreads();
    // 3a. multisection, S lanes (power of two, within one warp) per wanted eigenvalue
    {
        int S = NT / count;
        S = S >= 8 ? 8 : (S >= 4 ? 4 : (S >= 2 ? 2 : 1));
        const int t = tid / S, s = tid % S;
        const int gl = lane / S;  // group index inside the warp
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
                const int j = __popc((bits >> (gl * S)) & ((S == 32 ? 0u : (1u << S)) - 1u));
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
    __syncthreads();
    if constexpr (sizeof(R) == 8) {
        // 3a'. binary64 storage: refine each eigenvalue by binary64 multisection inside a bracket around the
        // fp32 estimate (checked, else the Gershgorin interval). With shifts accurate to ~eps64 ||T|| the
        // inverse iterations only need joint orthogonalisation for eigenvalues closer than 1e-9 ||T||
        // (the fp32 shifts forced it below 1e-3 ||T||: for the graded delay-mode spectra, p_q ~ e^-0.3q,
        // most kept eigenvalues formed one cluster and were solved one after another).
        int S = NT / count;
        S = S >= 8 ? 8 : (S >= 4 ? 4 : (S >= 2 ? 2 : 1));
        const int t = tid / S, s = tid % S;
        const int gl = lane / S;
        const int want = D - 1 - t;
        bool done = t >= count;
        const double lam0 = done ? 0.0 : lamv[t];
        double lo = lam0 - 4e-6 * tnorm, hi = lam0 + 4e-6 * tnorm;
        if (!done && !(sturm_count_f64(D, (const double*)sd, (const double*)se2, lo) <= want &&
                       sturm_count_f64(D, (const double*)sd, (const double*)se2, hi) > want)) {
            lo = glo;
            hi = ghi;
        }
        for (int it = 0; it < 80; ++it) {
            if (!done && hi - lo <= 8.0 * 2.220446049250313e-16 * fmax(fmax(fabs(lo), fabs(hi)), 1e-14 * tnorm))
                done = true;
            if (__all_sync(0xffffffffu, done)) break;
            const double step = (hi - lo) / (double)(S + 1);
            const double pt = lo + (double)(s + 1) * step;
            const bool le = !done && sturm_count_f64(D, (const double*)sd, (const double*)se2, pt) <= want;
            const unsigned bits = __ballot_sync(0xffffffffu, le);
            if (!done) {
                const int j = __popc((bits >> (gl * S)) & ((S == 32 ? 0u : (1u << S)) - 1u));
                const double nlo = j > 0 ? lo + (double)j * step : lo;
                const double nhi = j < S ? lo + (double)(j + 1) * step : hi;
                if (!(nlo >= lo && nhi <= hi && nlo < nhi) || (nlo == lo && nhi == hi)) done = true;
                else {
                    lo = nlo;
                    hi = nhi;
                }
            }
        }
        if (t < count && s == 0) lamv[t] = 0.5 * (lo + hi);
        __syncthreads();
    }
    __shared__ int s_rounds;
    if (tid == 0) {
        const double ctol = (sizeof(R) == 8 ? 1e-9 : 1e-3) * fmax(tnorm, 1e-300);
        int pos = 0, maxr = 0;
        for (int t = 0; t < count; ++t) {
            pos = (t > 0 && fabs(lamv[t - 1] - lamv[t]) <= ctol) ? pos + 1 : 0;
            scl[t] = pos;
            maxr = max(maxr, pos);
        }
        s_rounds = maxr + 1;
    }
    __syncthreads();
    const int rounds = s_rounds;
    GWT_CLK(t_ph2);
    // 3b. inverse iteration, thread t = eigenvalue t; the iterate lives in XR[i][t] (shared memory,
    // conflict free across t) so the thread keeps no D-long register array
    {
        const int t = tid;
#define LU_(arr, i) arr[(i) * count + t]
#define XV(i) XR[(i) * count + t]
        const R tiny = (R)fmax(eps * tnorm, sizeof(R) == 4 ? 1e-30 : 1e-290);
        // solves from the fp32 bisection shift (~2e-7 rel): 2 reach fp32 accuracy, 3 binary64
        constexpr int kSolves = sizeof(R) == 4 ? GWT_FP32_SOLVES : 3;
        for (int rd = 0; rd < rounds; ++rd) {
            if (t < count && scl[t] == rd) {
                const R lam = (R)lamv[t];
                uint32_t sw[DM / 32];
#pragma unroll
                for (int w2 = 0; w2 < DM / 32; ++w2) sw[w2] = 0u;
                R dcur = sd[0] - lam, ucur = se[0];
                for (int i = 0; i + 1 < D; ++i) {
                    const R sb = se[i], dn = sd[i + 1] - lam, en = (i + 2 < D) ? se[i + 1] : R(0);
                    // branch-free partial pivoting (the threads of a warp pivot differently: the
                    // if/else form serialised both paths)
                    const bool piv = !(fabs(dcur) >= fabs(sb));
                    const R di = piv ? sb : (dcur == R(0) ? tiny : dcur);
                    const R mult = ii_div(piv ? dcur : sb, di);
                    if (piv) sw[i >> 5] |= 1u << (i & 31);
                    LU_(DDv, i) = di;
                    const R ndc = piv ? ucur - mult * dn : dn - mult * ucur;
                    ucur = piv ? -mult * en : en;
                    dcur = ndc;
                    LU_(MLv, i) = mult;
                }
                LU_(DDv, D - 1) = dcur;
                for (int i = 0; i < D; ++i) {
                    R di = LU_(DDv, i);
                    if (fabs(di) < tiny) di = di < R(0) ? -tiny : tiny;
                    LU_(DDv, i) = ii_div(R(1), di);
                }
                for (int i = 0; i < D; ++i) XV(i) = R(1) + R(0.25) * (R)__sinf(0.7f * i + 1.3f * t);
                for (int it = 0; it <= kSolves; ++it) {
                    for (int s2 = t - rd; s2 < t; ++s2) {
                        R dot = R(0);
                        for (int i = 0; i < D; ++i) dot += XR[i * count + s2] * XV(i);
                        for (int i = 0; i < D; ++i) XV(i) -= dot * XR[i * count + s2];
                    }
                    R nn = R(0);
                    for (int i = 0; i < D; ++i) nn += XV(i) * XV(i);
                    const R inv = nn > R(0) ? R(1) / sqrt(nn) : R(1);
                    for (int i = 0; i < D; ++i) XV(i) *= inv;
                    if (it == kSolves) break;
                    R xi = XV(0);  // forward: row interchanges and multipliers, carried in registers
                    for (int i = 0; i + 1 < D; ++i) {
                        const R ml = LU_(MLv, i), xn = XV(i + 1);
                        const bool swp = (sw[i >> 5] >> (i & 31)) & 1u;
                        XV(i) = swp ? xn : xi;
                        xi = swp ? xi - ml * xn : xn - ml * xi;
                    }
                    XV(D - 1) = xi;
                    R x1 = R(0), x2 = R(0);  // back substitution with U, x[i+1], x[i+2] in registers
                    for (int i = D - 1; i >= 0; --i) {
                        R acc = XV(i);
                        const bool pvi = (sw[i >> 5] >> (i & 31)) & 1u;
                        if (i + 1 < D) {
                            // U's first superdiagonal as the factorisation formed it: d_{i+1} - lam after a row
                            // interchange, else the carried entry (e_0; -m_{i-1} e_i after an interchange at
                            // i - 1; e_i otherwise)
                            const bool pvm = i > 0 && ((sw[(i - 1) >> 5] >> ((i - 1) & 31)) & 1u);
                            const R du = pvi ? sd[i + 1] - lam : (pvm ? -LU_(MLv, i - 1) * se[i] : se[i]);
                            acc -= du * x1;
                        }
                        const R u2 = (i + 2 < D && pvi) ? se[i + 1] : R(0);
                        acc -= u2 * x2;
                        const R v = acc * LU_(DDv, i);
                        XV(i) = v;
                        x2 = x1;
                        x1 = v;
                    }
                    R mx = R(0);
                    for (int i = 0; i < D; ++i) mx = fmax(mx, fabs(XV(i)));
                    if (!(mx > R(0)) || !isfinite(mx)) {
                        if (fail) atomicExch(fail, 1);
                        break;
                    }
                    const R sc = ii_div(R(1), mx);
                    for (int i = 0; i < D; ++i) XV(i) *= sc;
                }
                double rq = 0.0;
                for (int i = 0; i < D; ++i) {
                    double tz = (double)sd[i] * XV(i);
                    if (i > 0) tz += (double)se[i - 1] * XV(i - 1);
                    if (i + 1 < D) tz += (double)se[i] * XV(i + 1);
                    rq += (double)XV(i) * tz;
                }
                lamv[t] = rq;
            }
            __syncthreads();
        }
#undef LU_
#undef XV
    }
    GWT_CLK(t_ph3);
    // 4. back-transform: 8 threads per eigenvector when count <= NT/8, else 4
    if (count * 8 <= NT) cta_backtransform<R, DM, 8>(D, count, LD, b, A, XR, dlt, tau, lamv, evals, out);
    else cta_backtransform<R, DM, 4>(D, count, LD, b, A, XR, dlt, tau, lamv, evals, out);
#ifdef GWT_PHASE_TIMERS
    if (b == 0 && tid == 0) {
        const long long t_ph4 = clock64();
        g_eig_phase[0] = t_ph1 - t_ph0;
        g_eig_phase[1] = t_ph2 - t_ph1;
        g_eig_phase[2] = t_ph3 - t_ph2;
        g_eig_phase[3] = t_ph4 - t_ph3;
    }
#endif
}
