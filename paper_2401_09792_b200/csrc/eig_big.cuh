// CTA-per-matrix Hermitian top-k eigensolver for 64 < D <= 256 in fp32 (c64 Grams, e.g. the C4
// transmit factor, N = 256). Included by k_eig.cu (inside namespace gwtk) after eig_cta.cuh.
//
// Same algorithm and conventions as k_heev_cr (reference leading_eigenvectors,
// proj/src/linalg.cpp:27-45 + phase_normalize_columns :11-25). The 256x256 complex64 matrix
// (512 KB) does not fit in shared memory, so it lives in the per-matrix global workspace where
// it stays L2-resident (148 concurrent matrices = 76 MB of the 126 MB L2); everything on the
// serial chains is in shared memory or registers:
//  1. Householder in panels of kPanel reflectors (the LAPACK latrd / her2k split): inside a panel the
//     trailing matrix is not rewritten; each step reads it once (p = A v, 16 loads in flight per
//     thread) and corrects with the panel's V, W columns held in shared memory
//     (p -= V (W^H v) + W (V^H v)); one rank-2*kPanel update per panel (4x4 register tiles) then
//     rewrites the trailing matrix. The per-reflector read-modify-write of the whole trailing matrix
//     (the old form: two L2 passes + one write per step, latency bound) is gone.
//  2. fp32 multisection on Sturm counts (8 lanes per wanted eigenvalue).
//  3. Inverse iteration, thread per eigenvalue, iterate in shared memory ([i][t], conflict free),
//     pivoted LU in the global workspace (L1-resident per thread column).
//  4. Back-transform with 8 threads per eigenvector (32 rows each in registers), vectors in
//     batches of 64 (counts up to 128: the C5 rank sweep n = 96); the reflectors are staged into
//     shared memory 32 at a time (zero-padded, so the apply loop runs unpredicated).
#pragma once

constexpr int kBigNT = 512;
constexpr int kPanel = 32;

__host__ __device__ inline size_t eig_big_region(int D, int count) {
    // union of the Householder panel (V, W: kPanel columns each) and the iterate XR [i][t] + the
    // back-transform staging of kPanel reflectors
    const size_t vw = (size_t)2 * kPanel * D * 8;
    const size_t xs = (((size_t)D * count * 4 + 15) & ~size_t(15)) + (size_t)kPanel * D * 8;
    return vw > xs ? vw : xs;
}

__host__ __device__ inline size_t eig_big_smem(int D, int count) {
    // tau, sub, dlt, sd, se, se2, fd, fe2, pA, lam, scl, red, xy, region
    return (size_t)D * (4 + 8 + 8 + 4 + 4 + 4 + 4 + 4 + 8) + (size_t)count * (8 + 4) + 2 * 16 * 8 + 2 * kPanel * 8 +
           eig_big_region(D, count) + 16 * 16;
}

__global__ void __launch_bounds__(kBigNT, 1) k_heev_big(int D, int count, double ctol_rel, const float2* __restrict__ in,
                                                        float2* __restrict__ out, double* __restrict__ evals,
                                                        float2* __restrict__ ws_a, float* __restrict__ ws_lu,
                                                        int* __restrict__ fail) {
    using R = float;
    using C = float2;
    constexpr int NT = kBigNT, DM = 256, Q = NT / DM, NW = NT / 32;
    extern __shared__ __align__(16) unsigned char smem_dyn[];
    const int tid = threadIdx.x, lane = tid % 32, wid = tid / 32;
    const int64_t b = blockIdx.x;
    const int LD = D;
    // shared carve-up
    unsigned char* p = smem_dyn;
    auto take = [&](size_t bytes) {
        unsigned char* r = p;
        p += (bytes + 15) & ~size_t(15);
        return r;
    };
    R* tau = reinterpret_cast<R*>(take((size_t)D * 4));
    C* sub = reinterpret_cast<C*>(take((size_t)D * 8));
    C* dlt = reinterpret_cast<C*>(take((size_t)D * 8));
    R* sd = reinterpret_cast<R*>(take((size_t)D * 4));
    R* se = reinterpret_cast<R*>(take((size_t)D * 4));
    R* se2 = reinterpret_cast<R*>(take((size_t)D * 4));
    float* fd = reinterpret_cast<float*>(take((size_t)D * 4));
    float* fe2 = reinterpret_cast<float*>(take((size_t)D * 4));
    double* lamv = reinterpret_cast<double*>(take((size_t)count * 8));
    int* scl = reinterpret_cast<int*>(take((size_t)count * 4));
    R* red = reinterpret_cast<R*>(take(2 * 16 * 8));
    C* xy = reinterpret_cast<C*>(take(2 * kPanel * 8));  // W^H v, V^H v of the current step
    C* pA = reinterpret_cast<C*>(take((size_t)D * 8));   // A v of the current step
    unsigned char* region = take(eig_big_region(D, count));
    C* Vp = reinterpret_cast<C*>(region);                       // [kPanel][D] panel reflectors
    C* Wp = Vp + (size_t)kPanel * D;                            // [kPanel][D] panel w vectors
    R* XR = reinterpret_cast<R*>(region);                       // [i][t] iterate / final z (after phase 1)
    C* Sg = reinterpret_cast<C*>(region + (((size_t)D * count * 4 + 15) & ~size_t(15)));  // staged reflectors
    __shared__ C s_x0;
    __shared__ int s_rounds;
    C* A = ws_a + b * (int64_t)D * D;
    const C* H = in + b * (int64_t)D * D;
    for (int idx = tid; idx < D * D; idx += NT) {
        const int i = idx % D, j = idx / D;
        if (i >= j) {
            C v = H[idx];
            if (i == j) v.y = 0.f;
            A[i + LD * j] = v;
            A[j + LD * i] = make_float2(v.x, -v.y);
        }
    }
    __syncthreads();
    GWT_CLK(t_ph0);
#ifdef GWT_PHASE_TIMERS
    long long hs[5] = {0, 0, 0, 0, 0}, hc = 0, hn = 0;
#define GWT_HS(slot) GWT_TICK(hn); hs[slot] += hn - hc; hc = hn;
#else
#define GWT_HS(slot)
#endif
    const int r = tid / Q, q = tid % Q;
    const bool row_ok = r < D;
    R* rt2 = red;
    R* rkp = red + NW;
    for (int k0 = 0; k0 + 2 < D; k0 += kPanel) {
        const int kend = min(k0 + kPanel, D - 2);  // steps k in [k0, kend)
        for (int k = k0; k < kend; ++k) {
            const int j = k - k0;
            GWT_TICK(hc);
            // (1) column k of the effective trailing matrix, rows >= k: A - sum_{i<j} (V_i W_i^H + W_i V_i^H)
            C a = make_float2(0.f, 0.f), corr = make_float2(0.f, 0.f);
            if (row_ok && r >= k) {
                for (int i = q; i < j; i += Q) {
                    cfmac(corr, Vp[i * D + r], Wp[i * D + k]);
                    cfmac(corr, Wp[i * D + r], Vp[i * D + k]);
                }
            }
            corr.x += __shfl_xor_sync(0xffffffffu, corr.x, 1);
            corr.y += __shfl_xor_sync(0xffffffffu, corr.y, 1);
            if (row_ok && r >= k) {
                const C a0 = A[r + LD * k];
                a = make_float2(a0.x - corr.x, a0.y - corr.y);
                if (q == 0 && r == k) A[k + LD * k] = make_float2(a.x, 0.f);
                if (q == 0 && r == k + 1) s_x0 = a;
            }
            {
                R part = (q == 0 && row_ok && r > k + 1) ? a.x * a.x + a.y * a.y : 0.f;
                part = rows_sum<Q>(part);
                if (lane == 0) rt2[wid] = part;
            }
            __syncthreads();  // [1] norm partials, x0
            GWT_HS(0)
            R t2 = 0.f;
#pragma unroll
            for (int w = 0; w < NW; ++w) t2 += rt2[w];
            const C x0 = s_x0;
            C al, v0;
            R tk;
            if (t2 == 0.f) {  // column already reduced: H = I (v = 0, w = 0)
                al = x0;
                v0 = make_float2(0.f, 0.f);
                tk = 0.f;
            } else {
                reflector(x0, t2, al, v0, tk);
            }
            const C v = (row_ok && r > k && t2 != 0.f) ? (r == k + 1 ? v0 : a) : make_float2(0.f, 0.f);
            if (q == 0 && row_ok) {
                Vp[j * D + r] = v;
                if (r > k) A[r + LD * k] = v;
            }
            if (tid == 0) {
                tau[k] = tk;
                sub[k] = al;
            }
            __syncthreads();  // [2] v visible
            GWT_HS(1)
            // (2) x = W^H v, y = V^H v over the panel's previous columns: warp w takes dot products
            // w, w + 16, w + 32, w + 48 as four independent chains
            const C* vj = Vp + j * D;
            if (wid < 2 * j) {
                const int nd = 2 * j;
                const C* src[4];
                C sacc[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int d = wid + NW * u;
                    src[u] = d < nd ? ((d & 1) ? Vp + (d >> 1) * D : Wp + (d >> 1) * D) : vj;
                    sacc[u] = make_float2(0.f, 0.f);
                }
                for (int c = k + 1 + lane; c < D; c += 32) {
                    const C vc = vj[c];
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (wid + NW * u < nd) cfmaconj(sacc[u], src[u][c], vc);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        sacc[u].x += __shfl_xor_sync(0xffffffffu, sacc[u].x, o);
                        sacc[u].y += __shfl_xor_sync(0xffffffffu, sacc[u].y, o);
                    }
                if (lane == 0) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int d = wid + NW * u;
                        if (d < nd) xy[(d & 1) * kPanel + (d >> 1)] = sacc[u];
                    }
                }
            }
            GWT_HS(2)
            // (3) p = A v over the rows k < r < D (the trailing matrix as of the panel start) by all threads:
            // Qm = 2..16 threads per active row as the trailing block shrinks, 16 loads in flight
            {
                const int nr = D - k - 1;
                const int Qm = nr > 128 ? 2 : nr > 64 ? 4 : nr > 32 ? 8 : 16;
                const int rr = k + 1 + tid / Qm, qm = tid % Qm;
                C p0 = make_float2(0.f, 0.f), p1 = make_float2(0.f, 0.f);
                if (rr < D) {
                    const C* arow = A + rr;
                    int c = k + 1 + qm;
                    for (; c + 15 * Qm < D; c += 16 * Qm) {
                        C av[16];
#pragma unroll
                        for (int u = 0; u < 16; ++u) av[u] = arow[LD * (c + u * Qm)];
#pragma unroll
                        for (int u = 0; u < 16; u += 2) {
                            cfma(p0, av[u], vj[c + u * Qm]);
                            cfma(p1, av[u + 1], vj[c + (u + 1) * Qm]);
                        }
                    }
                    for (; c + 3 * Qm < D; c += 4 * Qm) {
                        C av[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) av[u] = arow[LD * (c + u * Qm)];
                        cfma(p0, av[0], vj[c]);
                        cfma(p1, av[1], vj[c + Qm]);
                        cfma(p0, av[2], vj[c + 2 * Qm]);
                        cfma(p1, av[3], vj[c + 3 * Qm]);
                    }
                    for (; c < D; c += Qm) cfma(p0, arow[LD * c], vj[c]);
                }
                C ps = make_float2(p0.x + p1.x, p0.y + p1.y);
                for (int o = 1; o < Qm; o <<= 1) {
                    ps.x += __shfl_xor_sync(0xffffffffu, ps.x, o);
                    ps.y += __shfl_xor_sync(0xffffffffu, ps.y, o);
                }
                if (qm == 0 && rr < D) pA[rr] = ps;
            }
            GWT_HS(3)
            __syncthreads();  // [3] x, y visible
            C pv = (q == 0 && row_ok && r > k) ? pA[r] : make_float2(0.f, 0.f);
            if (row_ok && r > k) {
                for (int i = q; i < j; i += Q) {
                    const C xi = xy[i], yi = xy[kPanel + i];
                    const C vr = Vp[i * D + r], wr = Wp[i * D + r];
                    pv.x -= vr.x * xi.x - vr.y * xi.y + wr.x * yi.x - wr.y * yi.y;
                    pv.y -= vr.x * xi.y + vr.y * xi.x + wr.x * yi.y + wr.y * yi.x;
                }
            }
            pv.x += __shfl_xor_sync(0xffffffffu, pv.x, 1);
            pv.y += __shfl_xor_sync(0xffffffffu, pv.y, 1);
            pv = make_float2(pv.x * tk, pv.y * tk);
            {
                R kp = (q == 0 && row_ok && r > k) ? v.x * pv.x + v.y * pv.y : 0.f;
                kp = rows_sum<Q>(kp);
                if (lane == 0) rkp[wid] = kp;
            }
            __syncthreads();  // [4] v^H p partials
            R ks = 0.f;
#pragma unroll
            for (int w = 0; w < NW; ++w) ks += rkp[w];
            const R kk = 0.5f * tk * ks;
            if (q == 0 && row_ok)
                Wp[j * D + r] = (r > k) ? make_float2(pv.x - kk * v.x, pv.y - kk * v.y) : make_float2(0.f, 0.f);
            __syncthreads();  // [5] w visible (next column update, next dots)
            GWT_HS(4)
        }
        // Hermitian rank-2*nj update of the trailing matrix, rows and columns >= kend: warp tiles of 32 rows x 16
        // columns, lane (lr, lc) = (lane % 8, lane / 8) owns rows lr + 8x and columns lc + 4y (x, y < 4),
        // so every shared load is a broadcast of 8 (rows) or 4 (columns) consecutive entries
        const int nj = kend - k0;
        const int kb = kend & ~7;
        const int nwr = (D - kb + 31) / 32, nwc = (D - kb + 15) / 16;
        const int lr = lane % 8, lc = lane / 8;
        for (int wt = wid; wt < nwr * nwc; wt += NW) {
            // the lower triangle is computed, the upper mirrored (tiles wholly above the diagonal skip)
            if (kb + 32 * (wt % nwr) + 31 < kb + 16 * (wt / nwr)) continue;
            const int rb = kb + 32 * (wt % nwr) + lr, cb = kb + 16 * (wt / nwr) + lc;
            C acc[4][4];
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
                for (int y = 0; y < 4; ++y) acc[x][y] = make_float2(0.f, 0.f);
            for (int i = 0; i < nj; ++i) {
                const C* vi = Vp + i * D;
                const C* wi = Wp + i * D;
                C vr[4], wr[4], vc[4], wc[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int rr = min(rb + 8 * u, D - 1), cc = min(cb + 4 * u, D - 1);
                    vr[u] = vi[rr];
                    wr[u] = wi[rr];
                    vc[u] = vi[cc];
                    wc[u] = wi[cc];
                }
#pragma unroll
                for (int x = 0; x < 4; ++x)
#pragma unroll
                    for (int y = 0; y < 4; ++y) {
                        cfmac(acc[x][y], vr[x], wc[y]);
                        cfmac(acc[x][y], wr[x], vc[y]);
                    }
            }
#pragma unroll
            for (int y = 0; y < 4; ++y) {
                const int c = cb + 4 * y;
                if (c < kend || c >= D) continue;
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    const int rr = rb + 8 * x;
                    if (rr < c || rr >= D) continue;
                    C& e = A[rr + LD * c];
                    const C nv = make_float2(e.x - acc[x][y].x, e.y - acc[x][y].y);
                    e = nv;
                    if (rr > c) A[c + LD * rr] = make_float2(nv.x, -nv.y);
                }
            }
        }
        __syncthreads();
    }
    __syncthreads();
    GWT_CLK(t_ph1);
    // 2. tridiagonal + phases
    for (int i = tid; i < D; i += NT) sd[i] = A[i + LD * i].x;
    if (tid == 0) {
        C dl = make_float2(1.f, 0.f);
        dlt[0] = dl;
        for (int i = 0; i + 1 < D; ++i) {
            const C s = (i + 2 < D) ? sub[i] : A[(i + 1) + LD * i];
            const R mag = hypotf(s.x, s.y);
            se[i] = mag;
            se2[i] = mag * mag;
            if (mag > 0.f) dl = cmul(dl, make_float2(s.x / mag, s.y / mag));
            dlt[i + 1] = dl;
        }
        se[D - 1] = 0.f;
        se2[D - 1] = 0.f;
    }
    __syncthreads();
    double lo_p = 1e308, hi_p = -1e308, nrm_p = 0.0;
    for (int i = tid; i < D; i += NT) {
        const double rr = (double)(i > 0 ? se[i - 1] : 0.f) + (double)se[i];
        lo_p = fmin(lo_p, (double)sd[i] - rr);
        hi_p = fmax(hi_p, (double)sd[i] + rr);
        nrm_p = fmax(nrm_p, fabs((double)sd[i]) + rr);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo_p = fmin(lo_p, __shfl_xor_sync(0xffffffffu, lo_p, o));
        hi_p = fmax(hi_p, __shfl_xor_sync(0xffffffffu, hi_p, o));
        nrm_p = fmax(nrm_p, __shfl_xor_sync(0xffffffffu, nrm_p, o));
    }
    __shared__ double bred[3][NW];
    if (lane == 0) {
        bred[0][wid] = lo_p;
        bred[1][wid] = hi_p;
        bred[2][wid] = nrm_p;
    }
    __syncthreads();
    double glo = 1e308, ghi = -1e308, tnorm = 0.0;
#pragma unroll
    for (int w2 = 0; w2 < NW; ++w2) {
        glo = fmin(glo, bred[0][w2]);
        ghi = fmax(ghi, bred[1][w2]);
        tnorm = fmax(tnorm, bred[2][w2]);
    }
    const double eps = 1.1920928955078125e-07;
    glo -= 2.0 * eps * tnorm;
    ghi += 2.0 * eps * tnorm;
    const double inv_n = tnorm > 0.0 ? 1.0 / tnorm : 1.0;
    for (int i = tid; i < D; i += NT) {
        fd[i] = (float)((double)sd[i] * inv_n);
        fe2[i] = i > 0 ? (float)((double)se2[i - 1] * inv_n * inv_n) : 0.f;  // shifted (sturm_count_p32)
    }
    __syncthreads();
    {
        int S = NT / count;
        S = S >= 8 ? 8 : (S >= 4 ? 4 : (S >= 2 ? 2 : 1));
        const int t = tid / S, s = tid % S;
        const int gl = lane / S;
        const int want = D - 1 - t;
        float lo = (float)(glo * inv_n) - 1e-6f, hi = (float)(ghi * inv_n) + 1e-6f;
        bool done = t >= count;
        for (int it = 0; it < 96; ++it) {
            if (!done && hi - lo <= 2e-7f * fmaxf(fmaxf(fabsf(lo), fabsf(hi)), 1e-3f)) done = true;
            if (__all_sync(0xffffffffu, done)) break;
            const float step = (hi - lo) / (float)(S + 1);
            const float pt = lo + (float)(s + 1) * step;
            const bool le = !done && sturm_count_r<float>(D, fd, fe2, pt) <= want;
            const unsigned bits = __ballot_sync(0xffffffffu, le);
            if (!done) {
                const int j = __popc((bits >> (gl * S)) & ((1u << S) - 1u));
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
    if (tid == 0) {
        const double ctol = ctol_rel * fmax(tnorm, 1e-300);
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
    // 3b. inverse iteration: thread t = eigenvalue t; x in XR[i][t]; LU in the global workspace
    {
        const int t = tid;
        R* DDv = ws_lu + b * (int64_t)count * 3 * D;
        R* DUv = DDv + (int64_t)count * D;
        R* MLv = DUv + (int64_t)count * D;
#define LU_(arr, i) arr[(int64_t)(i) * count + t]
#define XV(i) XR[(i) * count + t]
        const R tiny = (R)fmax(eps * tnorm, 1e-30);
        constexpr int kSolves = 2;
        for (int rd = 0; rd < rounds; ++rd) {
            if (t < count && scl[t] == rd) {
                const R lam = (R)lamv[t];
                uint32_t sw[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
                R dcur = sd[0] - lam, ucur = se[0];
                for (int i = 0; i + 1 < D; ++i) {
                    const R sb = se[i], dn = sd[i + 1] - lam, en = (i + 2 < D) ? se[i + 1] : 0.f;
                    R mult;
                    if (fabsf(dcur) >= fabsf(sb)) {
                        const R di = dcur == 0.f ? tiny : dcur;
                        mult = ii_div(sb, di);
                        LU_(DDv, i) = di;
                        LU_(DUv, i) = ucur;
                        dcur = dn - mult * ucur;
                        ucur = en;
                    } else {
                        mult = ii_div(dcur, sb);
                        sw[i >> 5] |= 1u << (i & 31);
                        LU_(DDv, i) = sb;
                        LU_(DUv, i) = dn;
                        dcur = ucur - mult * dn;
                        ucur = -mult * en;
                    }
                    LU_(MLv, i) = mult;
                }
                LU_(DDv, D - 1) = dcur;
                for (int i = 0; i < D; ++i) {
                    R di = LU_(DDv, i);
                    if (fabsf(di) < tiny) di = di < 0.f ? -tiny : tiny;
                    LU_(DDv, i) = 1.f / di;
                }
                for (int i = 0; i < D; ++i) XV(i) = 1.f + 0.25f * __sinf(0.7f * i + 1.3f * t);
                for (int it = 0; it <= kSolves; ++it) {
                    for (int s2 = t - rd; s2 < t; ++s2) {
                        R dot = 0.f;
                        for (int i = 0; i < D; ++i) dot += XR[i * count + s2] * XV(i);
                        for (int i = 0; i < D; ++i) XV(i) -= dot * XR[i * count + s2];
                    }
                    R nn = 0.f;
                    for (int i = 0; i < D; ++i) nn += XV(i) * XV(i);
                    const R inv = nn > 0.f ? rsqrtf(nn) : 1.f;
                    for (int i = 0; i < D; ++i) XV(i) *= inv;
                    if (it == kSolves) break;
                    for (int i = 0; i + 1 < D; ++i) {
                        const R ml = LU_(MLv, i);
                        if ((sw[i >> 5] >> (i & 31)) & 1u) {
                            const R t0 = XV(i);
                            XV(i) = XV(i + 1);
                            XV(i + 1) = t0 - ml * XV(i + 1);
                        } else {
                            XV(i + 1) -= ml * XV(i);
                        }
                    }
                    R x2 = 0.f, x1 = 0.f;  // x[i+2], x[i+1]
                    for (int i = D - 1; i >= 0; --i) {
                        R acc = XV(i);
                        if (i + 1 < D) acc -= LU_(DUv, i) * x1;
                        if (i + 2 < D && ((sw[i >> 5] >> (i & 31)) & 1u)) acc -= se[i + 1] * x2;
                        const R xi = acc * LU_(DDv, i);
                        XV(i) = xi;
                        x2 = x1;
                        x1 = xi;
                    }
                    R mx = 0.f;
                    for (int i = 0; i < D; ++i) mx = fmaxf(mx, fabsf(XV(i)));
                    if (!(mx > 0.f) || !isfinite(mx)) {
                        if (fail) atomicExch(fail, 1);
                        break;
                    }
                    const R sc = 1.f / mx;
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
    // 4. back-transform, 8 threads per eigenvector (rows i = qb mod 8), vectors in batches of NT/8
    for (int tb = 0; tb < count; tb += NT / 8) {
        constexpr int QB = 8, RPT = DM / QB;
        const int t = tb + tid / QB, qb = tid % QB;
        const bool on = t < count;
        if (on && qb == 0 && evals) evals[b * count + t] = lamv[t];
        C y[RPT];
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
            const int i = qb + QB * u;
            y[u] = make_float2(0.f, 0.f);
            if (on && i < D) {
                const R z = XR[i * count + t];
                const C dl = dlt[i];
                y[u] = make_float2(dl.x * z, dl.y * z);
            }
        }
        // reflectors in blocks of kPanel, staged (rows <= k zeroed) into shared memory
        for (int khi = D - 3; khi >= 0; khi -= kPanel) {
            const int klo = max(0, khi - kPanel + 1);
            __syncthreads();  // previous block applied by every thread
            for (int idx = tid; idx < (khi - klo + 1) * D; idx += NT) {
                const int kk = idx / D, i = idx % D, k = klo + kk;
                Sg[idx] = i > k ? A[i + LD * k] : make_float2(0.f, 0.f);
            }
            __syncthreads();
            for (int k = khi; k >= klo; --k) {
                const R tk = tau[k];
                if (tk == 0.f) continue;
                const C* vk = Sg + (k - klo) * D;
                C dot = make_float2(0.f, 0.f);
#pragma unroll
                for (int u = 0; u < RPT; ++u) {
                    const int i = qb + QB * u;
                    if (i < D) cfmaconj(dot, vk[i], y[u]);
                }
#pragma unroll
                for (int o = 1; o < QB; o <<= 1) {
                    dot.x += __shfl_xor_sync(0xffffffffu, dot.x, o);
                    dot.y += __shfl_xor_sync(0xffffffffu, dot.y, o);
                }
                dot = make_float2(dot.x * tk, dot.y * tk);
#pragma unroll
                for (int u = 0; u < RPT; ++u) {
                    const int i = qb + QB * u;
                    if (i < D) {
                        const C pr = cmul(vk[i], dot);
                        y[u].x -= pr.x;
                        y[u].y -= pr.y;
                    }
                }
            }
        }
        R best = -1.f;
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
        C yb = make_float2(0.f, 0.f);
#pragma unroll
        for (int u = 0; u < RPT; ++u)
            if (qb + QB * u == bi) yb = y[u];
        const int owner = (lane & ~(QB - 1)) | (bi % QB);
        yb = shfl_c(yb, owner);
        if (on) {
            C fac = make_float2(1.f, 0.f);
            if (best > 0.f) {
                const R im = rsqrtf(best);
                fac = make_float2(yb.x * im, -yb.y * im);
            }
            C* ob = out + (b * count + t) * (int64_t)D;
#pragma unroll
            for (int u = 0; u < RPT; ++u) {
                const int i = qb + QB * u;
                if (i < D) ob[i] = cmul(y[u], fac);
            }
        }
    }
#ifdef GWT_PHASE_TIMERS
    if (b == 0 && tid == 0) {
        g_eig_phase[4] = hs[0] + hs[1];
        g_eig_phase[5] = hs[2];
        g_eig_phase[6] = hs[3];
        g_eig_phase[7] = hs[4];
        const long long t_ph4 = clock64();
        g_eig_phase[0] = t_ph1 - t_ph0;
        g_eig_phase[1] = t_ph2 - t_ph1;
        g_eig_phase[2] = t_ph3 - t_ph2;
        g_eig_phase[3] = t_ph4 - t_ph3;
    }
#endif
}
