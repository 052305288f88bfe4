// Batched Hermitian eigensolver for the Tucker factor updates, sm_100a.
//
// Reference: leading_eigenvectors (proj/src/linalg.cpp:27-45) -> Eigen
// SelfAdjointEigenSolver (Householder tridiagonalisation + implicit QR),
// reversed to descending order, then phase_normalize_columns (:11-25).
//
// B200 mapping: one CTA (256 threads) per matrix, fp64 throughout (the Gram
// may be c64; its eigenvectors are computed in binary64 and rounded once).
//  1. Householder reduction to Hermitian tridiagonal: each step is a
//     CTA-wide block reduction + a coalesced Hermitian mat-vec + a rank-2
//     update of the trailing block (workspace in global memory, L1/L2 resident).
//  2. Diagonal phase similarity to a real symmetric tridiagonal.
//  3. Implicit-shift QL: thread 0 generates each QL sweep's Givens sequence
//     into shared memory, all threads then apply it to their row of Z
//     (one row per thread), so the O(n^3) vector work is parallel.
//  4. Top-`count` selection, back-transform through the stored reflectors,
//     phase normalisation (largest-|.| entry real >= 0, lowest index on ties).
#include "kernels.cuh"

namespace gwtk {

constexpr int kEigThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x < 32) {
        s = threadIdx.x < kEigThreads / 32 ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) red[32] = s;
    }
    __syncthreads();
    return red[32];
}

// in: [batch][D][D] Hermitian (column-major; the lower triangle is read),
// out: [batch][count][D] top eigenvectors, evals (nullable): [batch][count].
// ws_a: [batch][D][D] double2, ws_z: [batch][D][D] double, ws_x: [batch][count][D] double2
template <class T>
__global__ void __launch_bounds__(kEigThreads) k_heev_topk(int D, int count, const cplx_t<T>* __restrict__ in,
                                                           cplx_t<T>* __restrict__ out, double* __restrict__ evals,
                                                           double2* __restrict__ ws_a, double* __restrict__ ws_z,
                                                           double2* __restrict__ ws_x, int* __restrict__ fail) {
    using C = cplx_t<T>;
    __shared__ double2 sv[256];   // Householder vector of the current step
    __shared__ double2 sp[256];   // p / w
    __shared__ double2 salpha[256];
    __shared__ double stau[256];
    __shared__ double sd[256], se[256];
    __shared__ double2 sdelta[256];
    __shared__ double rc[256], rs[256];
    __shared__ double red[33];
    __shared__ int sel[256];
    __shared__ int ctl[4];  // [0] done flag, [1] l, [2] m (rotation range)
    __shared__ double ctlf[2];  // f, tst1 (thread-0 state)
    const int64_t b = blockIdx.x;
    const int tid = threadIdx.x;
    double2* A = ws_a + b * (int64_t)D * D;
    double* Z = ws_z + b * (int64_t)D * D;
    const C* H = in + b * (int64_t)D * D;
    // load, Hermitian from the lower triangle
    for (int idx = tid; idx < D * D; idx += kEigThreads) {
        const int i = idx % D, j = idx / D;
        if (i >= j) {
            double2 v = to_d2(H[idx]);
            if (i == j) v.y = 0.0;
            A[i + (int64_t)D * j] = v;
            A[j + (int64_t)D * i] = make_double2(v.x, -v.y);
        }
    }
    __syncthreads();
    // 1. Householder tridiagonalisation
    for (int k = 0; k + 2 < D; ++k) {
        const int len = D - k - 1;
        double tail = 0.0;
        for (int r = tid; r < len; r += kEigThreads) {
            const double2 x = A[(k + 1 + r) + (int64_t)D * k];
            sv[r] = x;
            if (r >= 1) tail += x.x * x.x + x.y * x.y;
        }
        const double tail2 = block_sum(tail, red);
        if (tail2 == 0.0) {
            if (tid == 0) {
                stau[k] = 0.0;
                salpha[k] = A[(k + 1) + (int64_t)D * k];
            }
            __syncthreads();
            continue;
        }
        if (tid == 0) {
            const double2 x0 = sv[0];
            const double ax0 = hypot(x0.x, x0.y);
            const double xnorm = sqrt(tail2 + ax0 * ax0);
            const double2 ph = ax0 > 0.0 ? make_double2(x0.x / ax0, x0.y / ax0) : make_double2(1.0, 0.0);
            const double2 alpha = make_double2(-ph.x * xnorm, -ph.y * xnorm);
            const double2 v0 = make_double2(x0.x - alpha.x, x0.y - alpha.y);
            sv[0] = v0;
            stau[k] = 2.0 / (tail2 + v0.x * v0.x + v0.y * v0.y);
            salpha[k] = alpha;
        }
        __syncthreads();
        const double tau = stau[k];
        // p = tau * A22 v
        double2 pv = make_double2(0, 0);
        for (int r = tid; r < len; r += kEigThreads) {
            double2 acc = make_double2(0, 0);
            for (int c = 0; c < len; ++c) cfma(acc, A[(k + 1 + r) + (int64_t)D * (k + 1 + c)], sv[c]);
            acc.x *= tau;
            acc.y *= tau;
            sp[r] = acc;
        }
        __syncthreads();
        // K = tau/2 * v^H p  (Hermitian A22 => real)
        double part = 0.0;
        for (int r = tid; r < len; r += kEigThreads) part += sv[r].x * sp[r].x + sv[r].y * sp[r].y;
        const double kk = 0.5 * tau * block_sum(part, red);
        for (int r = tid; r < len; r += kEigThreads) sp[r] = make_double2(sp[r].x - kk * sv[r].x, sp[r].y - kk * sv[r].y);
        __syncthreads();
        // A22 -= v w^H + w v^H
        for (int idx = tid; idx < len * len; idx += kEigThreads) {
            const int r = idx % len, c = idx / len;
            double2 a = A[(k + 1 + r) + (int64_t)D * (k + 1 + c)];
            const double2 vr = sv[r], wr = sp[r], vc = sv[c], wc = sp[c];
            a.x -= vr.x * wc.x + vr.y * wc.y + wr.x * vc.x + wr.y * vc.y;
            a.y -= vr.y * wc.x - vr.x * wc.y + wr.y * vc.x - wr.x * vc.y;
            A[(k + 1 + r) + (int64_t)D * (k + 1 + c)] = a;
        }
        // keep the reflector in column k below the diagonal
        for (int r = tid; r < len; r += kEigThreads) A[(k + 1 + r) + (int64_t)D * k] = sv[r];
        __syncthreads();
    }
    // 2. tridiagonal (d, e) and phase similarity
    for (int r = tid; r < D; r += kEigThreads) sd[r] = A[r + (int64_t)D * r].x;
    __syncthreads();
    if (tid == 0) {
        double2 dl = make_double2(1.0, 0.0);
        sdelta[0] = dl;
        for (int i = 0; i + 1 < D; ++i) {
            double2 sub;
            if (i + 2 < D) sub = salpha[i];      // step i produced alpha_i (or kept the entry)
            else sub = A[(i + 1) + (int64_t)D * i];  // last sub-diagonal entry untouched
            const double mag = hypot(sub.x, sub.y);
            se[i] = mag;
            if (mag > 0.0) dl = cmul(dl, make_double2(sub.x / mag, sub.y / mag));
            sdelta[i + 1] = dl;
        }
        se[D - 1] = 0.0;
        ctl[0] = 0;
        ctl[1] = 0;
        ctlf[0] = 0.0;
        ctlf[1] = 0.0;
    }
    for (int idx = tid; idx < D * D; idx += kEigThreads) Z[idx] = (idx % D == idx / D) ? 1.0 : 0.0;
    __syncthreads();
    // 3. implicit QL; state machine driven by thread 0
    const double eps = 2.220446049250313e-16;
    int l_state = 0, m_state = -1, iter = 0;
    for (;;) {
        if (tid == 0) {
            double f = ctlf[0], tst1 = ctlf[1];
            int produced = 0;
            while (l_state < D && !produced) {
                const int l = l_state;
                if (m_state < 0) {  // entering l
                    tst1 = fmax(tst1, fabs(sd[l]) + fabs(se[l]));
                    int m = l;
                    while (m < D - 1 && !(fabs(se[m]) <= eps * tst1)) ++m;
                    m_state = m;
                    iter = 0;
                }
                const int m = m_state;
                if (m == l || fabs(se[l]) <= eps * tst1) {
                    sd[l] += f;
                    se[l] = 0.0;
                    ++l_state;
                    m_state = -1;
                    continue;
                }
                if (++iter > 300) {
                    if (fail) atomicExch(fail, 1);
                    sd[l] += f;
                    se[l] = 0.0;
                    ++l_state;
                    m_state = -1;
                    continue;
                }
                double gg = sd[l];
                double pp = (sd[l + 1] - gg) / (2.0 * se[l]);
                double r = hypot(pp, 1.0);
                if (pp < 0) r = -r;
                sd[l] = se[l] / (pp + r);
                sd[l + 1] = se[l] * (pp + r);
                const double dl1 = sd[l + 1];
                double hh = gg - sd[l];
                for (int i = l + 2; i < D; ++i) sd[i] -= hh;
                f += hh;
                pp = sd[m];
                double c = 1.0, c2 = 1.0, c3 = 1.0, s = 0.0, s2 = 0.0;
                const double el1 = se[l + 1];
                for (int i = m - 1; i >= l; --i) {
                    c3 = c2;
                    c2 = c;
                    s2 = s;
                    gg = c * se[i];
                    hh = c * pp;
                    r = hypot(pp, se[i]);
                    se[i + 1] = s * r;
                    s = se[i] / r;
                    c = pp / r;
                    pp = c * sd[i] - s * gg;
                    sd[i + 1] = hh + s * (c * gg + s * sd[i]);
                    rc[i] = c;
                    rs[i] = s;
                }
                pp = -s * s2 * c3 * el1 * se[l] / dl1;
                se[l] = s * pp;
                sd[l] = c * pp;
                ctl[1] = l;
                ctl[2] = m;
                produced = 1;
            }
            ctlf[0] = f;
            ctlf[1] = tst1;
            ctl[0] = produced ? 0 : 1;
        }
        __syncthreads();
        if (ctl[0]) break;
        const int l = ctl[1], m = ctl[2];
        for (int row = tid; row < D; row += kEigThreads) {
            double zip1 = Z[row + (int64_t)D * m];
            for (int i = m - 1; i >= l; --i) {
                const double zi = Z[row + (int64_t)D * i];
                Z[row + (int64_t)D * (i + 1)] = rs[i] * zi + rc[i] * zip1;
                zip1 = rc[i] * zi - rs[i] * zip1;
            }
            Z[row + (int64_t)D * l] = zip1;
        }
        __syncthreads();
    }
    // 4. select top-count (descending, lowest index first on ties)
    for (int r = tid; r < D; r += kEigThreads) {
        const double v = sd[r];
        int rk = 0;
        for (int s = 0; s < D; ++s) rk += (sd[s] > v || (sd[s] == v && s < r)) ? 1 : 0;
        if (rk < count) sel[rk] = r;
    }
    __syncthreads();
    double2* X = ws_x + b * (int64_t)count * D;
    for (int idx = tid; idx < count * D; idx += kEigThreads) {
        const int c = idx / D, r = idx % D;
        const double z = Z[r + (int64_t)D * sel[c]];
        X[idx] = make_double2(sdelta[r].x * z, sdelta[r].y * z);
    }
    if (evals)
        for (int c = tid; c < count; c += kEigThreads) evals[b * count + c] = sd[sel[c]];
    __syncthreads();
    // back-transform x <- H_0 H_1 ... H_{D-3} x, one warp per column
    const int warp = tid / 32, lane = tid % 32;
    for (int k = D - 3; k >= 0; --k) {
        const double tau = stau[k];
        if (tau != 0.0) {
            const int len = D - k - 1;
            for (int c = warp; c < count; c += kEigThreads / 32) {
                double2* xc = X + (int64_t)c * D + k + 1;
                double2 dot = make_double2(0, 0);
                for (int r = lane; r < len; r += 32) cfmaconj(dot, A[(k + 1 + r) + (int64_t)D * k], xc[r]);
                for (int o = 16; o > 0; o >>= 1) {
                    dot.x += __shfl_xor_sync(0xffffffffu, dot.x, o);
                    dot.y += __shfl_xor_sync(0xffffffffu, dot.y, o);
                }
                dot.x *= tau;
                dot.y *= tau;
                for (int r = lane; r < len; r += 32) {
                    const double2 v = A[(k + 1 + r) + (int64_t)D * k];
                    double2 x = xc[r];
                    double2 pr = cmul(v, dot);
                    x.x -= pr.x;
                    x.y -= pr.y;
                    xc[r] = x;
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
}

template <class T>
cudaError_t launch_heev_topk(int D, int count, int64_t batch, const void* in, void* out, double* evals, double2* ws_a,
                             double* ws_z, double2* ws_x, int* fail, cudaStream_t st) {
    if (D > 256 || D < 1) return cudaErrorInvalidValue;
    k_heev_topk<T><<<(unsigned)batch, kEigThreads, 0, st>>>(D, count, (const cplx_t<T>*)in, (cplx_t<T>*)out, evals,
                                                           ws_a, ws_z, ws_x, fail);
    return cudaGetLastError();
}

template cudaError_t launch_heev_topk<float>(int, int, int64_t, const void*, void*, double*, double2*, double*,
                                             double2*, int*, cudaStream_t);
template cudaError_t launch_heev_topk<double>(int, int, int64_t, const void*, void*, double*, double2*, double*,
                                              double2*, int*, cudaStream_t);

}  // namespace gwtk
