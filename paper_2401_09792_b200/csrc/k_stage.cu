// Per-stage SINR helper kernels for the reference's single-system stage API (sinr.hpp:113-124), used by
// the gwt:: drop-in's woodbury_inverse_apply. The batched hot path never calls these: its Cholesky and
// checks run fused inside K3 (k_sinr.cu).
#include "kernels.cuh"

namespace gwtk {

// Hermitian positive-definite solve X = Q^-1 B for a batch of m x m covariances and m x nrhs right-hand
// sides (column-major binary64 complex), the Eigen::LLT use of woodbury_inverse_apply
// (proj/src/sinr.cpp:205-227; B = Q - sigma^2 I) and filter_full (:113-127; B = H V): finite check,
// Cholesky of the lower triangle (a non-positive pivot fails), optional condition estimate
// (max/min Cholesky diagonal)^2 > 1e14, forward/back substitution per column. One thread per matrix,
// L in a global workspace (single small systems: latency, not throughput, matters here).
// status: 0 ok, 1 not positive definite, 2 condition estimate above 1e14, 4 non-finite input.
__global__ void k_hpd_solve(int m, int nrhs, int64_t batch, const double2* __restrict__ Q,
                            const double2* __restrict__ B, int check_cond, double2* __restrict__ Lw,
                            double2* __restrict__ T, int* __restrict__ status) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    const int64_t mm = (int64_t)m * m;
    const double2* q = Q + b * mm;
    const double2* rhs = B + b * (int64_t)m * nrhs;
    double2* l = Lw + b * mm;
    double2* t = T + b * (int64_t)m * nrhs;
    for (int64_t e = 0; e < mm; ++e)
        if (!isfinite(q[e].x) || !isfinite(q[e].y)) {
            status[b] = 4;
            return;
        }
    for (int64_t e = 0; e < (int64_t)m * nrhs; ++e)
        if (!isfinite(rhs[e].x) || !isfinite(rhs[e].y)) {
            status[b] = 4;
            return;
        }
    double dmax = 0.0, dmin = 1e308;
    for (int c = 0; c < m; ++c) {
        double d = q[c + (int64_t)m * c].x;
        for (int k = 0; k < c; ++k) {
            const double2 v = l[c + (int64_t)m * k];
            d -= v.x * v.x + v.y * v.y;
        }
        if (!(d > 0.0)) {
            status[b] = 1;
            return;
        }
        const double lcc = sqrt(d);
        dmax = fmax(dmax, lcc);
        dmin = fmin(dmin, lcc);
        l[c + (int64_t)m * c] = make_double2(lcc, 0.0);
        for (int r = c + 1; r < m; ++r) {
            double2 s = q[r + (int64_t)m * c];
            for (int k = 0; k < c; ++k) {  // s -= L[r][k] conj(L[c][k])
                const double2 a = l[r + (int64_t)m * k], bb = l[c + (int64_t)m * k];
                s.x -= a.x * bb.x + a.y * bb.y;
                s.y -= a.y * bb.x - a.x * bb.y;
            }
            l[r + (int64_t)m * c] = make_double2(s.x / lcc, s.y / lcc);
        }
    }
    if (check_cond && (dmax / dmin) * (dmax / dmin) > 1e14) {
        status[b] = 2;
        return;
    }
    for (int j = 0; j < nrhs; ++j) {
        double2* x = t + (int64_t)m * j;
        for (int i = 0; i < m; ++i) {  // forward: L y = b_j
            double2 acc = rhs[i + (int64_t)m * j];
            for (int k = 0; k < i; ++k) {
                const double2 a = l[i + (int64_t)m * k], y = x[k];
                acc.x -= a.x * y.x - a.y * y.y;
                acc.y -= a.x * y.y + a.y * y.x;
            }
            const double lii = l[i + (int64_t)m * i].x;
            x[i] = make_double2(acc.x / lii, acc.y / lii);
        }
        for (int i = m - 1; i >= 0; --i) {  // back: L^H x = y
            double2 acc = x[i];
            for (int k = i + 1; k < m; ++k) {  // (L^H)[i][k] = conj(L[k][i])
                const double2 a = l[k + (int64_t)m * i], y = x[k];
                acc.x -= a.x * y.x + a.y * y.y;
                acc.y -= a.x * y.y - a.y * y.x;
            }
            const double lii = l[i + (int64_t)m * i].x;
            x[i] = make_double2(acc.x / lii, acc.y / lii);
        }
    }
    status[b] = 0;
}

cudaError_t launch_hpd_solve(int m, int nrhs, int64_t batch, const void* Q, const void* B, int check_cond, void* Lw,
                             void* X, int* status, cudaStream_t st) {
    k_hpd_solve<<<(unsigned)((batch + 63) / 64), 64, 0, st>>>(m, nrhs, batch, (const double2*)Q, (const double2*)B,
                                                               check_cond, (double2*)Lw, (double2*)X, status);
    return cudaGetLastError();
}

}  // namespace gwtk
