// Per-thread small dense Hermitian kernels (M <= 8), shared by the SINR and
// Tucker paths. Matrices live in registers (compile-time indices).
#pragma once

#include "common.cuh"

namespace gwtk {

// Jacobi stop: sum_{p<q} |a_pq|^2 <= tol * sum_p a_pp^2. 1e-22 leaves eigenvector errors ~1e-11/gap
// (the c128 SINR parity bound is 1e-9); 1e-30 (full convergence) costs ~1-2 extra sweeps.
constexpr double kJacobiTol = 1e-22;

// ---------------------------------------------------------------------------
// Per-thread small Hermitian eigensolver (cyclic complex Jacobi, fp64), the
// rotation of the reference test oracle (proj/tests/support/oracles.hpp:31-97).
// Hermitian storage helpers for compile-time indices: only the lower triangle (i >= j) is kept.
template <int M>
__device__ __forceinline__ double2 hget(const double2 (&A)[M][M], int i, int j) {
    return i >= j ? A[i][j] : make_double2(A[j][i].x, -A[j][i].y);
}
template <int M>
__device__ __forceinline__ void hset(double2 (&A)[M][M], int i, int j, double2 v) {
    if (i >= j) A[i][j] = v;
    else A[j][i] = make_double2(v.x, -v.y);
}

// Per-thread small Hermitian eigensolver (cyclic complex Jacobi, fp64), the rotation of the
// reference test oracle (proj/tests/support/oracles.hpp:31-97). A is read and updated through its
// lower triangle only (the upper one is its mirror): a rotation updates the 2(M-2) off-block entries
// of columns p, q, the 2x2 block (p, q) and V, instead of full rows and columns of A (27 % fewer
// binary64 operations at M = 8, fewer live registers). On return A's diagonal holds the eigenvalues.
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
            for (int q = p + 1; q < M; ++q) off += A[q][p].x * A[q][p].x + A[q][p].y * A[q][p].y;
        }
        if (off <= kJacobiTol * dia || off == 0.0) break;
#pragma unroll
        for (int p = 0; p < M; ++p)
#pragma unroll
            for (int q = p + 1; q < M; ++q) {
                const double2 aqp = A[q][p];  // a_pq = conj(a_qp)
                const double b2 = aqp.x * aqp.x + aqp.y * aqp.y;
                if (b2 > 1e-300) {
                    // rotation angle in fp32 (only the convergence rate depends on it); the rotation
                    // itself (unit phase, c = 1/sqrt(1+t^2), s = t c) is exact in binary64
                    const double rb = frsqrt(b2);
                    const double phr = aqp.x * rb, phi = -aqp.y * rb;  // phase = apq/|apq|
                    const float tau = (float)((A[q][q].x - A[p][p].x) * (0.5 * rb));
                    const float tf = copysignf(1.0f, tau) / (fabsf(tau) + sqrtf(fmaf(tau, tau, 1.0f)));
                    const double tt = (double)tf;
                    const double c = frsqrt(fma(tt, tt, 1.0));
                    const double s = tt * c;
                    // U = [[c, s], [-s conj(ph), c conj(ph)]]
                    const double2 uqp = make_double2(-s * phr, s * phi);
                    const double2 uqq = make_double2(c * phr, -c * phi);
#pragma unroll
                    for (int r = 0; r < M; ++r) {  // A <- U^H A U on the off-block entries of columns p, q
                        if (r == p || r == q) continue;
                        const double2 arp = hget(A, r, p), arq = hget(A, r, q);
                        double2 np = make_double2(c * arp.x, c * arp.y);
                        cfma(np, arq, uqp);
                        double2 nq = make_double2(s * arp.x, s * arp.y);
                        cfma(nq, arq, uqq);
                        hset(A, r, p, np);
                        hset(A, r, q, nq);
                    }
                    {  // the 2x2 block: columns, then rows (as the full update restricted to p, q)
                        const double2 app = A[p][p], aqq = A[q][q], apq = make_double2(aqp.x, -aqp.y);
                        double2 cp_p = make_double2(c * app.x, c * app.y);
                        cfma(cp_p, apq, uqp);
                        double2 cq_p = make_double2(s * app.x, s * app.y);
                        cfma(cq_p, apq, uqq);
                        double2 cp_q = make_double2(c * aqp.x, c * aqp.y);
                        cfma(cp_q, aqq, uqp);
                        double2 cq_q = make_double2(s * aqp.x, s * aqp.y);
                        cfma(cq_q, aqq, uqq);
                        double2 npp = make_double2(c * cp_p.x, c * cp_p.y);
                        cfmaconj(npp, uqp, cp_q);
                        double2 nqp = make_double2(s * cp_p.x, s * cp_p.y);
                        cfmaconj(nqp, uqq, cp_q);
                        double2 nqq = make_double2(s * cq_p.x, s * cq_p.y);
                        cfmaconj(nqq, uqq, cq_q);
                        A[p][p] = make_double2(npp.x, 0.0);
                        A[q][q] = make_double2(nqq.x, 0.0);
                        A[q][p] = nqp;
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


}  // namespace gwtk
