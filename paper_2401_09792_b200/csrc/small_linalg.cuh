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
        if (off <= kJacobiTol * dia || off == 0.0) break;
#pragma unroll
        for (int p = 0; p < M; ++p)
#pragma unroll
            for (int q = p + 1; q < M; ++q) {
                const double b2 = A[p][q].x * A[p][q].x + A[p][q].y * A[p][q].y;
                if (b2 > 1e-300) {
                    // rotation angle in fp32 (only the convergence rate depends on it); the rotation
                    // itself (unit phase, c = 1/sqrt(1+t^2), s = t c) is exact in binary64
                    const double rb = rsqrt(b2);
                    const double phr = A[p][q].x * rb, phi = A[p][q].y * rb;  // phase = apq/|apq|
                    const float tau = (float)((A[q][q].x - A[p][p].x) * (0.5 * rb));
                    const float tf = copysignf(1.0f, tau) / (fabsf(tau) + sqrtf(fmaf(tau, tau, 1.0f)));
                    const double tt = (double)tf;
                    const double c = rsqrt(fma(tt, tt, 1.0));
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


}  // namespace gwtk
