// Binary64 re-orthonormalisation of fp32 eigenvector blocks (Cholesky-QR), c64 Tucker factors.
//
// The fp32 eigensolvers (eig_warp / eig_cta / eig_big) return the leading eigenvectors of the
// Gram of an unfolding with ~1e-5 loss of orthogonality at the BASELINE C3/C4 shapes (inverse
// iteration across eigenvalues that are close in the fp32 sense but outside one MGS cluster).
// The energy-split objective f = ||X||^2 - ||core||^2 and the reconstruction both assume
// orthonormal factors (decompose.cpp:28-38,146-193: Eigen's SelfAdjointEigenSolver returns an
// orthonormal basis), so a non-orthonormal factor shifts the NMSE at first order. This kernel
// restores orthonormality to the storage precision without moving the subspace:
//     S = V^H V (binary64),  S = R^H R (Cholesky),  V <- V R^{-1},
// then re-applies the eigensolvers' phase convention (largest-magnitude entry of each column
// real positive, first index on ties; linalg.cpp:11-30 phase_normalize_columns).
//
// One CTA per D x count block (column-major, D <= 256, count <= 128); V staged in shared memory as
// fp32 when it fits, S in shared memory in binary64.
#include <cfloat>

#include "kernels.cuh"

namespace gwtk {

namespace {
constexpr int kOrthNT = 256;
}

template <bool VSMEM>
__global__ void __launch_bounds__(kOrthNT) k_orth_cholqr(int D, int count, float2* __restrict__ V) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* S = reinterpret_cast<double2*>(smem_raw);               // [count][count], upper used
    float2* sV = reinterpret_cast<float2*>(S + (size_t)count * count);  // [count][D] when VSMEM
    float2* Vb = V + (size_t)blockIdx.x * D * count;
    const int tid = threadIdx.x;
    const float2* src = Vb;
    if (VSMEM) {
        for (int e = tid; e < D * count; e += kOrthNT) sV[e] = Vb[e];
        __syncthreads();
        src = sV;
    }
    // S(j, k) = sum_i conj(V(i, j)) V(i, k), j <= k
    const int npair = count * (count + 1) / 2;
    for (int e = tid; e < npair; e += kOrthNT) {
        // e -> (j, k) with j <= k, row-major over the upper triangle
        int j = 0, rem = e;
        while (rem >= count - j) { rem -= count - j; ++j; }
        const int k = j + rem;
        const float2* vj = src + (size_t)j * D;
        const float2* vk = src + (size_t)k * D;
        double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
        int i = 0;
        for (; i + 1 < D; i += 2) {
            cfmaconj(a0, to_d2(vj[i]), to_d2(vk[i]));
            cfmaconj(a1, to_d2(vj[i + 1]), to_d2(vk[i + 1]));
        }
        if (i < D) cfmaconj(a0, to_d2(vj[i]), to_d2(vk[i]));
        S[j * count + k] = make_double2(a0.x + a1.x, a0.y + a1.y);
    }
    __syncthreads();
    // Cholesky S = R^H R in place (upper triangle), right-looking, one warp; R(k, k) real > 0
    if (tid < 32) {
        for (int k = 0; k < count; ++k) {
            const double d = S[k * count + k].x;
            const double rkk = d > 0.0 ? sqrt(d) : 1.0;  // S ~ I; a non-positive pivot leaves the column as is
            const double inv = 1.0 / rkk;
            __syncwarp();
            for (int c = k + 1 + tid; c < count; c += 32) {
                double2 v = S[k * count + c];
                S[k * count + c] = make_double2(v.x * inv, v.y * inv);
            }
            if (tid == 0) S[k * count + k] = make_double2(rkk, 0.0);
            __syncwarp();
            // trailing update: S(j, c) -= conj(R(k, j)) R(k, c), k < j <= c
            const int rem = count - k - 1;
            const int ntr = rem * (rem + 1) / 2;
            for (int e = tid; e < ntr; e += 32) {
                int j = 0, r2 = e;
                while (r2 >= rem - j) { r2 -= rem - j; ++j; }
                const int jj = k + 1 + j, cc = jj + r2;
                const double2 a = S[k * count + jj], b = S[k * count + cc];
                double2 v = S[jj * count + cc];
                v.x -= a.x * b.x + a.y * b.y;
                v.y -= a.x * b.y - a.y * b.x;
                S[jj * count + cc] = v;
            }
            __syncwarp();
        }
    }
    __syncthreads();
    // V <- V R^{-1}: row i solves x R = v (forward substitution over columns), in place — row i
    // of V is read and written by one thread only
    float2* dst = VSMEM ? sV : Vb;
    for (int i = tid; i < D; i += kOrthNT) {
#pragma unroll 1
        for (int k = 0; k < count; ++k) {
            double2 acc = to_d2(dst[(size_t)k * D + i]);
            for (int j = 0; j < k; ++j) {
                const double2 r = S[j * count + k];
                const double2 xj = to_d2(dst[(size_t)j * D + i]);
                acc.x -= xj.x * r.x - xj.y * r.y;
                acc.y -= xj.x * r.y + xj.y * r.x;
            }
            const double inv = 1.0 / S[k * count + k].x;
            dst[(size_t)k * D + i] = from_d2<float2>(make_double2(acc.x * inv, acc.y * inv));
        }
    }
    __syncthreads();
    if (VSMEM) {
        for (int e = tid; e < D * count; e += kOrthNT) Vb[e] = sV[e];
        __syncthreads();
    }
    // phase convention: the largest-magnitude entry of each column real positive (first on ties)
    const int warp = tid >> 5, lane = tid & 31;
    for (int k = warp; k < count; k += kOrthNT / 32) {
        float2* col = Vb + (size_t)k * D;
        double best = -1.0;
        int bi = 0;
        for (int i = lane; i < D; i += 32) {
            const float2 v = col[i];
            const double mag = (double)v.x * v.x + (double)v.y * v.y;
            if (mag > best) { best = mag; bi = i; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        const float2 vb = col[bi];
        __syncwarp();
        if (best > 0.0) {
            const double im = rsqrt(best);
            const double2 fac = make_double2(vb.x * im, -vb.y * im);
            for (int i = lane; i < D; i += 32) col[i] = from_d2<float2>(cmul(to_d2(col[i]), fac));
        }
    }
}

template <class S, class D>
__global__ void k_cplx_convert(const S* __restrict__ in, D* __restrict__ out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = mk((decltype(D{}.x))in[i].x, (decltype(D{}.x))in[i].y);
}

cudaError_t launch_cplx_widen(const void* in, void* out, int64_t n, cudaStream_t st) {
    const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
    k_cplx_convert<float2, double2><<<blocks, 256, 0, st>>>((const float2*)in, (double2*)out, n);
    return cudaGetLastError();
}
cudaError_t launch_cplx_narrow(const void* in, void* out, int64_t n, cudaStream_t st) {
    const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
    k_cplx_convert<double2, float2><<<blocks, 256, 0, st>>>((const double2*)in, (float2*)out, n);
    return cudaGetLastError();
}

cudaError_t launch_orth_cholqr(int D, int count, int64_t batch, void* V, cudaStream_t st) {
    if (D < 1 || count < 1 || count > 128 || count > D || batch < 1) return cudaErrorInvalidValue;
    const size_t s_bytes = sizeof(double2) * (size_t)count * count;
    const size_t v_bytes = sizeof(float2) * (size_t)count * D;
    const bool vs = s_bytes + v_bytes <= 200 * 1024;
    const size_t sm = s_bytes + (vs ? v_bytes : 0);
    cudaError_t e;
    if (vs) {
        e = cudaFuncSetAttribute(k_orth_cholqr<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
        k_orth_cholqr<true><<<(unsigned)batch, kOrthNT, sm, st>>>(D, count, (float2*)V);
    } else {
        e = cudaFuncSetAttribute(k_orth_cholqr<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
        k_orth_cholqr<false><<<(unsigned)batch, kOrthNT, sm, st>>>(D, count, (float2*)V);
    }
    return cudaGetLastError();
}

}  // namespace gwtk
