// Groupwise Tucker compression (hot path a) building blocks, sm_100a.
//
// Reference: alternating_solve (proj/src/decompose.cpp:309-373) over
// rx/tx/delay_update_gram (:146-193), initial_factors (:248-300),
// compute_cores (:195-204), objective_value (:217-226). The reference forms
// each mode product through an explicit unfolding copy (tensor.cpp:36-114);
// here every mode product is ONE strided batched complex GEMM whose operand
// strides address the unfolding in place (no copies), batched over all links
// of all groups, and every update Gram is one batched Hermitian rank-k kernel
// whose reduction runs over all links that share the factor.
#include <cstdlib>

#include "kernels.cuh"

namespace gwtk {

// Tiled strided complex GEMM with conj(U): CTA tile (16*RT) rows x (16*CT) cols, 256 threads
// (16 x 16), RT x CT outputs per thread, K chunks of 16 staged in smem. The tile shape is picked
// per call from Cols (12/24-wide factor ranks would waste most of a 64-wide tile).
template <class T, int RT, int CT>
__global__ void __launch_bounds__(256) k_cgemm_conjU(Topo t, GemmDesc d, int links, const cplx_t<T>* __restrict__ in,
                                                      const cplx_t<T>* __restrict__ U, cplx_t<T>* __restrict__ out) {
    using C = cplx_t<T>;
    constexpr int TR = 16 * RT, TC = 16 * CT, KC = 16;
    __shared__ C sIn[KC][TR + 1];
    __shared__ C sU[KC][TC + 1];
    const int64_t item = blockIdx.z;
    const int64_t g = item / links;
    const int l = (int)(item % links);
    const int row0 = blockIdx.x * TR, col0 = blockIdx.y * TC;
    const int rows = d.R * d.S;
    const C* inb = in + item * d.in_item;
    const int64_t ublk = d.ublk >= 0 ? d.ublk : (int64_t)d.Kd * d.Cols;
    const int64_t ucol = d.ucol >= 0 ? d.ucol : (int64_t)d.Kd;
    const C* ub = U + factor_index(t, d.fkind, g, l) * ublk;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    C acc[RT][CT];
#pragma unroll
    for (int a = 0; a < RT; ++a)
#pragma unroll
        for (int b = 0; b < CT; ++b) acc[a][b] = czero<C>();
    const bool row_fast = d.rs_in == 1;
    for (int k0 = 0; k0 < d.Kd; k0 += KC) {
        for (int idx = threadIdx.x; idx < TR * KC; idx += 256) {
            int r, kk;
            if (row_fast) { r = idx % TR; kk = idx / TR; }
            else { kk = idx % KC; r = idx / KC; }
            const int row = row0 + r, k = k0 + kk;
            C v = czero<C>();
            if (row < rows && k < d.Kd)
                v = inb[(row % d.R) * d.rs_in + (int64_t)(row / d.R) * d.s_in + (int64_t)k * d.ks_in];
            sIn[kk][r] = v;
        }
        for (int idx = threadIdx.x; idx < TC * KC; idx += 256) {
            const int kk = idx % KC, c = idx / KC;
            const int col = col0 + c, k = k0 + kk;
            C v = czero<C>();
            if (col < d.Cols && k < d.Kd) {
                v = ub[(int64_t)k * d.uk + (int64_t)col * ucol];
                if (d.uconj) v = cconj(v);
            }
            sU[kk][c] = v;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) {
            C a[RT], b[CT];
#pragma unroll
            for (int q = 0; q < RT; ++q) a[q] = sIn[kk][ty + 16 * q];
#pragma unroll
            for (int q = 0; q < CT; ++q) b[q] = sU[kk][tx + 16 * q];
#pragma unroll
            for (int qa = 0; qa < RT; ++qa)
#pragma unroll
                for (int qb = 0; qb < CT; ++qb) cfma(acc[qa][qb], a[qa], b[qb]);
        }
        __syncthreads();
    }
    C* ob = out + item * d.out_item;
#pragma unroll
    for (int qa = 0; qa < RT; ++qa) {
        const int row = row0 + ty + 16 * qa;
        if (row >= rows) continue;
        const int64_t ro = (row % d.R) * d.rs_out + (int64_t)(row / d.R) * d.s_out;
#pragma unroll
        for (int qb = 0; qb < CT; ++qb) {
            const int col = col0 + tx + 16 * qb;
            if (col < d.Cols) ob[ro + (int64_t)col * d.cs_out] = acc[qa][qb];
        }
    }
}

__device__ __forceinline__ int set_size(const Topo& t, int kind) {
    switch (kind) {
        case FI_USER: return t.J;
        case FI_BASE: return t.J * t.K;
        case FI_LINK: return 1;
        default: return t.links();
    }
}
// r-th link of set `s` (s local to its group)
__device__ __forceinline__ int set_link(const Topo& t, int kind, int s, int r) {
    switch (kind) {
        case FI_USER: {  // s = i*K + j, r = k
            const int i = s / t.K, j = s % t.K;
            return (r * t.J + i) * t.K + j;
        }
        case FI_BASE: return s * t.J * t.K + r;  // links (s, i, j) contiguous
        case FI_LINK: return s;
        default: return r;
    }
}

// Batched Hermitian rank-k accumulation: CTA per (set, TD x TD output tile), TD = 16*Q.
template <class T, int Q>
__global__ void __launch_bounds__(256) k_gram(Topo t, GramDesc d, int sets_per_group, const cplx_t<T>* __restrict__ V,
                                              cplx_t<T>* __restrict__ out) {
    using C = cplx_t<T>;
    constexpr int TD = 16 * Q, KC = 16;
    __shared__ C sX[KC][TD + 1];
    __shared__ C sY[KC][TD + 1];
    const int64_t set = blockIdx.y;
    const int64_t g = set / sets_per_group;
    const int s = (int)(set % sets_per_group);
    const int tiles = (d.D + TD - 1) / TD;
    const int x0 = (blockIdx.x % tiles) * TD, y0 = (blockIdx.x / tiles) * TD;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    C acc[Q][Q];
#pragma unroll
    for (int a = 0; a < Q; ++a)
#pragma unroll
        for (int b = 0; b < Q; ++b) acc[a][b] = czero<C>();
    const int nl = set_size(t, d.set_kind);
    const int Tn = d.T1 * d.T2;
    const bool x_fast = d.xs == 1;
    for (int r = 0; r < nl; ++r) {
        const int l = set_link(t, d.set_kind, s, r);
        const C* vb = V + (g * t.links() + l) * d.v_item;
        for (int t0 = 0; t0 < Tn; t0 += KC) {
            for (int idx = threadIdx.x; idx < TD * KC; idx += 256) {
                int xi, kk;
                if (x_fast) { xi = idx % TD; kk = idx / TD; }
                else { kk = idx % KC; xi = idx / KC; }
                const int tt = t0 + kk;
                C vx = czero<C>(), vy = czero<C>();
                if (tt < Tn) {
                    const int64_t toff = (int64_t)(tt % d.T1) * d.t1s + (int64_t)(tt / d.T1) * d.t2s;
                    if (x0 + xi < d.D) vx = vb[(int64_t)(x0 + xi) * d.xs + toff];
                    if (y0 + xi < d.D) vy = vb[(int64_t)(y0 + xi) * d.xs + toff];
                }
                sX[kk][xi] = vx;
                sY[kk][xi] = vy;
            }
            __syncthreads();
#pragma unroll
            for (int kk = 0; kk < KC; ++kk) {
                C a[Q], b[Q];
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    a[q] = sX[kk][ty + 16 * q];
                    b[q] = sY[kk][tx + 16 * q];
                }
#pragma unroll
                for (int qa = 0; qa < Q; ++qa)
#pragma unroll
                    for (int qb = 0; qb < Q; ++qb) cfmac(acc[qa][qb], a[qa], b[qb]);
            }
            __syncthreads();
        }
    }
    C* ob = out + set * (int64_t)d.D * d.D;
#pragma unroll
    for (int qa = 0; qa < Q; ++qa) {
        const int x = x0 + ty + 16 * qa;
        if (x >= d.D) continue;
#pragma unroll
        for (int qb = 0; qb < Q; ++qb) {
            const int y = y0 + tx + 16 * qb;
            if (y < d.D) ob[x + (int64_t)d.D * y] = acc[qa][qb];
        }
    }
}

// Thin mode-1 product (Kd = KD <= 8, Cols <= 8, fibers contiguous: ks_in == 1):
// one thread per fiber, conj(U) broadcast from shared memory. Used for X x1 A^H
// and Y1 x1 A^H, where the generic 64x64 tile would be >90% padding.
template <class T, int KD>
__global__ void __launch_bounds__(256) k_mode1_thin(Topo t, GemmDesc d, int links, int64_t items,
                                                    const cplx_t<T>* __restrict__ in, const cplx_t<T>* __restrict__ U,
                                                    cplx_t<T>* __restrict__ out) {
    using C = cplx_t<T>;
    const int rows = d.R * d.S;
    const int64_t total = items * rows;
    const int64_t ublk = d.ublk >= 0 ? d.ublk : (int64_t)d.Kd * d.Cols;
    const int64_t ucol = d.ucol >= 0 ? d.ucol : (int64_t)d.Kd;
    for (int64_t gidx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gidx < total;
         gidx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t item = gidx / rows;
        const int row = (int)(gidx % rows);
        const int64_t g = item / links;
        const int l = (int)(item % links);
        const C* ub = U + factor_index(t, d.fkind, g, l) * ublk;
        const C* x = in + item * d.in_item + (row % d.R) * d.rs_in + (int64_t)(row / d.R) * d.s_in;
        C xv[KD];
#pragma unroll
        for (int kk = 0; kk < KD; ++kk) xv[kk] = x[kk];
        C* o = out + item * d.out_item + (row % d.R) * d.rs_out + (int64_t)(row / d.R) * d.s_out;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (c >= d.Cols) break;
            C acc = czero<C>();
#pragma unroll
            for (int kk = 0; kk < KD; ++kk) {
                C u = ub[(int64_t)kk * d.uk + (int64_t)c * ucol];
                if (d.uconj) u = cconj(u);
                cfma(acc, xv[kk], u);
            }
            o[(int64_t)c * d.cs_out] = acc;
        }
    }
}

// Thin Gram (D = MD <= 8, x fastest: xs == 1): one CTA per set; each thread
// accumulates a private MD x MD partial over strided columns, then a fixed-order
// shared-memory tree reduction (deterministic).
template <class T, int MD>
__global__ void __launch_bounds__(128) k_gram_thin(Topo t, GramDesc d, int sets_per_group,
                                                  const cplx_t<T>* __restrict__ V, cplx_t<T>* __restrict__ out) {
    using C = cplx_t<T>;
    using R = decltype(C{}.x);
    constexpr int NE = MD * (MD + 1) / 2;
    __shared__ C red[4][NE];
    const int64_t set = blockIdx.x;
    const int64_t g = set / sets_per_group;
    const int s = (int)(set % sets_per_group);
    C acc[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) acc[e] = czero<C>();
    const int nl = set_size(t, d.set_kind);
    const int Tn = d.T1 * d.T2;
    for (int r = 0; r < nl; ++r) {
        const int l = set_link(t, d.set_kind, s, r);
        const C* vb = V + (g * t.links() + l) * d.v_item;
        for (int tt = threadIdx.x; tt < Tn; tt += blockDim.x) {
            const C* col = vb + (int64_t)(tt % d.T1) * d.t1s + (int64_t)(tt / d.T1) * d.t2s;
            C x[MD];
#pragma unroll
            for (int a = 0; a < MD; ++a) x[a] = col[a];
            int e = 0;
#pragma unroll
            for (int a = 0; a < MD; ++a)
#pragma unroll
                for (int b = a; b < MD; ++b) cfmac(acc[e++], x[a], x[b]);
        }
    }
#pragma unroll
    for (int e = 0; e < NE; ++e) {
        for (int o = 16; o > 0; o >>= 1) {
            acc[e].x += __shfl_xor_sync(0xffffffffu, acc[e].x, o);
            acc[e].y += __shfl_xor_sync(0xffffffffu, acc[e].y, o);
        }
        if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32][e] = acc[e];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        C* ob = out + set * (int64_t)MD * MD;
        int e = 0;
        for (int a = 0; a < MD; ++a)
            for (int b = a; b < MD; ++b, ++e) {
                const C v = cadd(cadd(red[0][e], red[1][e]), cadd(red[2][e], red[3][e]));
                ob[a + MD * b] = v;
                ob[b + MD * a] = mk((R)v.x, (R)-v.y);
            }
    }
}

// Per-group sum of |v|^2 over `per_group` contiguous complex elements:
// deterministic (fixed tree), fp64 accumulation. One CTA per group.
template <class T>
__global__ void __launch_bounds__(256) k_group_sqnorm(const cplx_t<T>* __restrict__ v, int64_t per_group,
                                                      double* __restrict__ out) {
    // grid (groups, blocks per group): block b of group g sums a contiguous slice; out[g * gridDim.y + b]
    const int64_t g = blockIdx.x;
    const int64_t slice = (per_group + gridDim.y - 1) / gridDim.y;
    const int64_t e0 = (int64_t)blockIdx.y * slice, e1 = std::min(per_group, e0 + slice);
    const cplx_t<T>* b = v + g * per_group;
    double acc = 0.0;
    for (int64_t e = e0 + threadIdx.x; e < e1; e += 256) {
        const double2 x = to_d2(b[e]);
        acc += x.x * x.x + x.y * x.y;
    }
    __shared__ double red[256];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[g * gridDim.y + blockIdx.y] = red[0];
}

__global__ void k_sum_partials(const double* __restrict__ part, int nb, double* __restrict__ out) {
    const int64_t g = blockIdx.x;
    __shared__ double red[kSqnormMaxBlocks];
    red[threadIdx.x] = threadIdx.x < nb ? part[g * nb + threadIdx.x] : 0.0;
    __syncthreads();
    for (int w = kSqnormMaxBlocks / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[g] = red[0];
}

// trace[g*(stride) + slot] = energy[g] - captured[g]
__global__ void k_objective(int64_t ngroups, const double* __restrict__ energy, const double* __restrict__ captured,
                            double* __restrict__ trace, int stride, int slot) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g < ngroups) trace[g * stride + slot] = energy[g] - captured[g];
}

// Broadcast one factor per group to `copies` slots per group (shared model).
template <class T>
__global__ void k_broadcast(const cplx_t<T>* __restrict__ src, cplx_t<T>* __restrict__ dst, int64_t elems, int copies,
                            int64_t ngroups) {
    const int64_t total = ngroups * copies * elems;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = e / (copies * elems);
        dst[e] = src[g * elems + e % elems];
    }
}

// ---------------------------------------------------------------------------
template <class T>
cudaError_t launch_cgemm(const Topo& t, const GemmDesc& d, int64_t ngroups, const void* in, const void* U, void* out,
                         cudaStream_t st) {
    if (d.ks_in == 1 && d.Kd <= 8 && d.Cols <= 8) {
        const int64_t items = ngroups * t.links();
        const int64_t total = items * d.R * d.S;
        const unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 32);
        switch (d.Kd) {
#define GWT_THIN(KK) \
    case KK: k_mode1_thin<T, KK><<<blocks, 256, 0, st>>>(t, d, t.links(), items, (const cplx_t<T>*)in, (const cplx_t<T>*)U, (cplx_t<T>*)out); break;
            GWT_THIN(1) GWT_THIN(2) GWT_THIN(3) GWT_THIN(4) GWT_THIN(5) GWT_THIN(6) GWT_THIN(7) GWT_THIN(8)
#undef GWT_THIN
        }
        return cudaGetLastError();
    }
    const unsigned items = (unsigned)(ngroups * t.links());
    const int rows = d.R * d.S;
    if (d.Cols <= 16) {
        dim3 grid((rows + 127) / 128, (d.Cols + 15) / 16, items);
        k_cgemm_conjU<T, 8, 1><<<grid, 256, 0, st>>>(t, d, t.links(), (const cplx_t<T>*)in, (const cplx_t<T>*)U,
                                                      (cplx_t<T>*)out);
    } else if (d.Cols <= 32) {
        dim3 grid((rows + 63) / 64, (d.Cols + 31) / 32, items);
        k_cgemm_conjU<T, 4, 2><<<grid, 256, 0, st>>>(t, d, t.links(), (const cplx_t<T>*)in, (const cplx_t<T>*)U,
                                                      (cplx_t<T>*)out);
    } else {
        dim3 grid((rows + 63) / 64, (d.Cols + 63) / 64, items);
        k_cgemm_conjU<T, 4, 4><<<grid, 256, 0, st>>>(t, d, t.links(), (const cplx_t<T>*)in, (const cplx_t<T>*)U,
                                                      (cplx_t<T>*)out);
    }
    return cudaGetLastError();
}

template <class T>
cudaError_t launch_gram(const Topo& t, const GramDesc& d, int64_t ngroups, int sets_per_group, const void* V, void* out,
                        cudaStream_t st) {
    // complex64 Grams with D >= 64 on the tensor cores (3xTF32 tcgen05, k_tc.cu): opt-in (GWT_GRAM_TC=1)
    // until its staging pipeline beats the CUDA-core kernel
    if (sizeof(T) == 4 && d.D >= 64) {
        const char* e = std::getenv("GWT_GRAM_TC");
        if (e && std::atoi(e) != 0) return launch_gram_tc(t, d, ngroups, sets_per_group, V, out, st);
    }
    if (d.D <= 8 && d.xs == 1) {
        const unsigned blocks = (unsigned)(ngroups * sets_per_group);
        switch (d.D) {
#define GWT_GT(DD) \
    case DD: k_gram_thin<T, DD><<<blocks, 128, 0, st>>>(t, d, sets_per_group, (const cplx_t<T>*)V, (cplx_t<T>*)out); break;
            GWT_GT(1) GWT_GT(2) GWT_GT(3) GWT_GT(4) GWT_GT(5) GWT_GT(6) GWT_GT(7) GWT_GT(8)
#undef GWT_GT
        }
        return cudaGetLastError();
    }
    if (d.D <= 32) {
        const int tiles = (d.D + 31) / 32;
        dim3 grid(tiles * tiles, (unsigned)(ngroups * sets_per_group));
        k_gram<T, 2><<<grid, 256, 0, st>>>(t, d, sets_per_group, (const cplx_t<T>*)V, (cplx_t<T>*)out);
    } else {
        const int tiles = (d.D + 63) / 64;
        dim3 grid(tiles * tiles, (unsigned)(ngroups * sets_per_group));
        k_gram<T, 4><<<grid, 256, 0, st>>>(t, d, sets_per_group, (const cplx_t<T>*)V, (cplx_t<T>*)out);
    }
    return cudaGetLastError();
}

template <class T>
cudaError_t launch_group_sqnorm(const void* v, int64_t per_group, int64_t ngroups, double* out, double* partial,
                                cudaStream_t st) {
    // enough blocks to fill the GPU (~8 per SM), at least 16K elements each, at most kSqnormMaxBlocks per group
    int64_t nb = std::min<int64_t>((per_group + 16383) / 16384, (148 * 8 + ngroups - 1) / ngroups);
    nb = std::max<int64_t>(1, std::min<int64_t>(nb, kSqnormMaxBlocks));
    if (nb == 1) {
        k_group_sqnorm<T><<<dim3((unsigned)ngroups, 1), 256, 0, st>>>((const cplx_t<T>*)v, per_group, out);
        return cudaGetLastError();
    }
    k_group_sqnorm<T><<<dim3((unsigned)ngroups, (unsigned)nb), 256, 0, st>>>((const cplx_t<T>*)v, per_group, partial);
    k_sum_partials<<<(unsigned)ngroups, kSqnormMaxBlocks, 0, st>>>(partial, (int)nb, out);
    return cudaGetLastError();
}

cudaError_t launch_objective(int64_t ngroups, const double* energy, const double* captured, double* trace, int stride,
                             int slot, cudaStream_t st) {
    k_objective<<<(unsigned)((ngroups + 255) / 256), 256, 0, st>>>(ngroups, energy, captured, trace, stride, slot);
    return cudaGetLastError();
}

template <class T>
cudaError_t launch_broadcast(const void* src, void* dst, int64_t elems, int copies, int64_t ngroups, cudaStream_t st) {
    const int64_t total = ngroups * copies * elems;
    const unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
    k_broadcast<T><<<blocks, 256, 0, st>>>((const cplx_t<T>*)src, (cplx_t<T>*)dst, elems, copies, ngroups);
    return cudaGetLastError();
}

#define GWT_INST(T)                                                                                          \
    template cudaError_t launch_cgemm<T>(const Topo&, const GemmDesc&, int64_t, const void*, const void*, void*, \
                                         cudaStream_t);                                                      \
    template cudaError_t launch_gram<T>(const Topo&, const GramDesc&, int64_t, int, const void*, void*,          \
                                        cudaStream_t);                                                       \
    template cudaError_t launch_group_sqnorm<T>(const void*, int64_t, int64_t, double*, double*, cudaStream_t);          \
    template cudaError_t launch_broadcast<T>(const void*, void*, int64_t, int, int64_t, cudaStream_t);
GWT_INST(float)
GWT_INST(double)

}  // namespace gwtk
