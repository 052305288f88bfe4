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

#include <map>
#include <mutex>
#include <string>

namespace gwtk {

const char* env_once(const char* name) {
    static std::mutex mu;
    static std::map<std::string, std::pair<bool, std::string>> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(name);
    if (it == cache.end()) {
        const char* v = std::getenv(name);
        it = cache.emplace(name, std::make_pair(v != nullptr, v ? std::string(v) : std::string())).first;
    }
    return it->second.first ? it->second.second.c_str() : nullptr;
}


// Tiled strided batched complex GEMM with conj(U) (GemmDesc): CTA tile TR rows x TC cols of one item,
// 256 threads as NR x NC (NR = TR/RT, NC = TC/CT), RT x CT outputs per thread. The global offsets of
// each thread's staging elements are computed once (no per-chunk div/mod); the next K chunk is
// prefetched into registers while the current one is multiplied out of shared memory. TC is matched
// to the factor rank (8/12/16/24/32/48/64/96) so narrow ranks do not pad a wide tile.
template <class T, int TR, int TC, int RT, int CT>
__global__ void __launch_bounds__(256) k_cgemm_conjU(Topo t, GemmDesc d, int links, int64_t item0,
                                                      const cplx_t<T>* __restrict__ in, const cplx_t<T>* __restrict__ U,
                                                      cplx_t<T>* __restrict__ out) {
    using C = cplx_t<T>;
    constexpr int KC = 16, NR = TR / RT, NC = TC / CT;
    static_assert(NR * NC == 256, "256 threads");
    constexpr int EI = TR * KC / 256, EU = (TC * KC + 255) / 256;
    __shared__ C sIn[KC][TR + 1];
    __shared__ C sU[KC][TC + 1];
    const int64_t item = item0 + blockIdx.z;
    const int64_t g = item / links;
    const int l = (int)(item % links);
    const int row0 = blockIdx.x * TR, col0 = blockIdx.y * TC;
    const int rows = d.R * d.S;
    const int tid = threadIdx.x;
    const C* inb = in + item * d.in_item;
    const int64_t ublk = d.ublk >= 0 ? d.ublk : (int64_t)d.Kd * d.Cols;
    const int64_t ucol = d.ucol >= 0 ? d.ucol : (int64_t)d.Kd;
    const C* ub = U + factor_index(t, d.fkind, g, l) * ublk;
    const bool row_fast = d.rs_in == 1;
    int64_t goff[EI];
    int ekk[EI];
    bool erok[EI];
#pragma unroll
    for (int e = 0; e < EI; ++e) {
        const int idx = tid + 256 * e;
        int r, kk;
        if (row_fast) { r = idx % TR; kk = idx / TR; }
        else { kk = idx % KC; r = idx / KC; }
        const int row = row0 + r;
        ekk[e] = kk;
        erok[e] = row < rows;
        goff[e] = erok[e] ? (row % d.R) * d.rs_in + (int64_t)(row / d.R) * d.s_in + (int64_t)kk * d.ks_in : 0;
    }
    int64_t uoff[EU];
    int ukk[EU], uc[EU];
    bool uok[EU];
#pragma unroll
    for (int e = 0; e < EU; ++e) {
        const int idx = tid + 256 * e;
        ukk[e] = idx % KC;
        uc[e] = idx / KC;
        const int col = col0 + uc[e];
        uok[e] = idx < TC * KC && col < d.Cols;
        uoff[e] = uok[e] ? (int64_t)ukk[e] * d.uk + (int64_t)col * ucol : 0;
    }
    C pin[EI], pu[EU];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int e = 0; e < EI; ++e) {
            pin[e] = czero<C>();
            if (erok[e] && k0 + ekk[e] < d.Kd) pin[e] = inb[goff[e] + (int64_t)k0 * d.ks_in];
        }
#pragma unroll
        for (int e = 0; e < EU; ++e) {
            pu[e] = czero<C>();
            if (uok[e] && k0 + ukk[e] < d.Kd) {
                pu[e] = ub[uoff[e] + (int64_t)k0 * d.uk];
                if (d.uconj) pu[e] = cconj(pu[e]);
            }
        }
    };
    const int tx = tid % NC, ty = tid / NC;
    C acc[RT][CT];
#pragma unroll
    for (int a = 0; a < RT; ++a)
#pragma unroll
        for (int b = 0; b < CT; ++b) acc[a][b] = czero<C>();
    fetch(0);
    for (int k0 = 0; k0 < d.Kd; k0 += KC) {
        __syncthreads();
#pragma unroll
        for (int e = 0; e < EI; ++e) {
            const int idx = tid + 256 * e;
            if (row_fast) sIn[idx / TR][idx % TR] = pin[e];
            else sIn[idx % KC][idx / KC] = pin[e];
        }
#pragma unroll
        for (int e = 0; e < EU; ++e) {
            const int idx = tid + 256 * e;
            if (idx < TC * KC) sU[idx % KC][idx / KC] = pu[e];
        }
        __syncthreads();
        if (k0 + KC < d.Kd) fetch(k0 + KC);
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) {
            C a[RT], b[CT];
#pragma unroll
            for (int q = 0; q < RT; ++q) a[q] = sIn[kk][ty + NR * q];
#pragma unroll
            for (int q = 0; q < CT; ++q) b[q] = sU[kk][tx + NC * q];
#pragma unroll
            for (int qa = 0; qa < RT; ++qa)
#pragma unroll
                for (int qb = 0; qb < CT; ++qb) cfma(acc[qa][qb], a[qa], b[qb]);
        }
    }
    C* ob = out + item * d.out_item;
#pragma unroll
    for (int qa = 0; qa < RT; ++qa) {
        const int row = row0 + ty + NR * qa;
        if (row >= rows) continue;
        const int64_t ro = (row % d.R) * d.rs_out + (int64_t)(row / d.R) * d.s_out;
#pragma unroll
        for (int qb = 0; qb < CT; ++qb) {
            const int col = col0 + tx + NC * qb;
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

// Batched Hermitian rank-k accumulation (GramDesc). CTA = (lower-triangle TD x TD tile, set, K split),
// TD = 16*Q, 256 threads with Q x Q outputs each. The set's flattened reduction index
// k = link_in_set * T + t is mapped to global offsets chunk by chunk (a KC-entry shared table built
// one chunk ahead), so the per-element staging has no div/mod; the next K chunk is prefetched into registers while the current one is
// multiplied. With nsplit > 1 each split writes its partial D x D Gram to `out + split * D*D*sets`
// and k_gram_reduce sums them in a fixed order (deterministic).
template <class T, int Q, int KC>
__global__ void __launch_bounds__(256) k_gram(Topo t, GramDesc d, int sets_per_group, int64_t set0, int nsplit,
                                              int kspan, const cplx_t<T>* __restrict__ V, cplx_t<T>* __restrict__ out,
                                              int64_t split_stride) {
    using C = cplx_t<T>;
    constexpr int TD = 16 * Q, EL = TD * KC / 256;
    __shared__ C sX[KC][TD + 1];
    __shared__ C sY[KC][TD + 1];
    __shared__ int64_t koff[2][KC];  // global offsets of the current / next K chunk
    const int64_t set = set0 + blockIdx.y;
    const int64_t g = set / sets_per_group;
    const int s = (int)(set % sets_per_group);
    // lower-triangle tile index -> (xt >= yt)
    int xt = 0, yt = 0;
    {
        int rem = blockIdx.x;
        while (rem > xt) {
            ++xt;
            rem -= xt;
        }
        yt = rem;
    }
    const int x0 = xt * TD, y0 = yt * TD;
    const bool diag = xt == yt;
    const int nl = set_size(t, d.set_kind);
    const int Tn = d.T1 * d.T2;
    const int64_t ktot = (int64_t)nl * Tn;
    const int64_t kb = (int64_t)blockIdx.z * kspan;
    const int kn = (int)std::max<int64_t>(0, std::min<int64_t>(kspan, ktot - kb));
    const C* vg = V + g * t.links() * d.v_item;
    auto offsets = [&](int k0, int64_t* dst) {  // threads < KC: offset table of chunk k0
        const int k = k0 + threadIdx.x;
        if (threadIdx.x < KC && k < kn) {
            const int64_t kf = kb + k;
            const int li = (int)(kf / Tn), tt = (int)(kf % Tn);
            const int l = set_link(t, d.set_kind, s, li);
            dst[threadIdx.x] = (int64_t)l * d.v_item + (int64_t)(tt % d.T1) * d.t1s + (int64_t)(tt / d.T1) * d.t2s;
        }
    };
    offsets(0, koff[0]);
    __syncthreads();
    const bool x_fast = d.xs == 1;
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    C px[EL], py[EL];
    auto fetch = [&](int k0, const int64_t* ko) {
#pragma unroll
        for (int e = 0; e < EL; ++e) {
            const int idx = tid + 256 * e;
            int xi, kk;
            if (x_fast) { xi = idx % TD; kk = idx / TD; }
            else { kk = idx % KC; xi = idx / KC; }
            const int k = k0 + kk;
            px[e] = czero<C>();
            py[e] = czero<C>();
            if (k < kn) {
                const C* vb = vg + ko[kk];
                if (x0 + xi < d.D) px[e] = vb[(int64_t)(x0 + xi) * d.xs];
                if (!diag && y0 + xi < d.D) py[e] = vb[(int64_t)(y0 + xi) * d.xs];
            }
        }
    };
    C acc[Q][Q];
#pragma unroll
    for (int a = 0; a < Q; ++a)
#pragma unroll
        for (int b = 0; b < Q; ++b) acc[a][b] = czero<C>();
    fetch(0, koff[0]);
    for (int k0 = 0, c = 0; k0 < kn; k0 += KC, ++c) {
        __syncthreads();
#pragma unroll
        for (int e = 0; e < EL; ++e) {
            const int idx = tid + 256 * e;
            int xi, kk;
            if (x_fast) { xi = idx % TD; kk = idx / TD; }
            else { kk = idx % KC; xi = idx / KC; }
            sX[kk][xi] = px[e];
            if (!diag) sY[kk][xi] = py[e];
        }
        if (k0 + KC < kn) offsets(k0 + KC, koff[(c + 1) & 1]);
        __syncthreads();
        if (k0 + KC < kn) fetch(k0 + KC, koff[(c + 1) & 1]);
        const C(*sB)[TD + 1] = diag ? sX : sY;
#pragma unroll 8
        for (int kk = 0; kk < KC; ++kk) {
            C a[Q], b[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                a[q] = sX[kk][ty + 16 * q];
                b[q] = sB[kk][tx + 16 * q];
            }
#pragma unroll
            for (int qa = 0; qa < Q; ++qa)
#pragma unroll
                for (int qb = 0; qb < Q; ++qb) cfmac(acc[qa][qb], a[qa], b[qb]);
        }
    }
    C* ob = out + blockIdx.z * split_stride + set * (int64_t)d.D * d.D;
#pragma unroll
    for (int qa = 0; qa < Q; ++qa) {
        const int x = x0 + ty + 16 * qa;
        if (x >= d.D) continue;
#pragma unroll
        for (int qb = 0; qb < Q; ++qb) {
            const int y = y0 + tx + 16 * qb;
            if (y >= d.D) continue;
            ob[x + (int64_t)d.D * y] = acc[qa][qb];
            if (!diag) ob[y + (int64_t)d.D * x] = cconj(acc[qa][qb]);
        }
    }
}

// out[e] = sum_{s < nsplit} part[s * stride + e], e < n (fixed order)
template <class T>
__global__ void k_gram_reduce(const cplx_t<T>* __restrict__ part, int nsplit, int64_t stride, int64_t n,
                              cplx_t<T>* __restrict__ out) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        cplx_t<T> acc = part[e];
        for (int s = 1; s < nsplit; ++s) acc = cadd(acc, part[s * stride + e]);
        out[e] = acc;
    }
}

// Thin mode-1 product (Kd = KD <= 8, Cols <= 8, fibers contiguous: ks_in == 1):
// one thread per fiber, conj(U) broadcast from shared memory. Used for X x1 A^H
// and Y1 x1 A^H, where the generic 64x64 tile would be >90% padding.
template <class T, int KD>
__global__ void __launch_bounds__(256) k_mode1_thin(Topo t, GemmDesc d, int links, const cplx_t<T>* __restrict__ in,
                                                    const cplx_t<T>* __restrict__ U, cplx_t<T>* __restrict__ out) {
    // grid (items, row blocks of 256): the item's conj(U) (KD x Cols <= 8) is staged in shared memory once
    using C = cplx_t<T>;
    __shared__ C su[KD][8];
    const int64_t item = blockIdx.x;
    const int rows = d.R * d.S;
    const int row = blockIdx.y * 256 + threadIdx.x;
    if (threadIdx.x < KD * 8) {
        const int kk = threadIdx.x % KD, c = threadIdx.x / KD;
        C u = czero<C>();
        if (c < d.Cols) {
            const int64_t g = item / links;
            const int l = (int)(item % links);
            const int64_t ublk = d.ublk >= 0 ? d.ublk : (int64_t)d.Kd * d.Cols;
            const int64_t ucol = d.ucol >= 0 ? d.ucol : (int64_t)d.Kd;
            u = U[factor_index(t, d.fkind, g, l) * ublk + (int64_t)kk * d.uk + (int64_t)c * ucol];
            if (d.uconj) u = cconj(u);
        }
        su[kk][c] = u;
    }
    __syncthreads();
    if (row >= rows) return;
    const int rr = d.S == 1 ? row : row % d.R, rs = d.S == 1 ? 0 : row / d.R;
    const C* x = in + item * d.in_item + (int64_t)rr * d.rs_in + (int64_t)rs * d.s_in;
    C xv[KD];
#pragma unroll
    for (int kk = 0; kk < KD; ++kk) xv[kk] = x[kk];
    C* o = out + item * d.out_item + (int64_t)rr * d.rs_out + (int64_t)rs * d.s_out;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        if (c >= d.Cols) break;
        C acc = czero<C>();
#pragma unroll
        for (int kk = 0; kk < KD; ++kk) cfma(acc, xv[kk], su[kk][c]);
        o[(int64_t)c * d.cs_out] = acc;
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

// Early stop on the device (decompose.cpp:363-368): after sweep s, group g stops when
// trace[s] - trace[s+1] < 1e-10 * energy (NaN never stops, as on the host); its factors and core
// are copied to `frozen` at that point and restored by k_unfreeze after the last sweep, so the
// host never synchronises per sweep. stop = [G flags][G iterations_run][1 stopped count].
__global__ void k_stop_freeze(int64_t ngroups, const double* __restrict__ trace, const double* __restrict__ energy,
                              int stride, int s, int* __restrict__ stop, const char* __restrict__ A,
                              const char* __restrict__ B, const char* __restrict__ Cf, const char* __restrict__ Gc,
                              char* __restrict__ frozen, int64_t a_sz, int64_t b_sz, int64_t c_sz, int64_t g_sz) {
    const int64_t g = blockIdx.x;
    // stopped at an earlier sweep? (iterations_run is written as s+1 by this launch's block y = 0, so
    // the other blocks of this launch still see the group as running and copy their slices)
    const int itr = stop[ngroups + g];
    if (itr != 0 && itr <= s) return;
    const double dec = trace[g * stride + s] - trace[g * stride + s + 1];
    if (!(dec < 1e-10 * energy[g])) return;
    // byte sizes are multiples of 8 (complex64 and up)
    const int64_t tot = a_sz + b_sz + c_sz + g_sz;
    unsigned long long* fz = reinterpret_cast<unsigned long long*>(frozen + g * tot);
    const int64_t na = a_sz / 8, nb = b_sz / 8, nc = c_sz / 8, ng = g_sz / 8;
    const unsigned long long* sa = reinterpret_cast<const unsigned long long*>(A + g * a_sz);
    const unsigned long long* sb = reinterpret_cast<const unsigned long long*>(B + g * b_sz);
    const unsigned long long* sc = reinterpret_cast<const unsigned long long*>(Cf + g * c_sz);
    const unsigned long long* sg = reinterpret_cast<const unsigned long long*>(Gc + g * g_sz);
    const int64_t step = (int64_t)blockDim.x * gridDim.y;
    for (int64_t e = threadIdx.x + (int64_t)blockIdx.y * blockDim.x; e < na + nb + nc + ng; e += step)
        fz[e] = e < na ? sa[e] : e < na + nb ? sb[e - na] : e < na + nb + nc ? sc[e - na - nb] : sg[e - na - nb - nc];
    // the slices of the copy run in gridDim.y blocks; block y = 0 publishes the stop after its slice.
    // Other slices may still be copying when the flag is set: readers of the flag (k_unfreeze, the
    // next sweep's k_stop_freeze) run later on the same stream, after this whole grid completed.
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.y == 0) {
        stop[g] = 1;
        stop[ngroups + g] = s + 1;
        atomicAdd(stop + 2 * ngroups, 1);
    }
}

__global__ void k_unfreeze(int64_t ngroups, const int* __restrict__ stop, char* __restrict__ A, char* __restrict__ B,
                           char* __restrict__ Cf, char* __restrict__ Gc, const char* __restrict__ frozen, int64_t a_sz,
                           int64_t b_sz, int64_t c_sz, int64_t g_sz) {
    const int64_t g = blockIdx.x;
    if (!stop[g]) return;
    const int64_t tot = a_sz + b_sz + c_sz + g_sz;
    const unsigned long long* fz = reinterpret_cast<const unsigned long long*>(frozen + g * tot);
    const int64_t na = a_sz / 8, nb = b_sz / 8, nc = c_sz / 8, ng = g_sz / 8;
    unsigned long long* da = reinterpret_cast<unsigned long long*>(A + g * a_sz);
    unsigned long long* db = reinterpret_cast<unsigned long long*>(B + g * b_sz);
    unsigned long long* dc = reinterpret_cast<unsigned long long*>(Cf + g * c_sz);
    unsigned long long* dg = reinterpret_cast<unsigned long long*>(Gc + g * g_sz);
    for (int64_t e = threadIdx.x + (int64_t)blockIdx.y * blockDim.x; e < na + nb + nc + ng;
         e += (int64_t)blockDim.x * gridDim.y) {
        const unsigned long long v = fz[e];
        if (e < na) da[e] = v;
        else if (e < na + nb) db[e - na] = v;
        else if (e < na + nb + nc) dc[e - na - nb] = v;
        else dg[e - na - nb - nc] = v;
    }
}

cudaError_t launch_stop_freeze(int64_t ngroups, const double* trace, const double* energy, int stride, int s, int* stop,
                               const void* A, const void* B, const void* Cf, const void* Gc, void* frozen, int64_t a_sz,
                               int64_t b_sz, int64_t c_sz, int64_t g_sz, cudaStream_t st) {
    const int64_t words = (a_sz + b_sz + c_sz + g_sz) / 8;
    const dim3 grid((unsigned)ngroups, (unsigned)std::max<int64_t>(1, std::min<int64_t>(32, (words + 2047) / 2048)));
    k_stop_freeze<<<grid, 256, 0, st>>>(ngroups, trace, energy, stride, s, stop, (const char*)A,
                                                      (const char*)B, (const char*)Cf, (const char*)Gc, (char*)frozen,
                                                      a_sz, b_sz, c_sz, g_sz);
    return cudaGetLastError();
}

cudaError_t launch_unfreeze(int64_t ngroups, const int* stop, void* A, void* B, void* Cf, void* Gc, const void* frozen,
                            int64_t a_sz, int64_t b_sz, int64_t c_sz, int64_t g_sz, cudaStream_t st) {
    const int64_t words = (a_sz + b_sz + c_sz + g_sz) / 8;
    const dim3 grid((unsigned)ngroups, (unsigned)std::max<int64_t>(1, std::min<int64_t>(32, (words + 2047) / 2048)));
    k_unfreeze<<<grid, 256, 0, st>>>(ngroups, stop, (char*)A, (char*)B, (char*)Cf, (char*)Gc,
                                                   (const char*)frozen, a_sz, b_sz, c_sz, g_sz);
    return cudaGetLastError();
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
        dim3 grid((unsigned)items, (unsigned)((d.R * d.S + 255) / 256));
        switch (d.Kd) {
#define GWT_THIN(KK) \
    case KK: k_mode1_thin<T, KK><<<grid, 256, 0, st>>>(t, d, t.links(), (const cplx_t<T>*)in, (const cplx_t<T>*)U, (cplx_t<T>*)out); break;
            GWT_THIN(1) GWT_THIN(2) GWT_THIN(3) GWT_THIN(4) GWT_THIN(5) GWT_THIN(6) GWT_THIN(7) GWT_THIN(8)
#undef GWT_THIN
        }
        return cudaGetLastError();
    }
    const int64_t items = ngroups * t.links();
    const int rows = d.R * d.S;
    const cplx_t<T>* a = (const cplx_t<T>*)in;
    const cplx_t<T>* u = (const cplx_t<T>*)U;
    cplx_t<T>* o = (cplx_t<T>*)out;
#define GWT_GEMM(TR_, TC_, RT_, CT_)                                                                      \
    for (int64_t i0 = 0; i0 < items; i0 += 65535) {                                                       \
        dim3 grid((rows + TR_ - 1) / TR_, (d.Cols + TC_ - 1) / TC_, (unsigned)std::min<int64_t>(65535, items - i0)); \
        k_cgemm_conjU<T, TR_, TC_, RT_, CT_><<<grid, 256, 0, st>>>(t, d, t.links(), i0, a, u, o);          \
    }
    // short items (rows <= 64, e.g. W = Y1 x2 B^H with M*p = 48 rows at C2): 64-row tiles instead of
    // 128-row tiles that would run 60 % empty
    static const bool tr64 = !(env_once("GWT_GEMM_TR64") && std::atoi(env_once("GWT_GEMM_TR64")) == 0);
    if (tr64 && rows <= 64 && d.Cols <= 32) {
        if (d.Cols <= 8) GWT_GEMM(64, 8, 1, 2)
        else if (d.Cols <= 12) GWT_GEMM(64, 12, 1, 3)
        else if (d.Cols <= 16) GWT_GEMM(64, 16, 1, 4)
        else if (d.Cols <= 24) GWT_GEMM(64, 24, 2, 3)
        else GWT_GEMM(64, 32, 2, 4)
        return cudaGetLastError();
    }
    if (d.Cols <= 8) GWT_GEMM(128, 8, 2, 2)
    else if (d.Cols <= 12) GWT_GEMM(128, 12, 2, 3)
    else if (d.Cols <= 16) GWT_GEMM(128, 16, 2, 4)
    else if (d.Cols <= 24) GWT_GEMM(128, 24, 4, 3)
    else if (d.Cols <= 32) GWT_GEMM(128, 32, 4, 4)
    else if (d.Cols <= 48) GWT_GEMM(64, 48, 4, 3)
    else if (d.Cols <= 64) GWT_GEMM(64, 64, 4, 4)
    else GWT_GEMM(64, 96, 4, 6)
#undef GWT_GEMM
    return cudaGetLastError();
}

template <class T>
cudaError_t launch_gram(const Topo& t, const GramDesc& d, int64_t ngroups, int sets_per_group, const void* V, void* out,
                        void* part, size_t part_bytes, cudaStream_t st, bool allow_tc) {
    // complex64 Grams whose rows are contiguous blocks (the tx Gram of W2, N >= 128: C3, C4, C5) on the tensor
    // cores (k_tc.cu, TMA bulk-staged 3xTF32); GWT_GRAM_TC=0 keeps the CUDA-core kernel
    if (sizeof(T) == 4 && allow_tc && gram_tc_fits(d)) return launch_gram_tc(t, d, ngroups, sets_per_group, V, out, st);
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
    const int64_t sets = ngroups * sets_per_group;
    const int nl = d.set_kind == FI_USER ? t.J : d.set_kind == FI_BASE ? t.J * t.K : d.set_kind == FI_LINK ? 1 : t.links();
    const int64_t ktot = (int64_t)nl * d.T1 * d.T2;
    auto run = [&](auto kern, int TD, int KC) -> cudaError_t {
        const int tiles = (d.D + TD - 1) / TD, ntl = tiles * (tiles + 1) / 2;
        // K split: aim for >= 4 CTAs per SM, at least 8 chunks per split, limited by the partial buffer
        int nsplit = 1;
        const int64_t ctas = sets * ntl;
        if (part && ctas < 148 * 4) {
            // >= 2 chunks of KC per split (was 8): C2's per-sweep tx Grams (32 sets per lane, K = 384)
            // now split 6 ways instead of running 32 CTAs
            static const int minch = env_once("GWT_GRAM_MINCH") ? std::max(1, std::atoi(env_once("GWT_GRAM_MINCH"))) : 2;
            nsplit = (int)std::min<int64_t>((148 * 4 + ctas - 1) / ctas, std::max<int64_t>(1, ktot / (minch * KC)));
            const int64_t cap = (int64_t)(part_bytes / (sizeof(cplx_t<T>) * (size_t)d.D * d.D * sets));
            nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(nsplit, cap));
        }
        int kspan = (int)((ktot + nsplit - 1) / nsplit);
        kspan = (kspan + KC - 1) / KC * KC;
        nsplit = (int)((ktot + kspan - 1) / kspan);
        cplx_t<T>* dst = nsplit > 1 ? (cplx_t<T>*)part : (cplx_t<T>*)out;
        const int64_t stride = sets * (int64_t)d.D * d.D;
        for (int64_t s0 = 0; s0 < sets; s0 += 65535) {
            dim3 grid(ntl, (unsigned)std::min<int64_t>(65535, sets - s0), nsplit);
            kern<<<grid, 256, 0, st>>>(t, d, sets_per_group, s0, nsplit, kspan, (const cplx_t<T>*)V, dst, stride);
        }
        if (nsplit > 1) {
            const unsigned blocks = (unsigned)std::min<int64_t>((stride + 255) / 256, 148 * 16);
            k_gram_reduce<T><<<blocks, 256, 0, st>>>((const cplx_t<T>*)part, nsplit, stride, stride, (cplx_t<T>*)out);
        }
        return cudaGetLastError();
    };
    constexpr int KCb = sizeof(T) == 4 ? 32 : 16;
    // 32 x 32 lower-triangle tiles up to D = 64 (3 tiles instead of one full 64 x 64: 25 % less work,
    // 3x the CTAs; C2 Tucker 16.9 -> 16.2 ms with the split above); 64 x 64 tiles beyond
    static const char* td = env_once("GWT_GRAM_TD");
    const int tdmax = td ? std::atoi(td) : 64;
    if (d.D <= 32 || d.D <= tdmax) return run(k_gram<T, 2, KCb>, 32, KCb);
    return run(k_gram<T, 4, KCb>, 64, KCb);
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
    template cudaError_t launch_gram<T>(const Topo&, const GramDesc&, int64_t, int, const void*, void*, void*,   \
                                        size_t, cudaStream_t, bool);                                                 \
    template cudaError_t launch_group_sqnorm<T>(const void*, int64_t, int64_t, double*, double*, cudaStream_t);          \
    template cudaError_t launch_broadcast<T>(const void*, void*, int64_t, int, int64_t, cudaStream_t);
GWT_INST(float)
GWT_INST(double)

}  // namespace gwtk
