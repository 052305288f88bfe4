// Stage R fused with the pair Grams of stage S on the 5th-gen tensor cores (c64, paper_experiment
// scope): H~ never reaches HBM.
//
// Reference: assemble_channel_compressed (proj/src/channel.cpp:189-208) for the links of one user,
// H~_l(f) = G_l x3 conj(d_l(f)), d_l = C_l^H c_l(f), followed by the products the SINR stage takes
// of them (proj/src/sinr.cpp:162-254 through the Gram reformulation of k_sinr.cu):
//     A_u(f)     = H~_{iij}(f) H~_{iij}(f)^H                  (serving Gram -> precoder)
//     X_{u,k}(f) = H~_{kij}(f) H~_{kk0}(f)^H,   k != i        (interference through the anchor (k,0))
// written in the pair-Gram layout PG[g][f][user][J][m*m] (slot 0 serving, then k != i ascending;
// entry (a, b) at a + m b) that the eig + MMSE kernels consume.
//
// Per link the rebuild is a GEMM over the subcarriers:  H~^T[f, x] = sum_q E^T[f, q] G^T[q, x],
// E(q, f) = sum_r C(r, q) conj(c_r(f)), x = r + m c (the core's storage order). It runs as a real
// GEMM on tcgen05.mma.kind::tf32 with 3xTF32 splitting (hi*hi + hi*lo + lo*hi ~ fp32 accuracy):
//     A  = [Er | Ei]                       (128 subcarriers x 2p, K-major, from k_esplit)
//     B  = [Gi | Gr ; Gr | -Gi]            (2 XC rows x 2p, K-major, from k_bsplit: rows [0, XC) give Hi of the
//                                           x chunk, rows [XC, 2 XC) its Hr)
//     [Hi | Hr] = A * B^T                  (one MMA of N = 2 XC per k-step: the A slice is fetched once for both)
// (measured against two N = XC MMAs per k-step on B = [Gi | Gr | -Gi]: the small-N MMAs are paced by their
// operand fetch, not by the math). Both operands are staged by TMA bulk
// copies (cp.async.bulk + mbarrier complete_tx) from pre-split global buffers; the accumulators (Hr,
// Hi per link slot, two stages) live in TMEM with lane = subcarrier.
//
// CTA = (user, group); it walks the subcarrier tiles and, per tile, its J "jobs": job 0 = the
// serving link, job k = (interfering link (k,i,j), anchor link (k,k,0)). Warp roles:
//   warp 8  (whole warp, elect.sync issue): MMA issuer  per chunk 3 passes x p/4 k-steps x slots; loads the job's
//                         E tiles (A) itself
//   warp 9  (one thread): TMA producer   G chunk (B) per chunk, 2 B stages
//   warps 0-7           : Gram epilogue  two threads per subcarrier (TMEM lane quarter = warp % 4);
//                         tcgen05.ld -> binary64 -> DFMA accumulation of the entries of its rows
// Binary64 accumulation of the exact products of the fp32 H~ values keeps the Gram route free of
// the kappa^2 loss an fp32 Gram would add.
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"
#include "tc_sm100.cuh"

namespace gwtk {

namespace {

constexpr int kFT = 128;                          // subcarriers per tile = MMA M = TMEM lanes
constexpr int kEpiWarps = 8;                      // two Gram threads per subcarrier
constexpr int kRgThreads = (kEpiWarps + 2) * 32;  // + MMA warp + TMA warp

struct RgCfg {
    int m, n, p, mn, XC, nch, ks, tcols;
    uint32_t TA, TB;  // bytes of one A operand (128 x 2p fp32) / one B operand (2 XC x 2p fp32)
    uint32_t sbo_a, sbo_b;
    size_t smem;
};

RgCfg rg_cfg(const Topo& t, int XC) {
    RgCfg c{};
    c.m = t.m;
    c.n = t.n;
    c.p = t.p;
    c.mn = t.m * t.n;
    c.XC = XC;
    c.nch = c.mn / XC;
    c.ks = 2 * t.p / 8;
    c.TA = (uint32_t)kFT * 2 * t.p * 4;
    c.TB = (uint32_t)2 * XC * 2 * t.p * 4;
    c.sbo_a = (uint32_t)(2 * t.p / 4) * 128;
    c.sbo_b = (uint32_t)(2 * t.p / 4) * 128;
    c.smem = (size_t)4 * c.TA + (size_t)8 * c.TB;
    c.tcols = 8 * XC <= 32 ? 32 : (8 * XC <= 64 ? 64 : (8 * XC <= 128 ? 128 : 256));
    return c;
}

// canonical K-major no-swizzle offset (bytes) of element (row, k) in a tile with `sbo` bytes per 8 rows
__device__ __forceinline__ uint32_t kmaj(int row, int k, uint32_t sbo) {
    return (uint32_t)((row >> 3) * sbo + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4);
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// B operands: Bready[g][l][chunk][hi|lo] = rows n: [Gi | Gr], rows XC + n: [Gr | -Gi] (x = chunk*XC + n), K-major canonical.
__global__ void __launch_bounds__(256) k_bsplit(Topo t, RgCfg c, const float2* __restrict__ G,
                                               unsigned char* __restrict__ Bready) {
    const int ch = blockIdx.x, l = blockIdx.y;
    const int64_t g = blockIdx.z, gl = g * t.links() + l;
    const int p = c.p, XC = c.XC, x0 = ch * XC;
    const float2* Gl = G + gl * (int64_t)c.mn * p;
    unsigned char* hi = Bready + ((size_t)gl * c.nch + ch) * 2 * c.TB;
    unsigned char* lo = hi + c.TB;
    for (int e = threadIdx.x; e < XC * p; e += blockDim.x) {
        const int n = e % XC, q = e / XC;
        const float2 v = Gl[(int64_t)q * c.mn + x0 + n];
        const float vals[4] = {v.y, v.x, v.x, -v.y};
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            float h, r;
            tc::split_tf32_rn(vals[b], h, r);
            const uint32_t o = kmaj((b >> 1) * XC + n, (b & 1) * p + q, c.sbo_b);
            *reinterpret_cast<float*>(hi + o) = h;
            *reinterpret_cast<float*>(lo + o) = r;
        }
    }
}

// ---------------------------------------------------------------------------------------------
// A operands: Eready[g][l][tile][hi|lo] = [Er | Ei] rows = subcarriers of the tile, K-major canonical.
// One thread per subcarrier: conj phasors (binary64 argument reduction) and E = C^T c* in fp32.
template <int PQ>
__global__ void __launch_bounds__(2 * kFT) k_esplit(Topo t, RgCfg c, int Fc, int64_t f0, int ntiles,
                                                    const float2* __restrict__ Cd, const double* __restrict__ tau,
                                                    const double* __restrict__ freqs, unsigned char* __restrict__ Eready) {
    extern __shared__ __align__(16) unsigned char es_smem[];
    float2* ph = reinterpret_cast<float2*>(es_smem);  // [P][kFT]
    float2* sC = ph + (size_t)t.P * kFT;               // [P][PQ] (C_l transposed: q contiguous per tap)
    const int ti = blockIdx.x, l = blockIdx.y;
    const int64_t g = blockIdx.z, gl = g * t.links() + l;
    const int P = t.P, tid = threadIdx.x;
    const float2* Cl = Cd + gl * (int64_t)P * PQ;
    const double* tl = tau + gl * P;
    for (int e = tid; e < P * PQ; e += 2 * kFT) {
        const int q = e / P, r = e % P;  // coalesced read of the column-major P x p factor
        sC[r * PQ + q] = Cl[e];
    }
    for (int e = tid; e < P * kFT; e += 2 * kFT) {
        const int r = e / kFT, f = ti * kFT + e % kFT;
        ph[e] = f < Fc ? conj_coeff<float>(freqs[f0 + f], tl[r]) : make_float2(0.f, 0.f);
    }
    __syncthreads();
    // thread (subcarrier pair fp = (fl, fl + 64), q quarter qq): E(q, f) for q in [qq*QQ, qq*QQ + QQ);
    // per tap: 2 phasor loads and QQ/2 16-byte broadcast loads of C feed 8 QQ FFMA
    constexpr int QQ = PQ / 4;
    const int fl = tid % (kFT / 2), qq = tid / (kFT / 2);
    float2 e0[QQ], e1[QQ];
#pragma unroll
    for (int q = 0; q < QQ; ++q) e0[q] = e1[q] = make_float2(0.f, 0.f);
#pragma unroll 4
    for (int r = 0; r < P; ++r) {
        const float2 v0 = ph[r * kFT + fl], v1 = ph[r * kFT + fl + kFT / 2];
        const float2* cr = sC + r * PQ + qq * QQ;
        if constexpr (QQ % 2 == 0) {
#pragma unroll
            for (int q = 0; q < QQ; q += 2) {
                const float4 c2 = *reinterpret_cast<const float4*>(cr + q);
                const float2 ca = make_float2(c2.x, c2.y), cb = make_float2(c2.z, c2.w);
                cfma(e0[q], ca, v0);
                cfma(e1[q], ca, v1);
                cfma(e0[q + 1], cb, v0);
                cfma(e1[q + 1], cb, v1);
            }
        } else {
#pragma unroll
            for (int q = 0; q < QQ; ++q) {
                const float2 ca = cr[q];
                cfma(e0[q], ca, v0);
                cfma(e1[q], ca, v1);
            }
        }
    }
    unsigned char* hi = Eready + ((size_t)gl * ntiles + ti) * 2 * c.TA;
    unsigned char* lo = hi + c.TA;
    // K columns: [0, p) Er, [p, 2p) Ei
#pragma unroll
    for (int q = 0; q < QQ; ++q) {
        const int k = qq * QQ + q;
        const float v[4] = {e0[q].x, e0[q].y, e1[q].x, e1[q].y};
        const int rows[4] = {fl, fl, fl + kFT / 2, fl + kFT / 2};
        const int ks[4] = {k, PQ + k, k, PQ + k};
#pragma unroll
        for (int z = 0; z < 4; ++z) {
            float h, rr;
            tc::split_tf32_rn(v[z], h, rr);
            const uint32_t o = kmaj(rows[z], ks[z], c.sbo_a);
            *reinterpret_cast<float*>(hi + o) = h;
            *reinterpret_cast<float*>(lo + o) = rr;
        }
    }
}

// ---------------------------------------------------------------------------------------------
// Gram epilogue helpers (templated on the thread's half H so every accumulator index is static).
namespace {

// serving-Gram rows of half H: MP = 8 -> {0,7,2,5} / {1,6,3,4}; MP = 4 -> {0,3} / {1,2} (balanced
// lower-triangle entry counts: 18 / 18 and 5 / 5)
template <int MP, int H> __host__ __device__ constexpr int srow_n() { return MP / 2; }
template <int MP, int H> __host__ __device__ constexpr int srow(int idx) {
    return MP == 8 ? (H == 0 ? (idx == 0 ? 0 : idx == 1 ? 7 : idx == 2 ? 2 : 5)
                             : (idx == 0 ? 1 : idx == 1 ? 6 : idx == 2 ? 3 : 4))
                   : (H == 0 ? (idx == 0 ? 0 : 3) : (idx == 0 ? 1 : 2));
}
template <int MP, int H> __host__ __device__ constexpr int srow_off(int idx) {
    int o = 0;
    for (int z = 0; z < idx; ++z) o += srow<MP, H>(z) + 1;
    return o;
}
template <int MP> constexpr int kServAcc = MP == 8 ? 18 : 5;

#ifdef GWT_F2D_INT
// fp32 -> fp64 by exponent rebias on the integer pipe (F2F.F64.F32 issues at 16/clk/SM on the XU);
// exact for normal numbers, +-0 kept, fp32 subnormals (< 1.2e-38) flush to +-0, Inf/NaN kept non-finite
__device__ __forceinline__ double i2d(uint32_t b) {
    const uint32_t a = b & 0x7fffffffu;
    uint32_t hi = ((a >> 3) + 0x38000000u) | (b & 0x80000000u);
    hi = a < 0x00800000u ? (b & 0x80000000u) : hi;
    hi = a >= 0x7f800000u ? (hi | 0x7ff00000u) : hi;
    return __hiloint2double((int)hi, (int)(b << 29));
}
__device__ __forceinline__ double2 f2d(uint32_t re, uint32_t im) { return make_double2(i2d(re), i2d(im)); }
#else
__device__ __forceinline__ double2 f2d(uint32_t re, uint32_t im) {
    return make_double2((double)__uint_as_float(re), (double)__uint_as_float(im));
}
#endif

template <int MP>
__device__ __forceinline__ void tmem_ldmp(uint32_t taddr, uint32_t (&r)[MP]);
template <> __device__ __forceinline__ void tmem_ldmp<8>(uint32_t taddr, uint32_t (&r)[8]) { tc::tmem_ld8_nw(taddr, r); }
template <> __device__ __forceinline__ void tmem_ldmp<4>(uint32_t taddr, uint32_t (&r)[4]) { tc::tmem_ld4_nw(taddr, r); }

// TMEM columns of stage base col0: slot 0 Hi [0, XC), Hr [XC, 2XC); slot 1 Hi [2XC, 3XC), Hr [3XC, 4XC);
// within a slot, column x = r + MP c_local. Loads of column cl+1 are issued before the DFMAs of column cl
// (one tcgen05.wait::ld per column, after the arithmetic), so the TMEM latency hides behind the math.

// serving Gram: acc(row, r') += H(row, c) conj(H(r', c)), r' <= row, rows of half H
template <int MP, int H>
__device__ __forceinline__ void serving_chunk(uint32_t col0, int XC, double2 (&acc)[kServAcc<MP>]) {
    // single-buffered: 18 accumulators + the converted column leave no room for a second raw buffer
    for (int cl = 0; cl < XC / MP; ++cl) {
        uint32_t hr[MP], hi[MP];
        tmem_ldmp<MP>(col0 + XC + MP * cl, hr);
        tmem_ldmp<MP>(col0 + MP * cl, hi);
        tc::tmem_wait_ld();
        double2 v[MP];
#pragma unroll
        for (int r = 0; r < MP; ++r) v[r] = f2d(hr[r], hi[r]);
#pragma unroll
        for (int idx = 0; idx < srow_n<MP, H>(); ++idx) {
            const int row = srow<MP, H>(idx);
#pragma unroll
            for (int r2 = 0; r2 < MP; ++r2)
                if (r2 <= row) cfmac(acc[srow_off<MP, H>(idx) + r2], v[row], v[r2]);
        }
    }
}

// pair Gram, quarter (H, Q): acc(z, w) += Hx(H*RH + z, c) conj(Ha(Q*RH + w, c)), z, w < RH = MP / 2
template <int MP, int H, int Q>
__device__ __forceinline__ void pair_load(uint32_t col0, int XC, int cl, uint32_t (&xr)[4], uint32_t (&xi)[4],
                                          uint32_t (&ar)[4], uint32_t (&ai)[4]) {
    constexpr int RH = MP / 2;
    const uint32_t xo = MP * cl + (RH == 4 ? H * RH : 0), ao = MP * cl + (RH == 4 ? Q * RH : 0);
    tc::tmem_ld4_nw(col0 + XC + xo, xr);      // Hr of slot 0 (receive link)
    tc::tmem_ld4_nw(col0 + xo, xi);           // Hi of slot 0
    tc::tmem_ld4_nw(col0 + 3 * XC + ao, ar);  // Hr of slot 1 (anchor)
    tc::tmem_ld4_nw(col0 + 2 * XC + ao, ai);  // Hi of slot 1
}
template <int MP, int H, int Q>
__device__ __forceinline__ void pair_chunk(uint32_t col0, int XC, double2 (&acc)[MP * MP / 4]) {
    constexpr int RH = MP / 2;
    constexpr int xoff = RH == 4 ? 0 : H * RH, aoff = RH == 4 ? 0 : Q * RH;
    for (int cl = 0; cl < XC / MP; ++cl) {
        uint32_t xr[4], xi[4], ar[4], ai[4];
        pair_load<MP, H, Q>(col0, XC, cl, xr, xi, ar, ai);
        tc::tmem_wait_ld();
        double2 x[RH];
#pragma unroll
        for (int z = 0; z < RH; ++z) x[z] = f2d(xr[xoff + z], xi[xoff + z]);
#pragma unroll
        for (int w = 0; w < RH; ++w) {
            const double2 a = f2d(ar[aoff + w], ai[aoff + w]);
#pragma unroll
            for (int z = 0; z < RH; ++z) cfmac(acc[z * RH + w], x[z], a);
        }
    }
}

// pair Gram, all columns of the thread's rows: acc(z, r') += Hx(H*RH + z, c) conj(Ha(r', c))
template <int MP, int H>
__device__ __forceinline__ void pair_chunk_full(uint32_t col0, int XC, double2 (&acc)[MP * MP / 2]) {
    constexpr int RH = MP / 2;
    constexpr int xoff = RH == 4 ? 0 : H * RH;
    for (int cl = 0; cl < XC / MP; ++cl) {
        uint32_t xr[4], xi[4], ar[MP], ai[MP];
        const uint32_t xo = MP * cl + (RH == 4 ? H * RH : 0);
        tc::tmem_ld4_nw(col0 + XC + xo, xr);
        tc::tmem_ld4_nw(col0 + xo, xi);
        tmem_ldmp<MP>(col0 + 3 * XC + MP * cl, ar);
        tmem_ldmp<MP>(col0 + 2 * XC + MP * cl, ai);
        tc::tmem_wait_ld();
        double2 x[RH];
#pragma unroll
        for (int z = 0; z < RH; ++z) x[z] = f2d(xr[xoff + z], xi[xoff + z]);
#pragma unroll
        for (int w = 0; w < MP; ++w) {
            const double2 a = f2d(ar[w], ai[w]);
#pragma unroll
            for (int z = 0; z < RH; ++z) cfmac(acc[z * MP + w], x[z], a);
        }
    }
}

// 32-byte store (two adjacent double2; sm_100 256-bit global stores): the thread's rows are contiguous per column,
// and the PG rows of the warp's 32 subcarriers are 64 KB apart, so every store instruction is 32 separate requests
// (16-byte stores: 8 % of the kernel's stall samples on the LSU queue; C4 R+Gram 41.2 -> 38.9 ms per 64 groups)
__device__ __forceinline__ void st_pair32(double2* p, double2 a, double2 b) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y) : "memory");
}
template <int MP, int H>
__device__ __forceinline__ void write_serving(double2* __restrict__ out, int m, const double2 (&acc)[kServAcc<MP>]) {
#pragma unroll
    for (int idx = 0; idx < srow_n<MP, H>(); ++idx) {
        const int row = srow<MP, H>(idx);
        // lower-triangle entries (row, r2 < row): strided by a column, one 16-byte store each
#pragma unroll
        for (int r2 = 0; r2 < MP; ++r2)
            if (r2 < row) out[row + m * r2] = acc[srow_off<MP, H>(idx) + r2];
        // their conjugates and the diagonal fill column `row`, rows 0..row: contiguous, 32-byte stores
        double2 cj[MP];
#pragma unroll
        for (int r2 = 0; r2 < MP; ++r2)
            if (r2 <= row) cj[r2] = make_double2(acc[srow_off<MP, H>(idx) + r2].x, r2 == row ? 0.0 : -acc[srow_off<MP, H>(idx) + r2].y);
#pragma unroll
        for (int r2 = 0; r2 < MP; r2 += 2) {
            if (r2 + 1 <= row && m == MP) st_pair32(out + r2 + m * row, cj[r2], cj[r2 + 1]);
            else {
                if (r2 <= row) out[r2 + m * row] = cj[r2];
                if (r2 + 1 <= row) out[r2 + 1 + m * row] = cj[r2 + 1];
            }
        }
    }
}
template <int MP, int H>
__device__ __forceinline__ void write_pair_full(double2* __restrict__ out, int m, const double2 (&acc)[MP * MP / 2]) {
    constexpr int RH = MP / 2;
    if constexpr (RH % 2 == 0) {
        if (m == MP) {
#pragma unroll
            for (int w = 0; w < MP; ++w)
#pragma unroll
                for (int z = 0; z < RH; z += 2) st_pair32(out + (H * RH + z) + m * w, acc[z * MP + w], acc[(z + 1) * MP + w]);
            return;
        }
    }
#pragma unroll
    for (int z = 0; z < RH; ++z)
#pragma unroll
        for (int w = 0; w < MP; ++w) out[(H * RH + z) + m * w] = acc[z * MP + w];
}
template <int MP, int H, int Q>
__device__ __forceinline__ void write_pair(double2* __restrict__ out, int m, const double2 (&acc)[MP * MP / 4]) {
    constexpr int RH = MP / 2;
#pragma unroll
    for (int z = 0; z < RH; ++z)
#pragma unroll
        for (int w = 0; w < RH; ++w) out[(H * RH + z) + m * (Q * RH + w)] = acc[z * RH + w];
}

struct EpiCtx {
    uint64_t* t_full;
    uint64_t* t_empty;
    uint32_t tcol;  // tmem base + lane quarter
    int XC, nch;
};

// one whole job of the epilogue (all chunks + the PG write); KIND 0 = serving, 1 / 2 = pair quarter Q = 0 / 1,
// 3 = whole pair rows of the thread's half
template <int MP, int H, int KIND>
__device__ __forceinline__ void epi_job(const EpiCtx& e, uint32_t& cnt, bool valid, double2* __restrict__ out, int m) {
    constexpr int NA = KIND == 0 ? kServAcc<MP> : (KIND == 3 ? MP * MP / 2 : MP * MP / 4);
    double2 acc[NA];
#pragma unroll
    for (int z = 0; z < NA; ++z) acc[z] = make_double2(0.0, 0.0);
    for (int ch = 0; ch < e.nch; ++ch, ++cnt) {
        const int st = cnt & 1;
        const uint32_t use = cnt >> 1;
        tc::mbar_wait(&e.t_full[st], use & 1);
        tc::fence_after_sync();
        const uint32_t col0 = e.tcol + (uint32_t)(st * 4 * e.XC);
#ifdef GWT_RG_PROBE_NOEPI
        if (ch == 0)
#endif
        if constexpr (KIND == 0) serving_chunk<MP, H>(col0, e.XC, acc);
        else if constexpr (KIND == 3) pair_chunk_full<MP, H>(col0, e.XC, acc);
        else pair_chunk<MP, H, KIND - 1>(col0, e.XC, acc);
        tc::fence_before_sync();
        tc::mbar_arrive(&e.t_empty[st]);
    }
    if (valid) {
        if constexpr (KIND == 0) write_serving<MP, H>(out, m, acc);
        else if constexpr (KIND == 3) write_pair_full<MP, H>(out, m, acc);
        else write_pair<MP, H, KIND - 1>(out, m, acc);
    }
}

}  // namespace

// Control state of the producer threads: TMA bulk loads (TMA warp) and tcgen05.mma issue (MMA warp) over
// a flat sequence of chunks (tile, job, chunk). Jobs per tile: 0 = serving link; then for each cell k != i
// two jobs (the two quarters Q of the pair Gram's columns, same links: receive (k,i,j) in slot 0, anchor
// (k,k,0) in slot 1). Splitting the pair Gram into column halves keeps 16 binary64 accumulators per
// thread, which leaves registers for double-buffered TMEM loads at 10 warps (the tensor cores recompute
// the pair's H~ once more; they are not the binding pipe).
struct RgCtrl {
    const RgCfg* c;
    unsigned char* sA;
    unsigned char* sB;
    const unsigned char* Bready;
    const unsigned char* Eready;
    uint64_t *a_full, *a_empty, *b_full, *b_empty, *t_full, *t_empty;
    uint32_t tb;
    int64_t g;
    int links, ntiles, njobs, nch, total;
    int i, j, J, K, split;  // split: 2 jobs (column quarters) per pair, else 1
    __device__ __forceinline__ int job_link(int jb, int slot) const {
        if (jb == 0) return (i * J + i) * K + j;
        int k = (jb - 1) / split;
        if (k >= i) ++k;
        return slot == 0 ? (k * J + i) * K + j : (k * J + k) * K;
    }
    __device__ __forceinline__ void tma_b(int k) const {  // B operands of flat chunk k into stage k & 1
        const int st = k & 1, use = k >> 1;
        const int job = k / nch, ch = k % nch, jb = job % njobs;
        const int ns = jb == 0 ? 1 : 2;
        if (use > 0) tc::mbar_wait(&b_empty[st], (use - 1) & 1);
        tc::mbar_arrive_expect_tx(&b_full[st], (uint32_t)ns * 2 * c->TB);
        for (int sl = 0; sl < ns; ++sl) {
            const int64_t gl = g * links + job_link(jb, sl);
            tc::bulk_g2s(sB + ((size_t)st * 2 + sl) * 2 * c->TB, Bready + ((size_t)gl * nch + ch) * 2 * c->TB,
                         2 * c->TB, &b_full[st]);
        }
    }
    __device__ __forceinline__ void tma_a(int job, int sl) const {
        const int jb = job % njobs, ti = job / njobs;
        const int64_t gl = g * links + job_link(jb, sl);
        tc::bulk_g2s(sA + (size_t)sl * 2 * c->TA, Eready + ((size_t)gl * ntiles + ti) * 2 * c->TA, 2 * c->TA, a_full);
    }
#ifdef GWT_RG_TIMERS
#define RG_T0 long long t0_ = clock64()
#define RG_TA(i) do { long long t1_ = clock64(); tm[i] += t1_ - t0_; t0_ = t1_; } while (0)
    mutable long long tm[4] = {0, 0, 0, 0};
#else
#define RG_T0
#define RG_TA(i)
#endif
    // The MMA warp walks the chunk sequence as a whole warp (the waits are warp-wide) and issues TMA / tcgen05.mma /
    // tcgen05.commit under elect.sync: in a `lane == 0` region the compiler wraps every uniform-datapath instruction
    // (UTCHMMA, UTCBAR) in an ELECT / BRA.U.ANY loop — 126 cycles per MMA on the lone issuing thread
    // (tools/micro/mma_fetch.cu: 242 vs 48 cycles per N = 64 MMA) — while under elect.sync with the k-steps
    // unrolled the MMAs issue back to back and run at their shared-memory operand fetch rate.
    template <int KS>
    __device__ __forceinline__ void issue(uint32_t d, uint64_t dAh, uint64_t dAl, uint64_t dBh, uint64_t dBl,
                                          uint32_t idesc) const {
#ifdef GWT_RG_PROBE_1PASS
        constexpr int NP = 1;
#else
        constexpr int NP = 3;
#endif
#pragma unroll
        for (int pass = 0; pass < NP; ++pass) {
            const uint64_t da = pass == 2 ? dAl : dAh;
            const uint64_t db = pass == 1 ? dBl : dBh;
#pragma unroll
            for (int kk = 0; kk < KS; ++kk)
                tc::mma_tf32(d, da + 16 * kk, db + 16 * kk, idesc, (pass > 0 || kk > 0) ? 1u : 0u);
        }
    }
    __device__ __forceinline__ void mma(int k) const {  // all MMAs of flat chunk k (loads the job's A first)
        RG_T0;
        const int st = k & 1, use = k >> 1;
        const int job = k / nch, ch = k % nch, jb = job % njobs;
        const int ns = jb == 0 ? 1 : 2;
        const int XC = c->XC;
        if (ch == 0) {
            // A of this job: job 0 uses slot 0 and prefetches the first pair's anchor into slot 1; the first
            // pair's quarter 0 then loads slot 0 alone; quarter 1 reuses both slots; later pairs load both
            if (job > 0) tc::mbar_wait(a_empty, (job - 1) & 1);
            if (tc::elect_one()) {
                const int pk = (jb - 1) / split, q = (jb - 1) % split;
                const int nload = jb == 0 ? (njobs > 1 ? 2 : 1) : (q == 1 ? 0 : (pk == 0 ? 1 : 2));
                tc::mbar_arrive_expect_tx(a_full, (uint32_t)nload * 2 * c->TA);
                if (jb == 0) {
                    tma_a(job, 0);
                    if (njobs > 1) tma_a(job + 1, 1);
                } else if (q == 0) {
                    tma_a(job, 0);
                    if (pk > 0) tma_a(job, 1);
                }
            }
            __syncwarp();
            tc::mbar_wait(a_full, job & 1);
        }
        RG_TA(0);
        tc::mbar_wait(&b_full[st], use & 1);
        RG_TA(1);
        if (use > 0) tc::mbar_wait(&t_empty[st], (use - 1) & 1);
        RG_TA(2);
        tc::fence_after_sync();
        const uint32_t idesc = tc::idesc_tf32(kFT, 2 * XC);
        if (tc::elect_one()) {
            for (int sl = 0; sl < ns; ++sl) {
                const uint32_t dI = tb + (uint32_t)(st * 4 * XC + sl * 2 * XC);  // columns [Hi | Hr] of this slot
                const uint32_t ab = tc::smem_u32(sA + (size_t)sl * 2 * c->TA);
                const uint32_t bb = tc::smem_u32(sB + ((size_t)st * 2 + sl) * 2 * c->TB);
                // descriptor start-address field = addr >> 4 (14 bits, smem < 256 KB): k-step kk adds 16
                const uint64_t dAh = tc::smem_desc(ab, 128, c->sbo_a), dAl = tc::smem_desc(ab + c->TA, 128, c->sbo_a);
                const uint64_t dBh = tc::smem_desc(bb, 128, c->sbo_b), dBl = tc::smem_desc(bb + c->TB, 128, c->sbo_b);
                switch (c->ks) {
                    case 2: issue<2>(dI, dAh, dAl, dBh, dBl, idesc); break;
                    case 3: issue<3>(dI, dAh, dAl, dBh, dBl, idesc); break;
                    case 4: issue<4>(dI, dAh, dAl, dBh, dBl, idesc); break;
                    case 6: issue<6>(dI, dAh, dAl, dBh, dBl, idesc); break;
                    default: issue<8>(dI, dAh, dAl, dBh, dBl, idesc); break;
                }
            }
            tc::commit(&b_empty[st]);
            tc::commit(&t_full[st]);
            if (ch == nch - 1) tc::commit(a_empty);
        }
        __syncwarp();
        RG_TA(3);
    }
};

template <int MP, bool SPLIT>
__global__ void __launch_bounds__(kRgThreads, 1) k_rgram(Topo t, RgCfg c, int Fc, int ntiles, int64_t pf0, int64_t Fs,
                                                         const unsigned char* __restrict__ Bready,
                                                         const unsigned char* __restrict__ Eready,
                                                         double2* __restrict__ PG) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint64_t a_full, a_empty, b_full[2], b_empty[2], t_full[2], t_empty[2];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int u = blockIdx.x, users = t.users();
    const int64_t g = blockIdx.y;
    const int J = t.J, K = t.K;
    const int XC = c.XC, nch = c.nch;
    if (warp == 0) tc::tmem_alloc(&tmem_base, c.tcols);
    if (tid == 32) {
        tc::mbar_init(&a_full, 1);
        tc::mbar_init(&a_empty, 1);
        for (int s = 0; s < 2; ++s) {
            tc::mbar_init(&b_full[s], 1);
            tc::mbar_init(&b_empty[s], 1);
            tc::mbar_init(&t_full[s], 1);
            tc::mbar_init(&t_empty[s], kEpiWarps * 32);
        }
        tc::fence_barrier_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tb = tmem_base;
    constexpr int SP = SPLIT ? 2 : 1;
    const int njobs = 1 + SP * (J - 1);
    const int total = ntiles * njobs * nch;
    const RgCtrl ctl{&c, smem, smem + 4 * c.TA, Bready, Eready, &a_full, &a_empty, b_full, b_empty, t_full, t_empty,
                     tb, g, t.links(), ntiles, njobs, nch, total, u / K, u % K, J, K, SP};
    if (warp == kEpiWarps) {  // MMA warp
        for (int k = 0; k < total; ++k) ctl.mma(k);
#ifdef GWT_RG_TIMERS
        if (lane == 0 && blockIdx.x == 3 && blockIdx.y == 5)
            printf("mma thread: chunks %d  a_full %lld  b_full %lld  t_empty %lld  issue %lld (cycles per chunk)\n", total,
                   ctl.tm[0] / total, ctl.tm[1] / total, ctl.tm[2] / total, ctl.tm[3] / total);
#endif
        __syncwarp();
    } else if (warp == kEpiWarps + 1) {  // TMA warp
        if (lane == 0)
            for (int k = 0; k < total; ++k) ctl.tma_b(k);
        __syncwarp();
    } else {
        // ---------------- Gram epilogue: thread (subcarrier fl of the tile, half h)
        const int q4 = warp & 3, h = warp >> 2;
        const int fl = 32 * q4 + lane;
        const uint32_t lanebase = (uint32_t)(32 * q4) << 16;
        const int m = c.m, S = J;
        uint32_t cnt = 0;
        const EpiCtx ec{t_full, t_empty, tb + lanebase, XC, nch};
        for (int ti = 0; ti < ntiles; ++ti) {
            const int f = ti * kFT + fl;
            const bool valid = f < Fc;
            const int64_t row = ((int64_t)g * Fs + pf0 + f) * users + u;
            for (int jb = 0; jb < njobs; ++jb) {
                const int slot = jb == 0 ? 0 : 1 + (jb - 1) / SP, q = jb == 0 ? 0 : (jb - 1) % SP;
                double2* out = PG + (row * S + slot) * (int64_t)m * m;
                if (jb == 0) {
                    if (h == 0) epi_job<MP, 0, 0>(ec, cnt, valid, out, m);
                    else epi_job<MP, 1, 0>(ec, cnt, valid, out, m);
                } else if (!SPLIT) {
                    if (h == 0) epi_job<MP, 0, 3>(ec, cnt, valid, out, m);
                    else epi_job<MP, 1, 3>(ec, cnt, valid, out, m);
                } else if (q == 0) {
                    if (h == 0) epi_job<MP, 0, 1>(ec, cnt, valid, out, m);
                    else epi_job<MP, 1, 1>(ec, cnt, valid, out, m);
                } else {
                    if (h == 0) epi_job<MP, 0, 2>(ec, cnt, valid, out, m);
                    else epi_job<MP, 1, 2>(ec, cnt, valid, out, m);
                }
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (warp == 0) tc::tmem_dealloc(tb, c.tcols);
}

// ---------------------------------------------------------------------------------------------
// host side

namespace {
bool rg_pick(const Topo& t, RgCfg& c) {
    if (!(t.m == 4 || t.m == 8) || t.p % 4 != 0 || t.p > 32 || (t.p != 8 && t.p != 12 && t.p != 16 && t.p != 24 && t.p != 32))
        return false;
    for (int XC : {32, 16}) {
        if ((t.m * t.n) % XC != 0 || XC % t.m != 0) continue;
        c = rg_cfg(t, XC);
        if (c.smem <= 220 * 1024) return true;
    }
    return false;
}
}  // namespace

bool rgram_fits(const Topo& t) {
    RgCfg c;
    return t.L <= t.m && rg_pick(t, c);
}

size_t rgram_bready_bytes(const Topo& t, int64_t ngroups) {
    RgCfg c;
    if (!rg_pick(t, c)) return 0;
    return (size_t)ngroups * t.links() * c.nch * 2 * c.TB;
}

size_t rgram_eready_bytes(const Topo& t, int64_t ngroups, int Fc) {
    RgCfg c;
    if (!rg_pick(t, c)) return 0;
    const int ntiles = (Fc + kFT - 1) / kFT;
    return (size_t)ngroups * t.links() * ntiles * 2 * c.TA;
}

cudaError_t launch_rgram_prep(const Topo& t, int64_t ngroups, const void* G, void* Bready, cudaStream_t st) {
    RgCfg c;
    if (!rg_pick(t, c)) return cudaErrorNotSupported;
    dim3 grid(c.nch, t.links(), (unsigned)ngroups);
    k_bsplit<<<grid, 256, 0, st>>>(t, c, (const float2*)G, (unsigned char*)Bready);
    return cudaGetLastError();
}

cudaError_t launch_rgram(const Topo& t, int64_t ngroups, int Fc, int64_t f0, int64_t pf0, int64_t Fs, const void* Cd,
                         const double* tau, const double* freqs, const void* Bready, void* Eready, double2* PG,
                         cudaStream_t st) {
    RgCfg c;
    if (!rg_pick(t, c)) return cudaErrorNotSupported;
    const int ntiles = (Fc + kFT - 1) / kFT;
    dim3 ge(ntiles, t.links(), (unsigned)ngroups);
    const size_t es_sm = sizeof(float2) * ((size_t)t.P * kFT + (size_t)t.P * t.p);
    cudaError_t e0;
    switch (t.p) {
#define GWT_ES(PQ) \
    case PQ:                                                                                                         \
        if ((e0 = cudaFuncSetAttribute(k_esplit<PQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)es_sm)) != cudaSuccess) \
            return e0;                                                                                               \
        k_esplit<PQ><<<ge, 2 * kFT, es_sm, st>>>(t, c, Fc, f0, ntiles, (const float2*)Cd, tau, freqs, (unsigned char*)Eready); \
        break;
        GWT_ES(8) GWT_ES(12) GWT_ES(16) GWT_ES(24) GWT_ES(32)
#undef GWT_ES
        default: return cudaErrorNotSupported;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    dim3 grid(t.users(), (unsigned)ngroups);
    static const bool split = [] {
        const char* v = env_once("GWT_RGRAM_SPLIT");
        return v && std::atoi(v) != 0;
    }();
#define GWT_RG(MPV, SPV)                                                                                            \
    do {                                                                                                            \
        e = cudaFuncSetAttribute(k_rgram<MPV, SPV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);      \
        if (e != cudaSuccess) return e;                                                                             \
        k_rgram<MPV, SPV><<<grid, kRgThreads, c.smem, st>>>(t, c, Fc, ntiles, pf0, Fs, (const unsigned char*)Bready, \
                                                            (const unsigned char*)Eready, PG);                       \
    } while (0)
    if (t.m == 8) {
        if (split) GWT_RG(8, true);
        else GWT_RG(8, false);
    } else {
        if (split) GWT_RG(4, true);
        else GWT_RG(4, false);
    }
#undef GWT_RG
    return cudaGetLastError();
}

}  // namespace gwtk
