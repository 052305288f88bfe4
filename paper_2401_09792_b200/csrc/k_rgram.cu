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
//     B  = [Gi | Gr | -Gi]                 (x chunk of XC rows x 3p, K-major, from k_bsplit)
//     Hi = A * B[:, 0:2p]^T,   Hr = A * B[:, p:3p]^T        (two MMAs sharing A, k-step pointer offsets)
// so the real-form doubling costs no extra operand storage. Both operands are staged by TMA bulk
// copies (cp.async.bulk + mbarrier complete_tx) from pre-split global buffers; the accumulators (Hr,
// Hi per link slot, two stages) live in TMEM with lane = subcarrier.
//
// CTA = (user, group); it walks the subcarrier tiles and, per tile, its J "jobs": job 0 = the
// serving link, job k = (interfering link (k,i,j), anchor link (k,k,0)). Warp roles:
//   warp 8  (one thread): TMA producer   E tile (A) per job, G chunk (B) per chunk, 2 B stages
//   warp 9  (one thread): MMA issuer     per chunk 3 passes x p/4 k-steps x {Hi, Hr} x slots
//   warps 0-7           : Gram epilogue  two threads per subcarrier (TMEM lane quarter = warp % 4);
//                         tcgen05.ld -> binary64 -> DFMA accumulation of the entries of its rows
// Binary64 accumulation of the exact products of the fp32 H~ values keeps the Gram route free of
// the kappa^2 loss an fp32 Gram would add.
#include "kernels.cuh"
#include "tc_sm100.cuh"

namespace gwtk {

namespace {

constexpr int kFT = 128;                          // subcarriers per tile = MMA M = TMEM lanes
constexpr int kEpiWarps = 8;                      // two Gram threads per subcarrier
constexpr int kRgThreads = (kEpiWarps + 2) * 32;  // + TMA warp + MMA warp

struct RgCfg {
    int m, n, p, mn, XC, nch, ks, tcols;
    uint32_t TA, TB;  // bytes of one A operand (128 x 2p fp32) / one B operand (XC x 3p fp32)
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
    c.TB = (uint32_t)XC * 3 * t.p * 4;
    c.sbo_a = (uint32_t)(2 * t.p / 4) * 128;
    c.sbo_b = (uint32_t)(3 * t.p / 4) * 128;
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
// B operands: Bready[g][l][chunk][hi|lo] = [Gi | Gr | -Gi] rows x = chunk*XC + n, K-major canonical.
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
        const float vals[3] = {v.y, v.x, -v.y};
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            float h, r;
            tc::split_tf32_rn(vals[b], h, r);
            const uint32_t o = kmaj(n, b * p + q, c.sbo_b);
            *reinterpret_cast<float*>(hi + o) = h;
            *reinterpret_cast<float*>(lo + o) = r;
        }
    }
}

// ---------------------------------------------------------------------------------------------
// A operands: Eready[g][l][tile][hi|lo] = [Er | Ei] rows = subcarriers of the tile, K-major canonical.
// One thread per subcarrier: conj phasors (binary64 argument reduction) and E = C^T c* in fp32.
template <int PQ>
__global__ void __launch_bounds__(kFT) k_esplit(Topo t, RgCfg c, int Fc, int64_t f0, int ntiles,
                                                const float2* __restrict__ Cd, const double* __restrict__ tau,
                                                const double* __restrict__ freqs, unsigned char* __restrict__ Eready) {
    const int ti = blockIdx.x, l = blockIdx.y;
    const int64_t g = blockIdx.z, gl = g * t.links() + l;
    const int P = t.P, fl = threadIdx.x, f = ti * kFT + fl;
    const float2* Cl = Cd + gl * (int64_t)P * PQ;
    const double* tl = tau + gl * P;
    float2 e[PQ];
#pragma unroll
    for (int q = 0; q < PQ; ++q) e[q] = make_float2(0.f, 0.f);
    if (f < Fc) {
        const double fr = freqs[f0 + f];
#pragma unroll 2
        for (int r = 0; r < P; ++r) {
            const float2 ph = conj_coeff<float>(fr, tl[r]);
#pragma unroll
            for (int q = 0; q < PQ; ++q) cfma(e[q], Cl[q * P + r], ph);
        }
    }
    unsigned char* hi = Eready + ((size_t)gl * ntiles + ti) * 2 * c.TA;
    unsigned char* lo = hi + c.TA;
#pragma unroll
    for (int k4 = 0; k4 < 2 * PQ; k4 += 4) {
        float4 h, r;
        float v[4];
        if (k4 < PQ) {
#pragma unroll
            for (int z = 0; z < 4; ++z) v[z] = e[(k4 + z) % PQ].x;
        } else {
#pragma unroll
            for (int z = 0; z < 4; ++z) v[z] = e[(k4 + z) % PQ].y;
        }
        tc::split_tf32_rn(v[0], h.x, r.x);
        tc::split_tf32_rn(v[1], h.y, r.y);
        tc::split_tf32_rn(v[2], h.z, r.z);
        tc::split_tf32_rn(v[3], h.w, r.w);
        const uint32_t o = kmaj(fl, k4, c.sbo_a);
        *reinterpret_cast<float4*>(hi + o) = h;
        *reinterpret_cast<float4*>(lo + o) = r;
    }
}

// ---------------------------------------------------------------------------------------------
// Gram epilogue helpers (templated on the thread's half H so every accumulator index is static).
namespace {

// serving-Gram rows of half H: MP = 8 -> {0,7,2,5} / {1,6,3,4}; MP = 4 -> {0,3} / {1,2} (balanced
// lower-triangle entry counts: 18 / 18 and 5 / 5)
template <int MP, int H> __host__ __device__ constexpr int srow_n() { return MP / 2; }
template <int MP, int H> __host__ __device__ constexpr int srow(int idx) {
    // MP = 8: h0 {0,7,2,5}, h1 {1,6,3,4};  MP = 4: h0 {0,3}, h1 {1,2}
    return MP == 8 ? (H == 0 ? (idx == 0 ? 0 : idx == 1 ? 7 : idx == 2 ? 2 : 5)
                             : (idx == 0 ? 1 : idx == 1 ? 6 : idx == 2 ? 3 : 4))
                   : (H == 0 ? (idx == 0 ? 0 : 3) : (idx == 0 ? 1 : 2));
}
template <int MP, int H> __host__ __device__ constexpr int srow_off(int idx) {
    int o = 0;
    for (int z = 0; z < idx; ++z) o += srow<MP, H>(z) + 1;
    return o;
}

__device__ __forceinline__ double2 f2d(uint32_t re, uint32_t im) {
    return make_double2((double)__uint_as_float(re), (double)__uint_as_float(im));
}

template <int MP>
__device__ __forceinline__ void tmem_ldmp(uint32_t taddr, uint32_t (&r)[MP]);
template <> __device__ __forceinline__ void tmem_ldmp<8>(uint32_t taddr, uint32_t (&r)[8]) { tc::tmem_ld8_nw(taddr, r); }
template <> __device__ __forceinline__ void tmem_ldmp<4>(uint32_t taddr, uint32_t (&r)[4]) { tc::tmem_ld4_nw(taddr, r); }

// one chunk of the serving Gram: acc(row, r') += H(row, c) conj(H(r', c)), r' <= row
template <int MP, int H>
__device__ __forceinline__ void serving_chunk(uint32_t col0, int XC, double2 (&acc)[32]) {
    for (int cl = 0; cl < XC / MP; ++cl) {
        uint32_t hr[MP], hi[MP];
        tmem_ldmp<MP>(col0 + XC + MP * cl, hr);  // Hr of slot 0
        tmem_ldmp<MP>(col0 + MP * cl, hi);       // Hi of slot 0
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

// one chunk of the pair Gram: acc(row - H*MP/2, r') += Hx(row, c) conj(Ha(r', c)), rows of half H
template <int MP, int H>
__device__ __forceinline__ void pair_chunk(uint32_t col0, int XC, double2 (&acc)[32]) {
    constexpr int RH = MP / 2;
    for (int cl = 0; cl < XC / MP; ++cl) {
        uint32_t ar[MP], ai[MP];
        uint32_t xr[RH], xi[RH];
        tmem_ldmp<MP>(col0 + 3 * XC + MP * cl, ar);  // Hr of slot 1 (anchor)
        tmem_ldmp<MP>(col0 + 2 * XC + MP * cl, ai);  // Hi of slot 1
        if constexpr (RH == 4) {
            tc::tmem_ld4_nw(col0 + XC + MP * cl + H * RH, xr);
            tc::tmem_ld4_nw(col0 + MP * cl + H * RH, xi);
        } else {
            uint32_t t4r[4], t4i[4];
            tc::tmem_ld4_nw(col0 + XC + MP * cl, t4r);
            tc::tmem_ld4_nw(col0 + MP * cl, t4i);
            tc::tmem_wait_ld();
#pragma unroll
            for (int z = 0; z < RH; ++z) {
                xr[z] = t4r[H * RH + z];
                xi[z] = t4i[H * RH + z];
            }
        }
        tc::tmem_wait_ld();
        double2 x[RH];
#pragma unroll
        for (int z = 0; z < RH; ++z) x[z] = f2d(xr[z], xi[z]);
#pragma unroll
        for (int r2 = 0; r2 < MP; ++r2) {
            const double2 a = f2d(ar[r2], ai[r2]);
#pragma unroll
            for (int z = 0; z < RH; ++z) cfmac(acc[z * MP + r2], x[z], a);
        }
    }
}

template <int MP, int H>
__device__ __forceinline__ void write_serving(double2* __restrict__ out, int m, const double2 (&acc)[32]) {
#pragma unroll
    for (int idx = 0; idx < srow_n<MP, H>(); ++idx) {
        const int row = srow<MP, H>(idx);
#pragma unroll
        for (int r2 = 0; r2 < MP; ++r2) {
            if (r2 <= row) {
                double2 v = acc[srow_off<MP, H>(idx) + r2];
                if (r2 == row) v.y = 0.0;
                out[row + m * r2] = v;
                if (r2 != row) out[r2 + m * row] = make_double2(v.x, -v.y);
            }
        }
    }
}

template <int MP, int H>
__device__ __forceinline__ void write_pair(double2* __restrict__ out, int m, const double2 (&acc)[32]) {
    constexpr int RH = MP / 2;
#pragma unroll
    for (int z = 0; z < RH; ++z)
#pragma unroll
        for (int r2 = 0; r2 < MP; ++r2) out[(H * RH + z) + m * r2] = acc[z * MP + r2];
}

}  // namespace

template <int MP>
__global__ void __launch_bounds__(kRgThreads, 1) k_rgram(Topo t, RgCfg c, int Fc, int ntiles, int64_t pf0, int64_t Fs,
                                                         const unsigned char* __restrict__ Bready,
                                                         const unsigned char* __restrict__ Eready,
                                                         double2* __restrict__ PG) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint64_t a_full, a_empty, b_full[2], b_empty[2], t_full[2], t_empty[2];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int u = blockIdx.x, users = t.users(), links = t.links();
    const int64_t g = blockIdx.y;
    const int J = t.J, K = t.K, i = u / K, j = u % K;
    const int XC = c.XC, nch = c.nch;
    unsigned char* sA = smem;                 // [slot][hi | lo]
    unsigned char* sB = smem + 4 * c.TA;      // [stage][slot][hi | lo]
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
    // link of slot `slot` in job jb: job 0 = serving (i,i,j); job jb > 0: k = jb-th cell != i,
    // slot 0 = receive link (k,i,j), slot 1 = anchor (k,k,0)
    auto job_link = [&](int jb, int slot) -> int {
        if (jb == 0) return (i * J + i) * K + j;
        int k = jb - 1;
        if (k >= i) ++k;
        return slot == 0 ? (k * J + i) * K + j : (k * J + k) * K;
    };
    const int njobs = J;

    if (warp == kEpiWarps) {
        // ---------------- TMA producer
        if (lane == 0) {
            uint32_t cnt = 0, nj = 0;
            for (int ti = 0; ti < ntiles; ++ti) {
                for (int jb = 0; jb < njobs; ++jb, ++nj) {
                    const int ns = jb == 0 ? 1 : 2;
                    if (nj > 0) tc::mbar_wait(&a_empty, (nj - 1) & 1);
                    tc::mbar_arrive_expect_tx(&a_full, (uint32_t)ns * 2 * c.TA);
                    for (int sl = 0; sl < ns; ++sl) {
                        const int64_t gl = g * links + job_link(jb, sl);
                        tc::bulk_g2s(sA + (size_t)sl * 2 * c.TA, Eready + ((size_t)gl * ntiles + ti) * 2 * c.TA,
                                     2 * c.TA, &a_full);
                    }
                    for (int ch = 0; ch < nch; ++ch, ++cnt) {
                        const int st = cnt & 1;
                        const uint32_t use = cnt >> 1;
                        if (use > 0) tc::mbar_wait(&b_empty[st], (use - 1) & 1);
                        tc::mbar_arrive_expect_tx(&b_full[st], (uint32_t)ns * 2 * c.TB);
                        for (int sl = 0; sl < ns; ++sl) {
                            const int64_t gl = g * links + job_link(jb, sl);
                            tc::bulk_g2s(sB + ((size_t)st * 2 + sl) * 2 * c.TB, Bready + ((size_t)gl * nch + ch) * 2 * c.TB,
                                         2 * c.TB, &b_full[st]);
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == kEpiWarps + 1) {
        // ---------------- MMA issuer
        if (lane == 0) {
            const uint32_t idesc = tc::idesc_tf32(kFT, XC);
            const uint32_t roff = (uint32_t)(c.p / 4) * 128;  // B[:, p:3p] = [Gr | -Gi]
            uint32_t cnt = 0, nj = 0;
            for (int ti = 0; ti < ntiles; ++ti) {
                for (int jb = 0; jb < njobs; ++jb, ++nj) {
                    const int ns = jb == 0 ? 1 : 2;
                    tc::mbar_wait(&a_full, nj & 1);
                    tc::fence_after_sync();
                    for (int ch = 0; ch < nch; ++ch, ++cnt) {
                        const int st = cnt & 1;
                        const uint32_t use = cnt >> 1;
                        tc::mbar_wait(&b_full[st], use & 1);
                        if (use > 0) tc::mbar_wait(&t_empty[st], (use - 1) & 1);
                        tc::fence_after_sync();
                        for (int sl = 0; sl < ns; ++sl) {
                            const uint32_t dI = tb + (uint32_t)(st * 4 * XC + sl * 2 * XC), dR = dI + XC;
                            const uint32_t ab = tc::smem_u32(sA + (size_t)sl * 2 * c.TA);
                            const uint32_t bb = tc::smem_u32(sB + ((size_t)st * 2 + sl) * 2 * c.TB);
#pragma unroll 1
                            for (int pass = 0; pass < 3; ++pass) {
                                const uint32_t a0 = ab + (pass == 2 ? c.TA : 0u);
                                const uint32_t b0 = bb + (pass == 1 ? c.TB : 0u);
                                for (int kk = 0; kk < c.ks; ++kk) {
                                    const uint64_t da = tc::smem_desc(a0 + kk * 256, 128, c.sbo_a);
                                    const uint64_t dbi = tc::smem_desc(b0 + kk * 256, 128, c.sbo_b);
                                    const uint64_t dbr = tc::smem_desc(b0 + roff + kk * 256, 128, c.sbo_b);
                                    const uint32_t acc = (pass > 0 || kk > 0) ? 1u : 0u;
                                    tc::mma_tf32(dI, da, dbi, idesc, acc);
                                    tc::mma_tf32(dR, da, dbr, idesc, acc);
                                }
                            }
                        }
                        tc::commit(&b_empty[st]);
                        tc::commit(&t_full[st]);
                    }
                    tc::commit(&a_empty);
                }
            }
        }
        __syncwarp();
    } else {
        // ---------------- Gram epilogue: thread (subcarrier fl of the tile, half h)
        const int q4 = warp & 3, h = warp >> 2;
        const int fl = 32 * q4 + lane;
        const uint32_t lanebase = (uint32_t)(32 * q4) << 16;
        const int m = c.m, S = J;
        uint32_t cnt = 0;
        for (int ti = 0; ti < ntiles; ++ti) {
            const int f = ti * kFT + fl;
            const bool valid = f < Fc;
            const int64_t row = ((int64_t)g * Fs + pf0 + f) * users + u;
            for (int jb = 0; jb < njobs; ++jb) {
                double2 acc[32];
#pragma unroll
                for (int z = 0; z < 32; ++z) acc[z] = make_double2(0.0, 0.0);
                for (int ch = 0; ch < nch; ++ch, ++cnt) {
                    const int st = cnt & 1;
                    const uint32_t use = cnt >> 1;
                    tc::mbar_wait(&t_full[st], use & 1);
                    tc::fence_after_sync();
                    const uint32_t col0 = tb + lanebase + (uint32_t)(st * 4 * XC);
                    if (jb == 0) {
                        if (h == 0) serving_chunk<MP, 0>(col0, XC, acc);
                        else serving_chunk<MP, 1>(col0, XC, acc);
                    } else {
                        if (h == 0) pair_chunk<MP, 0>(col0, XC, acc);
                        else pair_chunk<MP, 1>(col0, XC, acc);
                    }
                    tc::fence_before_sync();
                    tc::mbar_arrive(&t_empty[st]);
                }
                if (valid) {
                    double2* out = PG + (row * S + jb) * (int64_t)m * m;
                    if (jb == 0) {
                        if (h == 0) write_serving<MP, 0>(out, m, acc);
                        else write_serving<MP, 1>(out, m, acc);
                    } else {
                        if (h == 0) write_pair<MP, 0>(out, m, acc);
                        else write_pair<MP, 1>(out, m, acc);
                    }
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
    switch (t.p) {
#define GWT_ES(PQ) \
    case PQ: k_esplit<PQ><<<ge, kFT, 0, st>>>(t, c, Fc, f0, ntiles, (const float2*)Cd, tau, freqs, (unsigned char*)Eready); break;
        GWT_ES(8) GWT_ES(12) GWT_ES(16) GWT_ES(24) GWT_ES(32)
#undef GWT_ES
        default: return cudaErrorNotSupported;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    dim3 grid(t.users(), (unsigned)ngroups);
    if (t.m == 8) {
        e = cudaFuncSetAttribute(k_rgram<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
        if (e != cudaSuccess) return e;
        k_rgram<8><<<grid, kRgThreads, c.smem, st>>>(t, c, Fc, ntiles, pf0, Fs, (const unsigned char*)Bready,
                                                     (const unsigned char*)Eready, PG);
    } else {
        e = cudaFuncSetAttribute(k_rgram<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
        if (e != cudaSuccess) return e;
        k_rgram<4><<<grid, kRgThreads, c.smem, st>>>(t, c, Fc, ntiles, pf0, Fs, (const unsigned char*)Bready,
                                                     (const unsigned char*)Eready, PG);
    }
    return cudaGetLastError();
}

}  // namespace gwtk
