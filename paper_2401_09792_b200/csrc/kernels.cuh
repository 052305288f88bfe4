// Kernel launch interface shared by the C-ABI layer (capi.cu) and the
// kernel translation units. Host-callable launchers only; no torch types.
#pragma once

#include <algorithm>
#include "common.cuh"

namespace gwtk {

// Which factor a batch item (group g, link l) multiplies with.
enum FactorIndex : int { FI_LINK = 0, FI_BASE = 1, FI_USER = 2, FI_GROUP = 3 };

__device__ __forceinline__ int64_t factor_index(const Topo& t, int kind, int64_t g, int l) {
    const int k = l / (t.J * t.K);
    const int rem = l % (t.J * t.K);
    switch (kind) {
        case FI_LINK: return g * t.links() + l;
        case FI_BASE: return g * t.J + k;
        case FI_USER: return g * t.users() + rem;  // rem = i*K + j
        default: return g;
    }
}

struct GemmDesc {
    // Out(row, col) = sum_k In(row, k) * conj(U(k, col)),   row in [0, R*S), k < Kd, col < Cols
    // In(row, k)  at in  + item*in_item  + (row % R)*rs_in  + (row / R)*s_in  + k*ks_in
    // Out(row,col) at out + item*out_item + (row % R)*rs_out + (row / R)*s_out + col*cs_out
    // U(k, col)   at u + factor_index(item)*ublk + k*uk + col*ucol, conjugated when uconj
    // (default: column-major Kd x Cols block, conjugated -> mode product with U^H)
    int R, S, Kd, Cols;
    int64_t in_item, rs_in, s_in, ks_in;
    int64_t out_item, rs_out, s_out, cs_out;
    int fkind;
    int64_t ublk = -1, uk = 1, ucol = -1;
    int uconj = 1;
};

struct GramDesc {
    // Out[set](x, y) = sum_{links of set} sum_{t < T1*T2} V(x, t) conj(V(y, t)), x,y < D
    // V(x, t) at v + item*v_item + x*xs + (t % T1)*t1s + (t / T1)*t2s, item = g*links + l
    int D, T1, T2;
    int64_t v_item, xs, t1s, t2s;
    int set_kind;  // FI_USER (rx: links (k,i,j) over k), FI_BASE (tx), FI_LINK (delay), FI_GROUP (pooled)
};


// k_tucker.cu
template <class T> cudaError_t launch_cgemm(const Topo& t, const GemmDesc& d, int64_t ngroups, const void* in,
                                            const void* U, void* out, cudaStream_t st);
// part (nullable): scratch for K-split partial Grams (used when few sets would leave SMs idle)
// allow_tc: the tensor-core Gram for row-block unfoldings (the context's GWT_GRAM_TC, read at ctx creation)
template <class T> cudaError_t launch_gram(const Topo& t, const GramDesc& d, int64_t ngroups, int sets_per_group,
                                           const void* V, void* out, void* part, size_t part_bytes, cudaStream_t st,
                                           bool allow_tc = true);
// tuning / diagnostic switch read once per process (the per-call hot paths never call getenv)
const char* env_once(const char* name);
// per-group ||v||^2 in fp64; deterministic two-level reduction through `partial`
// (ngroups * kSqnormMaxBlocks doubles) when a group spans many blocks
constexpr int kSqnormMaxBlocks = 128;
template <class T> cudaError_t launch_group_sqnorm(const void* v, int64_t per_group, int64_t ngroups, double* out,
                                                   double* partial, cudaStream_t st);
cudaError_t launch_stop_freeze(int64_t ngroups, const double* trace, const double* energy, int stride, int s, int* stop,
                               const void* A, const void* B, const void* Cf, const void* Gc, void* frozen, int64_t a_sz,
                               int64_t b_sz, int64_t c_sz, int64_t g_sz, cudaStream_t st);
cudaError_t launch_unfreeze(int64_t ngroups, const int* stop, void* A, void* B, void* Cf, void* Gc, const void* frozen,
                            int64_t a_sz, int64_t b_sz, int64_t c_sz, int64_t g_sz, cudaStream_t st);
cudaError_t launch_hpd_solve(int m, int nrhs, int64_t batch, const void* Q, const void* B, int check_cond, void* Lw,
                             void* X, int* status, cudaStream_t st);
cudaError_t launch_objective(int64_t ngroups, const double* energy, const double* captured, double* trace, int stride,
                             int slot, cudaStream_t st);
template <class T> cudaError_t launch_broadcast(const void* src, void* dst, int64_t elems, int copies, int64_t ngroups,
                                                cudaStream_t st);
bool gram_tc_fits(const GramDesc& d);  // k_tc.cu: rows = contiguous T1-complex blocks (tx Gram of W2), D >= 128
cudaError_t launch_gram_tc(const Topo& t, const GramDesc& d, int64_t ngroups, int sets_per_group, const void* V,
                           void* out, cudaStream_t st);  // k_tc.cu (c64, 3xTF32 tcgen05)
// k_eig.cu
template <class T> cudaError_t launch_heev_topk(int D, int count, int64_t batch, const void* in, void* out,
                                                double* evals, double2* ws_a, double* ws_z, double2* ws_x, int* fail,
                                                cudaStream_t st);
// k_orth.cu: binary64 Cholesky-QR re-orthonormalisation of fp32 eigenvector blocks (+ phase convention)
cudaError_t launch_orth_cholqr(int D, int count, int64_t batch, void* V, cudaStream_t st);
cudaError_t launch_cplx_widen(const void* in, void* out, int64_t n, cudaStream_t st);   // c64 -> c128
cudaError_t launch_cplx_narrow(const void* in, void* out, int64_t n, cudaStream_t st);  // c128 -> c64
size_t heev_ws_a_elems(int D);
size_t heev_ws_z_elems(int D, int count);
// k_sinr.cu
template <class T> cudaError_t launch_rebuild(const Topo& t, int ngroups, int Fc, int64_t f0, int64_t Ftot,
                                              const void* Cd, const void* G, const double* tau, const double* freqs,
                                              const void* coeffs, void* H, cudaStream_t st);
template <class T> cudaError_t launch_pair_gram(const Topo& t, int scope, int S, int Fc, int ngroups, int64_t f0,
                                                int64_t Ftot, const void* H, double2* PG, cudaStream_t st);
// k_rebuild.cu: SGEMM-tiled rebuild for large cores (c64, m n >= 256)
bool rebuild_mm_fits(const Topo& t);
cudaError_t launch_rebuild_mm(const Topo& t, int ngroups, int Fc, int64_t f0, const void* Cd, const void* G,
                              const double* tau, const double* freqs, void* H, cudaStream_t st);
// k_rgram.cu: stage R fused with the pair Grams on tcgen05 (c64, paper scope, m in {4, 8}): pre-split
// B operands of the cores once per call (launch_rgram_prep), then per subcarrier chunk the E operands
// and the Gram kernel writing PG[g][f - pf0][user][J][m*m]
bool rgram_fits(const Topo& t);
size_t rgram_bready_bytes(const Topo& t, int64_t ngroups);
size_t rgram_eready_bytes(const Topo& t, int64_t ngroups, int Fc);
cudaError_t launch_rgram_prep(const Topo& t, int64_t ngroups, const void* G, void* Bready, cudaStream_t st);
cudaError_t launch_rgram(const Topo& t, int64_t ngroups, int Fc, int64_t f0, int64_t pf0, int64_t Fs, const void* Cd,
                         const double* tau, const double* freqs, const void* Bready, void* Eready, double2* PG,
                         cudaStream_t st);
// k_users.cu: stage S for the paper scope (serving Gram, eig, anchor precoders, interference, MMSE)
bool sinr_users_fits(const Topo& t, size_t csize);
template <class T> cudaError_t launch_sinr_users(const Topo& t, int64_t nslices, int fc, int64_t Ftot, int64_t f0,
                                                 double sigma, const void* H, double* sinr, double* signal,
                                                 int* status, cudaStream_t st);
// PG mode of the same kernel: Grams precomputed by k_rgram (PG[item][user][J][m*m]), binary64 throughout
bool sinr_users_pg_fits(const Topo& t);
cudaError_t launch_sinr_users_pg(const Topo& t, int64_t nslices, int fc, int64_t Ftot, int64_t f0, double sigma,
                                 const double2* PG, double* sinr, double* signal, int* status, cudaStream_t st);
cudaError_t launch_sinr_small(const Topo& t, int scope, int S, int64_t items, double sigma, int fc, int64_t Ftot,
                              int64_t f0, const double2* PG, double* EG, double* sinr, double* signal, int* status,
                              cudaStream_t st);

}  // namespace gwtk
