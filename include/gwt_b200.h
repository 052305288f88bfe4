/*
 * gwt_b200.h — C ABI of the B200-native groupwise-Tucker / compressed-SINR
 * hot path (arXiv 2401.09792). Plain pointers and sizes only; no torch or
 * C++ types cross this boundary, and no exceptions: every entry point returns
 * a gwt_status and gwt_last_error(ctx) holds the reference's message text.
 *
 * Reference interface each entry point replaces (paths relative to
 * /root/reference/proj):
 *   gwt_groupwise_solve      <- gwt::groupwise_solve  include/gwtucker/decompose.hpp:126-128
 *                               (flag GWT_SOLVE_POOLED: gwt::shared_solve decompose.hpp:132-134;
 *                                includes compute_cores decompose.hpp:110 and the
 *                                SolveTrace of decompose.hpp:33-41)
 *   gwt_sinr_compressed      <- gwt::run_compressed_pipeline  include/gwtucker/sinr.hpp:136-137,
 *                               batched over F coefficient grids generated from per-tap
 *                               delays: c_q(f) = exp(+j 2 pi f tau_q)
 *   gwt_sinr_compressed_coeffs <- gwt::run_compressed_pipeline with explicit coefficient
 *                               vectors (ChannelSet::coeffs, channel.hpp:50), F grids
 *   gwt_assemble_compressed  <- gwt::assemble_channel_compressed channel.hpp:78-79 /
 *                               assemble_all_compressed sinr.hpp:111-114 (batched)
 *   gwt_leading_eigenvectors <- gwt::leading_eigenvectors  include/gwtucker/linalg.hpp:16
 *   gwt_reconstruct          <- gwt::reconstruct (decompress)  include/gwtucker/decompose.hpp:84
 *   gwt_flop_estimate        <- gwt::flop_estimate  include/gwtucker/sinr.hpp:148-149
 *   gwt_mode_product         <- gwt::mode_product  include/gwtucker/tensor.hpp:70 (batched)
 *   gwt_sinr_full            <- gwt::run_full_pipeline  include/gwtucker/sinr.hpp:134 (batched over F grids)
 *   gwt_hpd_solve            <- the Eigen::LLT solves of woodbury_inverse_apply (sinr.cpp:205-227) and
 *                               filter_full (sinr.cpp:113-127), batched
 *
 * Layouts. Complex = interleaved (re, im) pairs: float2 for
 * GWT_C64, double2 for GWT_C128 — layout-compatible with std::complex.
 *   X     [groups][links][P][N][M]   channel tensors, mode-1 fastest (tensor.hpp:15-18)
 *   A     [groups][users][m][M]      rx factor per user, column-major M x m
 *   B     [groups][J][n][N]          tx factor per base, column-major N x n
 *   C     [groups][links][p][P]      delay factor per link, column-major P x p
 *   G     [groups][links][p][n][m]   cores, mode-1 fastest
 *   tau   [groups][links][P]         per-tap delays in seconds (binary64)
 *   freqs [F]                        subcarrier frequencies in Hz (binary64)
 *   coeffs[groups][F][links][P]      explicit coefficient vectors (complex, dtype)
 *   sinr, signal [groups][F][users][L] binary64, stream inner (SinrReport, sinr.hpp:51-62)
 *   status [groups][F][users]        int32 gwt_item_status per (subcarrier, user)
 * with link = (k*J + i)*K + j and user = i*K + j (channel.hpp:53-56).
 *
 * Memory: with GWT_MEM_HOST every array argument is a host pointer (copied
 * in/out inside the call, on the context's stream); with GWT_MEM_DEVICE every
 * array argument is a device pointer on the context's device. Calls are
 * synchronous: results are complete when the call returns.
 */
#ifndef GWT_B200_H
#define GWT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gwt_ctx gwt_ctx;

typedef enum {
    GWT_OK = 0,
    GWT_INVALID_ARGUMENT = 1, /* reference throws std::invalid_argument */
    GWT_RUNTIME_ERROR = 2,    /* reference throws std::runtime_error */
    GWT_CUDA_ERROR = 3,
    GWT_NO_DEVICE = 4
} gwt_status;

typedef enum { GWT_C64 = 0, GWT_C128 = 1 } gwt_dtype;
typedef enum { GWT_MEM_HOST = 0, GWT_MEM_DEVICE = 1 } gwt_mem;
typedef enum { GWT_SCOPE_FULL = 0, GWT_SCOPE_PAPER = 1 } gwt_scope; /* InterferenceScope channel.hpp:33 */

/* Per-(subcarrier, user) outcome of the batched SINR; the C++ wrapper rethrows
 * the reference's exception for the first failing item in reference order. The low
 * byte is the code; GWT_ITEM_NEG_DENOM carries the first failing stream r in bits
 * 8+ (status = 3 + 256 r) for the reference's "... negative for stream r ..." text.
 * GWT_ITEM_RANK_DEFICIENT raises nothing (the reference's SVD completes such a
 * precoder with arbitrary null-space columns; the Gram route flags the item). */
typedef enum {
    GWT_ITEM_OK = 0,
    GWT_ITEM_NOT_PD = 1,        /* "woodbury_inverse_apply: covariance is numerically singular" sinr.cpp:211-212 */
    GWT_ITEM_ILL_COND = 2,      /* "... (condition estimate above 1e14)" sinr.cpp:216-218 */
    GWT_ITEM_NEG_DENOM = 3,     /* "sinr: interference-plus-noise power is negative ..." sinr.cpp:35-37 */
    GWT_ITEM_NONFINITE = 4,     /* "...: non-finite input" sinr.cpp:23-26 */
    GWT_ITEM_RANK_DEFICIENT = 5 /* a precoder singular value is zero (measure-zero input) */
} gwt_item_status;

/* SystemTopology (channel.hpp:13-27) */
typedef struct {
    int32_t num_cells;      /* J */
    int32_t users_per_cell; /* K */
    int32_t rx_antennas;    /* M */
    int32_t tx_antennas;    /* N */
    int32_t num_taps;       /* P */
    int32_t num_streams;    /* L */
    double noise_std;       /* sigma */
} gwt_topology;

/* CompressionRanks (decompose.hpp:18-24) */
typedef struct {
    int32_t m, n, p;
} gwt_ranks;

/* FlopLedger (flops.hpp:10-31) */
typedef struct {
    int64_t reconstruct, precoder, covariance, inverse, filter, sinr;
} gwt_ledger;

#define GWT_SOLVE_EARLY_STOP 1u /* reference stop rule decrease < 1e-10*energy (decompose.cpp:363-368) */
#define GWT_SOLVE_POOLED 2u     /* shared model: one rx and one tx factor pooled over all links */
#define GWT_SOLVE_INIT 4u       /* A, B, C hold a warm start on entry (decompose.hpp:127 `init`) */

int gwt_ctx_create(gwt_ctx** out, int device);
void gwt_ctx_destroy(gwt_ctx* ctx);
const char* gwt_last_error(const gwt_ctx* ctx);
/* Use an external CUDA stream (cudaStream_t passed as void*); NULL = the ctx's own non-blocking stream.
   The legacy default stream is passed as cudaStreamLegacy ((void*)1), not NULL. Every call is ordered
   after prior work on the bound stream and synchronises it before returning. */
int gwt_ctx_set_stream(gwt_ctx* ctx, void* stream);
/* Number of kernel launches issued through this ctx since creation. */
int64_t gwt_ctx_launch_count(const gwt_ctx* ctx);
/* Device time (ms, CUDA events on the ctx stream) of the last call's stages:
 * [0] whole call, [1] Tucker init, [2] Tucker sweeps, [3] cores/objective,
 * [4] rebuild, [5] pair Grams, [6] eig+MMSE, [7] host<->device copies. */
int gwt_ctx_stage_times(const gwt_ctx* ctx, double* ms8);

int gwt_groupwise_solve(gwt_ctx* ctx, const gwt_topology* topo, const gwt_ranks* ranks, int64_t ngroups,
                        gwt_dtype dtype, gwt_mem mem, const void* X, int32_t sweeps, uint32_t flags, void* A, void* B,
                        void* C, void* G, double* trace /* [groups][sweeps+1] */, int32_t* iters /* [groups] */,
                        double* energy /* [groups] */);

int gwt_sinr_compressed(gwt_ctx* ctx, const gwt_topology* topo, const gwt_ranks* ranks, int64_t ngroups,
                        gwt_dtype dtype, gwt_mem mem, const void* C, const void* G, const double* tau,
                        const double* freqs, int64_t F, gwt_scope scope, double* sinr, double* signal,
                        int32_t* status, gwt_ledger* ledger /* nullable, host */);

int gwt_sinr_compressed_coeffs(gwt_ctx* ctx, const gwt_topology* topo, const gwt_ranks* ranks, int64_t ngroups,
                               gwt_dtype dtype, gwt_mem mem, const void* C, const void* G, const void* coeffs,
                               int64_t F, gwt_scope scope, double* sinr, double* signal, int32_t* status,
                               gwt_ledger* ledger);

/* Full-size SINR on the uncompressed channels H(f) = X x3 c(f)^* (the e_c / R_t comparator).
 * tau/freqs when coeffs == NULL (coeffs: [groups][F][links][P]). M <= 8. */
int gwt_sinr_full(gwt_ctx* ctx, const gwt_topology* topo, int64_t ngroups, gwt_dtype dtype, gwt_mem mem,
                  const void* X, const double* tau, const double* freqs, const void* coeffs, int64_t F,
                  gwt_scope scope, double* sinr, double* signal, int32_t* status, gwt_ledger* ledger);

/* H~ [groups][F][links][n][m] (column-major m x n per item). tau/freqs when coeffs == NULL. */
int gwt_assemble_compressed(gwt_ctx* ctx, const gwt_topology* topo, const gwt_ranks* ranks, int64_t ngroups,
                            gwt_dtype dtype, gwt_mem mem, const void* C, const void* G, const double* tau,
                            const double* freqs, const void* coeffs, int64_t F, void* H);

/* Batched leading_eigenvectors: H [batch][n][n] Hermitian (column-major),
 * out [batch][count][n]: leading `count` eigenvectors, descending, phase-normalised. */
int gwt_leading_eigenvectors(gwt_ctx* ctx, int32_t n, int32_t count, int64_t batch, gwt_dtype dtype, gwt_mem mem,
                             const void* H, void* out, double* evals /* nullable [batch][count] */);

/* X^ = G x1 A x2 B x3 C per link: X [groups][links][P][N][M]. */
int gwt_reconstruct(gwt_ctx* ctx, const gwt_topology* topo, const gwt_ranks* ranks, int64_t ngroups,
                    gwt_dtype dtype, gwt_mem mem, const void* A, const void* B, const void* C, const void* G,
                    void* X);

/* Y[b] = X[b] x_mode U (tensor.hpp:68-70): X [batch][d3][d2][d1] mode-1 fastest, U rows x dim(mode)
 * column-major, shared by the batch; Y has dim(mode) replaced by `rows`. */
int gwt_mode_product(gwt_ctx* ctx, gwt_dtype dtype, gwt_mem mem, int64_t batch, int32_t d1, int32_t d2, int32_t d3,
                     const void* X, int32_t rows, const void* U, int32_t mode, void* Y);

/* X = Q^-1 B for `batch` m x m Hermitian positive-definite Q and m x nrhs B (complex128, column-major)
 * through a binary64 Cholesky on the device: the LLT of woodbury_inverse_apply (sinr.cpp:205-227,
 * B = Q - sigma^2 I, check_cond = 1) and filter_full (sinr.cpp:113-127, B = H V, check_cond = 0).
 * status[b]: 0 ok, 1 not positive definite, 2 condition estimate above 1e14 (check_cond), 4
 * non-finite input; the C++ drop-in rethrows the reference's exception texts. */
int gwt_hpd_solve(gwt_ctx* ctx, int32_t m, int32_t nrhs, int64_t batch, gwt_mem mem, const void* Q, const void* B,
                  int32_t check_cond, void* X, int32_t* status);

/* Closed-form system ledger (sinr.cpp:353-382); path 0 = full, 1 = compressed. Host only. */
int gwt_flop_estimate(const gwt_topology* topo, const gwt_ranks* ranks, int32_t path, gwt_ledger* out);

/* Seeded synthetic channels of BASELINE.json: one ray per tap,
 * ULA half-wavelength steering, angles U(-pi/3, pi/3), a_q ~ CN(0, p_q),
 * p_q ∝ exp(-decay*q) normalised, tau_q ~ U(0, max_delay). Host buffers; groups
 * [group0, group0+ngroups) of the stream defined by `seed`. nthreads host threads. */
int gwt_generate_channels(const gwt_topology* topo, int64_t group0, int64_t ngroups, uint64_t seed, double pdp_decay,
                          double max_delay, gwt_dtype dtype, void* X, double* tau, int32_t nthreads);

#ifdef __cplusplus
}
#endif

#endif /* GWT_B200_H */
