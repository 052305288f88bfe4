// gwt:: drop-in API (B200 backend) — mirrors proj/include/gwtucker/sinr.hpp (pipeline level).
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "gwtucker/channel.hpp"
#include "gwtucker/decompose.hpp"
#include "gwtucker/flops.hpp"

namespace gwt {

struct CompressedChannels {
    SystemTopology topology;
    CompressionRanks ranks;
    std::vector<Matrix> h;
    const Matrix& at(int k, int i, int j) const {
        return h[(k * topology.num_cells + i) * topology.users_per_cell + j];
    }
};

/// Top-L SVD of a serving channel (sinr.hpp:14-20): V (n x L), singular values, U (m x L).
struct Precoder {
    Matrix v;
    std::vector<double> singular_values;
    Matrix u;
};

struct StreamSinr {
    double signal_power = 0.0;
    double sinr = 0.0;  // linear scale
};

/// Small-form representation of the full covariance inverse (sinr.hpp:116-119).
struct WoodburyInverse {
    Matrix t;  // m x m, Qs^-1 (Qs - sigma^2 I)
    double inv_sigma_sq = 0.0;
};

struct SinrReport {
    int num_cells = 0;
    int users_per_cell = 0;
    int num_streams = 0;
    std::vector<double> signal_power;  // user-major, stream inner
    std::vector<double> sinr;
    FlopLedger ledger;
    double seconds = 0.0;
    int user_index(int i, int j) const { return i * users_per_cell + j; }
    double sinr_at(int i, int j, int r) const { return sinr[user_index(i, j) * num_streams + r]; }
};

std::vector<std::pair<int, int>> scope_pairs(const SystemTopology& topology, InterferenceScope scope, int i, int j);

CompressedChannels assemble_all_compressed(const SystemTopology& topology, const GroupwiseFactorSet& factors,
                                           const std::vector<Vector>& coeffs, FlopLedger* ledger = nullptr);

struct AssembledChannels {
    SystemTopology topology;
    std::vector<Matrix> h;  // num_links(), each M x N
    const Matrix& at(int k, int i, int j) const {
        return h[(k * topology.num_cells + i) * topology.users_per_cell + j];
    }
};

// Single-system stage API of the full-size path (sinr.hpp:69-89) and the whole-system evaluation on
// assembled channels (sinr.hpp:128-129), the reference's literal per-user route: device SVD
// (truncated_svd) and device Cholesky solve (gwt_hpd_solve), Matrix products on the host side.
// run_full_pipeline below is the batched device path of the same computation.
AssembledChannels assemble_all_full(const ChannelSet& channels, FlopLedger* ledger = nullptr);
Precoder precoder_full(const Matrix& h, int streams, FlopLedger* ledger = nullptr);
std::vector<Precoder> precoders_full(const AssembledChannels& assembled, FlopLedger* ledger = nullptr);
Matrix covariance_full(const AssembledChannels& assembled, const std::vector<Precoder>& precoders,
                       InterferenceScope scope, int i, int j, FlopLedger* ledger = nullptr);
Matrix filter_full(const Matrix& q, const Matrix& h_serving, const Matrix& v_serving, FlopLedger* ledger = nullptr);
std::vector<StreamSinr> sinr_full(const Matrix& w, const Matrix& q, const Matrix& h_serving, const Matrix& v_serving,
                                  FlopLedger* ledger = nullptr);
SinrReport evaluate_assembled(const AssembledChannels& assembled, InterferenceScope scope, FlopLedger initial = {});
/// Individual-model evaluation (sinr.hpp:141-143): per-link factors rebuilt at full size, then the full path.
SinrReport run_reconstructed_pipeline(const SystemTopology& topology, const std::vector<TuckerFactors>& links,
                                      const std::vector<Vector>& coeffs, InterferenceScope scope);

// Single-system stage API of the compressed path (sinr.hpp:99-124). The batched pipeline below runs
// these stages fused on the device; the stage functions keep the reference's building blocks for
// callers that compose them: the SVD and the Cholesky run on the device (truncated_svd ->
// batched eigensolver, woodbury_inverse_apply -> gwt_hpd_solve), the m x n products and the
// per-stream formula use the Matrix type like the Eigen expressions they replace.
Precoder precoder_compressed(const Matrix& h_small, int streams, FlopLedger* ledger = nullptr);
std::vector<Precoder> precoders_compressed(const CompressedChannels& compressed, FlopLedger* ledger = nullptr);
Matrix covariance_compressed(const CompressedChannels& compressed, const std::vector<Precoder>& precoders,
                             InterferenceScope scope, int i, int j, FlopLedger* ledger = nullptr);
WoodburyInverse woodbury_inverse_apply(const Matrix& q_small, double sigma, FlopLedger* ledger = nullptr);
Matrix filter_compressed(const WoodburyInverse& inverse, const Matrix& h_serving, const Matrix& v_serving,
                         FlopLedger* ledger = nullptr);
std::vector<StreamSinr> sinr_compressed(const Matrix& w_small, const Matrix& q_small, const Matrix& h_serving,
                                        const Matrix& v_serving, FlopLedger* ledger = nullptr);

/// B200: rebuild + precoder + covariance + Woodbury/Cholesky + filter + SINR in batched kernels.
SinrReport run_compressed_pipeline(const SystemTopology& topology, const GroupwiseFactorSet& factors,
                                   const std::vector<Vector>& coeffs, InterferenceScope scope);

/// Batched extension: one report per coefficient grid (subcarrier), all on the device in one call.
std::vector<SinrReport> run_compressed_pipeline_batched(const SystemTopology& topology,
                                                        const GroupwiseFactorSet& factors,
                                                        const std::vector<std::vector<Vector>>& coeffs_per_grid,
                                                        InterferenceScope scope);

/// Full-size comparator (sinr.hpp:134): H(f) = X x3 c^* per link, SVD precoders, MMSE SINR — batched
/// kernels on the device (gwt_sinr_full; M <= 8).
SinrReport run_full_pipeline(const ChannelSet& channels, InterferenceScope scope);

enum class PipelinePath { full, compressed };
FlopLedger flop_estimate(const SystemTopology& topology, const CompressionRanks& ranks, PipelinePath path);

}  // namespace gwt
