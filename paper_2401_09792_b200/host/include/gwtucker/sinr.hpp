// gwt:: drop-in API (B200 backend) — mirrors proj/include/gwtucker/sinr.hpp (pipeline level).
#pragma once

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

/// B200: rebuild + precoder + covariance + Woodbury/Cholesky + filter + SINR in batched kernels.
SinrReport run_compressed_pipeline(const SystemTopology& topology, const GroupwiseFactorSet& factors,
                                   const std::vector<Vector>& coeffs, InterferenceScope scope);

/// Batched extension: one report per coefficient grid (subcarrier), all on the device in one call.
std::vector<SinrReport> run_compressed_pipeline_batched(const SystemTopology& topology,
                                                        const GroupwiseFactorSet& factors,
                                                        const std::vector<std::vector<Vector>>& coeffs_per_grid,
                                                        InterferenceScope scope);

enum class PipelinePath { full, compressed };
FlopLedger flop_estimate(const SystemTopology& topology, const CompressionRanks& ranks, PipelinePath path);

}  // namespace gwt
