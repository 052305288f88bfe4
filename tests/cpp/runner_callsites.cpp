// Compile-only check (tests/test_abi.py::test_runner_callsites_compile): the way the reference's
// control plane drives the hot path — proj/src/runner.cpp:82-113 (compress / run_compressed_once:
// model switch, structured bindings of the solver pairs, IndividualResult, the two compressed
// pipelines) and :115-140 (run_full_pipeline timing fields, ledgers) — compiles unchanged against the
// drop-in headers. Written against the public API only; ExperimentConfig (config.hpp, control plane,
// out of scope) is replaced by a local struct with the fields those call sites read.
#include <string>
#include <utility>
#include <vector>

#include "gwtucker/channel.hpp"
#include "gwtucker/decompose.hpp"
#include "gwtucker/flops.hpp"
#include "gwtucker/sinr.hpp"

namespace {

struct LocalConfig {
    gwt::ModelKind model = gwt::ModelKind::groupwise;
    gwt::CompressionRanks ranks;
    int iters = 20;
    gwt::InterferenceScope scope{};
};

struct Compressed {
    gwt::SolveTrace trace;
    gwt::GroupwiseFactorSet factors;
    std::vector<gwt::TuckerFactors> links;
};

Compressed compress_like(const LocalConfig& cfg, const gwt::ChannelSet& channels) {
    Compressed out;
    if (cfg.model == gwt::ModelKind::individual) {
        gwt::IndividualResult r = gwt::individual_solve(channels, cfg.ranks, cfg.iters);
        out.links = std::move(r.links);
        out.trace = std::move(r.trace);
    } else if (cfg.model == gwt::ModelKind::shared) {
        auto [fs, trace] = gwt::shared_solve(channels, cfg.ranks, cfg.iters);
        out.factors = std::move(fs);
        out.trace = std::move(trace);
    } else {
        auto [fs, trace] = gwt::groupwise_solve(channels, cfg.ranks, cfg.iters);
        out.factors = std::move(fs);
        out.trace = std::move(trace);
    }
    return out;
}

gwt::SinrReport evaluate_like(const LocalConfig& cfg, const gwt::ChannelSet& channels, const Compressed& run) {
    if (cfg.model == gwt::ModelKind::individual)
        return gwt::run_reconstructed_pipeline(channels.topology, run.links, channels.coeffs, cfg.scope);
    return gwt::run_compressed_pipeline(channels.topology, run.factors, channels.coeffs, cfg.scope);
}

double timing_like(const LocalConfig& cfg, const gwt::ChannelSet& channels, const Compressed& run) {
    const gwt::SinrReport full = gwt::run_full_pipeline(channels, cfg.scope);
    const gwt::SinrReport comp = evaluate_like(cfg, channels, run);
    const gwt::FlopLedger lf = full.ledger, lc = comp.ledger;
    (void)lf;
    (void)lc;
    const std::string name = gwt::model_name(gwt::model_from_name("groupwise"));
    return full.seconds + comp.seconds + static_cast<double>(name.size());
}

}  // namespace

// referenced so the functions above are not discarded before type checking
void* gwt_runner_callsites_probe[] = {reinterpret_cast<void*>(&compress_like), reinterpret_cast<void*>(&timing_like)};
