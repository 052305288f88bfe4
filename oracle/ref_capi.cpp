// ORACLE — TEST INFRASTRUCTURE ONLY. Flat C entry points over the REFERENCE'S OWN
// sources (/root/reference/proj/src/{tensor,linalg,channel,decompose,sinr,archive,
// metrics}.cpp, compiled unchanged against oracle/eigen_shim by oracle/Makefile `ref`
// into oracle/_ref/libgwtref.so). Used only by tests/ to pin the oracle restatement
// (oracle/gwt_oracle.cpp) to the reference itself. Array layouts are the product's
// (DESIGN.md §3): interleaved binary64 complex, tensors mode-1 fastest, factor
// matrices column-major, links k-major then i then j.
#include <complex>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "gwtucker/archive.hpp"
#include "gwtucker/channel.hpp"
#include "gwtucker/decompose.hpp"
#include "gwtucker/sinr.hpp"

namespace {

using gwt::Cplx;

void put_err(char* err, int len, const char* msg) {
    if (err && len > 0) {
        std::strncpy(err, msg, static_cast<std::size_t>(len) - 1);
        err[len - 1] = 0;
    }
}

template <class F>
int guarded(char* err, int len, F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        put_err(err, len, e.what());
        return 1;
    } catch (const std::runtime_error& e) {
        put_err(err, len, e.what());
        return 2;
    } catch (const std::exception& e) {
        put_err(err, len, e.what());
        return 3;
    }
}

const Cplx* cc(const double* p) { return reinterpret_cast<const Cplx*>(p); }
Cplx* cp(double* p) { return reinterpret_cast<Cplx*>(p); }

gwt::Matrix load(const Cplx* p, int r, int c) {
    gwt::Matrix m(r, c);
    std::copy(p, p + static_cast<std::size_t>(r) * c, m.data());
    return m;
}
void store(const gwt::Matrix& m, Cplx* p) { std::copy(m.data(), m.data() + m.size(), p); }

gwt::SystemTopology topo(int J, int K, int M, int N, int P, int L, double sigma) {
    gwt::SystemTopology t;
    t.num_cells = J;
    t.users_per_cell = K;
    t.rx_antennas = M;
    t.tx_antennas = N;
    t.num_taps = P;
    t.num_streams = L;
    t.noise_std = sigma;
    return t;
}

}  // namespace

extern "C" {

// gwt::groupwise_solve (decompose.cpp:309-381; the reference's own stop rule) per group.
// X [g][links][P][N][M]; outputs A [g][users][m][M], B [g][J][n][N], C [g][links][p][P],
// G [g][links][p][n][m], trace [g][sweeps+1] (entries past iterations_run left 0), iters [g].
int ref_groupwise_solve(int J, int K, int M, int N, int P, int m, int n, int p, long long ngroups, const double* X,
                        int sweeps, int pooled, double* A, double* B, double* Cf, double* G, double* trace, int* iters,
                        char* err, int len) {
    return guarded(err, len, [&] {
        const int links = J * J * K, users = J * K;
        const std::size_t ts = static_cast<std::size_t>(M) * N * P;
        for (long long g = 0; g < ngroups; ++g) {
            gwt::ChannelSet cs;
            cs.topology = topo(J, K, M, N, P, 1, 0.1);
            for (int l = 0; l < links; ++l) {
                gwt::Tensor3 x(M, N, P);
                std::copy(cc(X) + (g * links + l) * ts, cc(X) + (g * links + l + 1) * ts, x.data());
                cs.tensors.push_back(std::move(x));
                cs.coeffs.push_back(gwt::Vector::Zero(P));
            }
            gwt::CompressionRanks r;
            r.m = m;
            r.n = n;
            r.p = p;
            auto res = pooled ? gwt::shared_solve(cs, r, sweeps) : gwt::groupwise_solve(cs, r, sweeps);
            const auto& f = res.first;
            for (int u = 0; u < users; ++u) store(f.rx_factors[u], cp(A) + (g * users + u) * M * m);
            for (int k = 0; k < J; ++k) store(f.tx_factors[k], cp(B) + (g * J + k) * N * n);
            for (int l = 0; l < links; ++l) {
                store(f.delay_factors[l], cp(Cf) + (g * links + l) * P * p);
                const gwt::Tensor3& core = f.cores[l];
                std::copy(core.data(), core.data() + core.size(), cp(G) + (g * links + l) * m * n * p);
            }
            for (std::size_t s = 0; s < res.second.objective.size() && s < static_cast<std::size_t>(sweeps) + 1; ++s)
                trace[g * (sweeps + 1) + static_cast<long long>(s)] = res.second.objective[s];
            iters[g] = res.second.iterations_run;
        }
    });
}

// gwt::run_compressed_pipeline (sinr.cpp:296-326) per (group, subcarrier):
// C [g][links][p][P], G [g][links][p][n][m], coeffs [g][F][links][P]; sinr/signal [g][F][users][L].
int ref_sinr_compressed(int J, int K, int P, int m, int n, int p, int L, double sigma, int scope, long long ngroups,
                        const double* Cf, const double* G, const double* coeffs, long long F, double* sinr,
                        double* signal, long long* ledger6, char* err, int len) {
    return guarded(err, len, [&] {
        const int links = J * J * K, users = J * K;
        const gwt::SystemTopology t = topo(J, K, m, n, P, L, sigma);
        for (long long g = 0; g < ngroups; ++g) {
            gwt::GroupwiseFactorSet fs;
            fs.num_cells = J;
            fs.users_per_cell = K;
            fs.ranks.m = m;
            fs.ranks.n = n;
            fs.ranks.p = p;
            for (int l = 0; l < links; ++l) {
                fs.delay_factors.push_back(load(cc(Cf) + (g * links + l) * P * p, P, p));
                gwt::Tensor3 core(m, n, p);
                std::copy(cc(G) + (g * links + l) * m * n * p, cc(G) + (g * links + l + 1) * m * n * p, core.data());
                fs.cores.push_back(std::move(core));
            }
            for (long long f = 0; f < F; ++f) {
                std::vector<gwt::Vector> co;
                for (int l = 0; l < links; ++l) co.push_back(load(cc(coeffs) + ((g * F + f) * links + l) * P, P, 1));
                const gwt::SinrReport rep = gwt::run_compressed_pipeline(
                    t, fs, co, scope == 0 ? gwt::InterferenceScope::full : gwt::InterferenceScope::paper_experiment);
                std::copy(rep.sinr.begin(), rep.sinr.end(), sinr + (g * F + f) * users * L);
                std::copy(rep.signal_power.begin(), rep.signal_power.end(), signal + (g * F + f) * users * L);
                if (ledger6 && g == 0 && f == 0) {
                    ledger6[0] = rep.ledger.reconstruct;
                    ledger6[1] = rep.ledger.precoder;
                    ledger6[2] = rep.ledger.covariance;
                    ledger6[3] = rep.ledger.inverse;
                    ledger6[4] = rep.ledger.filter;
                    ledger6[5] = rep.ledger.sinr;
                }
            }
        }
    });
}

// gwt::run_full_pipeline (sinr.cpp:259-294) per (group, subcarrier) on X [g][links][P][N][M].
int ref_sinr_full(int J, int K, int M, int N, int P, int L, double sigma, int scope, long long ngroups,
                  const double* X, const double* coeffs, long long F, double* sinr, double* signal, char* err,
                  int len) {
    return guarded(err, len, [&] {
        const int links = J * J * K, users = J * K;
        const std::size_t ts = static_cast<std::size_t>(M) * N * P;
        for (long long g = 0; g < ngroups; ++g) {
            gwt::ChannelSet cs;
            cs.topology = topo(J, K, M, N, P, L, sigma);
            for (int l = 0; l < links; ++l) {
                gwt::Tensor3 x(M, N, P);
                std::copy(cc(X) + (g * links + l) * ts, cc(X) + (g * links + l + 1) * ts, x.data());
                cs.tensors.push_back(std::move(x));
                cs.coeffs.push_back(gwt::Vector::Zero(P));
            }
            for (long long f = 0; f < F; ++f) {
                for (int l = 0; l < links; ++l) cs.coeffs[l] = load(cc(coeffs) + ((g * F + f) * links + l) * P, P, 1);
                const gwt::SinrReport rep = gwt::run_full_pipeline(
                    cs, scope == 0 ? gwt::InterferenceScope::full : gwt::InterferenceScope::paper_experiment);
                std::copy(rep.sinr.begin(), rep.sinr.end(), sinr + (g * F + f) * users * L);
                std::copy(rep.signal_power.begin(), rep.signal_power.end(), signal + (g * F + f) * users * L);
            }
        }
    });
}

// gwt::generate_channel_set (channel.cpp:154-180): X [links][P][N][M], coeffs [links][P].
int ref_generate_channel_set(int J, int K, int M, int N, int P, int rays, double tap_decay, double rician,
                             double coeff_decay, unsigned long long seed, double* X, double* coeffs, char* err,
                             int len) {
    return guarded(err, len, [&] {
        gwt::GeneratorParams gp;
        gp.rays_per_slice = rays;
        gp.tap_decay = tap_decay;
        gp.rician_factor = rician;
        gp.coeff_decay = coeff_decay;
        const gwt::ChannelSet cs = gwt::generate_channel_set(topo(J, K, M, N, P, 1, 0.1), gp, seed);
        const std::size_t ts = static_cast<std::size_t>(M) * N * P;
        for (std::size_t l = 0; l < cs.tensors.size(); ++l) {
            std::copy(cs.tensors[l].data(), cs.tensors[l].data() + ts, cp(X) + l * ts);
            std::copy(cs.coeffs[l].data(), cs.coeffs[l].data() + P, cp(coeffs) + l * P);
        }
    });
}

// gwt::save_archive (archive.cpp:178-229), groupwise/shared model; factors as ref_groupwise_solve outputs
// for ONE group, coeffs [links][P].
int ref_save_archive(const char* path, int model, int J, int K, int M, int N, int P, int m, int n, int p,
                     const double* A, const double* B, const double* Cf, const double* G, const double* coeffs,
                     char* err, int len) {
    return guarded(err, len, [&] {
        const int links = J * J * K, users = J * K;
        gwt::GroupwiseFactorSet fs;
        fs.num_cells = J;
        fs.users_per_cell = K;
        fs.ranks.m = m;
        fs.ranks.n = n;
        fs.ranks.p = p;
        for (int u = 0; u < users; ++u) fs.rx_factors.push_back(load(cc(A) + u * M * m, M, m));
        for (int k = 0; k < J; ++k) fs.tx_factors.push_back(load(cc(B) + k * N * n, N, n));
        std::vector<gwt::Vector> co;
        for (int l = 0; l < links; ++l) {
            fs.delay_factors.push_back(load(cc(Cf) + l * P * p, P, p));
            gwt::Tensor3 core(m, n, p);
            std::copy(cc(G) + l * m * n * p, cc(G) + (l + 1) * m * n * p, core.data());
            fs.cores.push_back(std::move(core));
            co.push_back(load(cc(coeffs) + l * P, P, 1));
        }
        gwt::save_archive(path, model == 1 ? gwt::ModelKind::shared : gwt::ModelKind::groupwise, fs, co);
    });
}

// gwt::model_name / model_from_name (decompose.cpp:42-56)
const char* ref_model_name(int kind) {
    return gwt::model_name(kind == 0 ? gwt::ModelKind::individual
                                     : kind == 1 ? gwt::ModelKind::shared : gwt::ModelKind::groupwise);
}
int ref_model_from_name(const char* name, char* err, int len) {
    int out = -1;
    const int rc = guarded(err, len, [&] {
        const gwt::ModelKind k = gwt::model_from_name(name);
        out = k == gwt::ModelKind::individual ? 0 : k == gwt::ModelKind::shared ? 1 : 2;
    });
    return rc ? -1 - rc : out;
}

}  // extern "C"
