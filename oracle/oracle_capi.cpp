// ORACLE — TEST INFRASTRUCTURE ONLY. Flat C entry points over the oracle
// restatement so pytest (ctypes) and bench.py's CPU-baseline leg can drive it.
// Array layouts are the product's: complex numbers are
// interleaved binary64 pairs, tensors mode-1 fastest, factor matrices
// column-major, grids k-major then i then j.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <thread>

#include "gwt_oracle.hpp"

using namespace orc;

namespace {

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

const Cplx* cp(const double* p) { return reinterpret_cast<const Cplx*>(p); }
Cplx* cp(double* p) { return reinterpret_cast<Cplx*>(p); }

Mat load_mat(const Cplx* p, int r, int c) {
    Mat m(r, c);
    std::copy(p, p + static_cast<std::size_t>(r) * c, m.a.begin());
    return m;
}
void store_mat(const Mat& m, Cplx* p) { std::copy(m.a.begin(), m.a.end(), p); }

Tensor3 load_t(const Cplx* p, int d1, int d2, int d3) {
    Tensor3 t(d1, d2, d3);
    std::copy(p, p + t.a.size(), t.a.begin());
    return t;
}

Topology topo(int J, int K, int M, int N, int P, int L, double sigma) {
    Topology t;
    t.J = J; t.K = K; t.M = M; t.N = N; t.P = P; t.L = L; t.sigma = sigma;
    return t;
}

// Run body(g) for g in [0, ngroups) on `nthreads` std::threads; groups are
// independent. First error (lowest group) wins.
template <class F>
int for_groups(std::int64_t ngroups, int nthreads, char* err, int len, F&& body) {
    nthreads = std::max(1, std::min<int>(nthreads, static_cast<int>(std::max<std::int64_t>(1, ngroups))));
    std::vector<int> codes(static_cast<std::size_t>(ngroups), 0);
    std::vector<std::string> msgs(static_cast<std::size_t>(ngroups));
    std::atomic<std::int64_t> next{0};
    auto worker = [&]() {
        for (;;) {
            const std::int64_t g = next.fetch_add(1);
            if (g >= ngroups) break;
            char buf[512] = {0};
            codes[g] = guarded(buf, sizeof(buf), [&] { body(g); });
            msgs[g] = buf;
        }
    };
    if (nthreads == 1) {
        worker();
    } else {
        std::vector<std::thread> th;
        for (int t = 0; t < nthreads; ++t) th.emplace_back(worker);
        for (auto& t : th) t.join();
    }
    for (std::int64_t g = 0; g < ngroups; ++g)
        if (codes[g]) {
            put_err(err, len, msgs[g].c_str());
            return codes[g];
        }
    return 0;
}

void load_factor_set(FactorSet& fs, const Topology& t, const Ranks& r, const Cplx* A, const Cplx* B, const Cplx* C,
                     const Cplx* G) {
    fs.J = t.J; fs.K = t.K; fs.ranks = r;
    fs.rx.resize(t.users());
    fs.tx.resize(t.J);
    fs.delay.resize(t.links());
    for (int u = 0; u < t.users(); ++u) fs.rx[u] = load_mat(A + static_cast<std::size_t>(u) * t.M * r.m, t.M, r.m);
    for (int k = 0; k < t.J; ++k) fs.tx[k] = load_mat(B + static_cast<std::size_t>(k) * t.N * r.n, t.N, r.n);
    for (int l = 0; l < t.links(); ++l) fs.delay[l] = load_mat(C + static_cast<std::size_t>(l) * t.P * r.p, t.P, r.p);
    if (G) {
        fs.cores.resize(t.links());
        const std::size_t cs = static_cast<std::size_t>(r.m) * r.n * r.p;
        for (int l = 0; l < t.links(); ++l) fs.cores[l] = load_t(G + l * cs, r.m, r.n, r.p);
    }
}

void add_ledger(std::int64_t* out, const Ledger& l) {
    if (!out) return;
    out[0] += l.reconstruct; out[1] += l.precoder; out[2] += l.covariance;
    out[3] += l.inverse; out[4] += l.filter; out[5] += l.sinr;
}

}  // namespace

extern "C" {

int orc_generate_reference(int J, int K, int M, int N, int P, int rays, double tap_decay, double rician,
                           double coeff_decay, unsigned long long seed, double* X, double* coeffs, char* err, int len) {
    return guarded(err, len, [&] {
        Topology t = topo(J, K, M, N, P, 1, 0.1);
        GenParams gp;
        gp.rays = rays; gp.tap_decay = tap_decay; gp.rician = rician; gp.coeff_decay = coeff_decay;
        if (gp.rays < 1) throw std::invalid_argument("generator: rays_per_slice must be >= 1");
        if (!(gp.tap_decay > 0)) throw std::invalid_argument("generator: tap_decay must be > 0");
        if (!(gp.rician > 0)) throw std::invalid_argument("generator: rician_factor must be > 0");
        if (!(gp.coeff_decay > 0)) throw std::invalid_argument("generator: coeff_decay must be > 0");
        std::vector<Tensor3> xs;
        std::vector<std::vector<Cplx>> cs;
        generate_reference_set(t, gp, seed, xs, cs);
        const std::size_t ts = static_cast<std::size_t>(M) * N * P;
        for (std::size_t l = 0; l < xs.size(); ++l) {
            std::copy(xs[l].a.begin(), xs[l].a.end(), cp(X) + l * ts);
            std::copy(cs[l].begin(), cs[l].end(), cp(coeffs) + l * P);
        }
    });
}

int orc_heev(int n, const double* A, double* evals, double* evecs, char* err, int len) {
    return guarded(err, len, [&] {
        Eig e = hermitian_eig(load_mat(cp(A), n, n));
        std::copy(e.values.begin(), e.values.end(), evals);
        store_mat(e.vectors, cp(evecs));
    });
}

int orc_leading_eigenvectors(int n, const double* A, int count, double* out, char* err, int len) {
    return guarded(err, len, [&] { store_mat(leading_eigenvectors(load_mat(cp(A), n, n), count), cp(out)); });
}

int orc_truncated_svd(int r, int c, const double* A, int count, double* U, double* S, double* V, char* err, int len) {
    return guarded(err, len, [&] {
        Svd s = truncated_svd(load_mat(cp(A), r, c), count);
        store_mat(s.u, cp(U));
        std::copy(s.s.begin(), s.s.end(), S);
        store_mat(s.v, cp(V));
    });
}

int orc_mode_product(int d1, int d2, int d3, const double* X, int ur, int uc, const double* U, int mode, double* Y,
                     char* err, int len) {
    return guarded(err, len, [&] {
        Tensor3 y = mode_product(load_t(cp(X), d1, d2, d3), load_mat(cp(U), ur, uc), mode);
        std::copy(y.a.begin(), y.a.end(), cp(Y));
    });
}

int orc_contract_mode3(int d1, int d2, int d3, const double* X, int clen, const double* c, double* H, char* err,
                       int len) {
    return guarded(err, len, [&] {
        std::vector<Cplx> cv(cp(c), cp(c) + clen);
        store_mat(contract_mode3(load_t(cp(X), d1, d2, d3), cv), cp(H));
    });
}

int orc_hosvd(int d1, int d2, int d3, const double* X, int m, int n, int p, double* A, double* B, double* C,
              double* G, char* err, int len) {
    return guarded(err, len, [&] {
        Ranks r{m, n, p};
        Hosvd h = hosvd(load_t(cp(X), d1, d2, d3), r);
        store_mat(h.rx, cp(A)); store_mat(h.tx, cp(B)); store_mat(h.delay, cp(C));
        std::copy(h.core.a.begin(), h.core.a.end(), cp(G));
    });
}

int orc_hooi(int d1, int d2, int d3, const double* X, int m, int n, int p, int sweeps, double* A, double* B,
             double* C, double* G, double* trace, int* iters, char* err, int len) {
    return guarded(err, len, [&] {
        Ranks r{m, n, p};
        Hosvd h;
        Trace tr = hooi(load_t(cp(X), d1, d2, d3), r, sweeps, nullptr, h);
        store_mat(h.rx, cp(A)); store_mat(h.tx, cp(B)); store_mat(h.delay, cp(C));
        std::copy(h.core.a.begin(), h.core.a.end(), cp(G));
        for (std::size_t s = 0; s < static_cast<std::size_t>(sweeps) + 1; ++s)
            trace[s] = tr.objective[std::min(s, tr.objective.size() - 1)];
        *iters = tr.iterations_run;
    });
}

int orc_reconstruct(int M, int N, int P, int m, int n, int p, const double* A, const double* B, const double* C,
                    const double* G, double* X, char* err, int len) {
    return guarded(err, len, [&] {
        Tensor3 x = reconstruct(load_t(cp(G), m, n, p), load_mat(cp(A), M, m), load_mat(cp(B), N, n), load_mat(cp(C), P, p));
        std::copy(x.a.begin(), x.a.end(), cp(X));
    });
}

// groupwise (pooled=0) or shared (pooled=1) alternating solve over
// `ngroups` independent channel sets. trace: [ngroups][sweeps+1] (entries
// after an early stop repeat the final objective). init (nullable) = A,B,C.
int orc_alternating_solve(int J, int K, int M, int N, int P, int m, int n, int p, long long ngroups, const double* X,
                          int sweeps, int early_stop, int pooled, const double* initA, const double* initB,
                          const double* initC, int nthreads, double* A, double* B, double* C, double* G, double* trace,
                          int* iters, double* energy, char* err, int len) {
    const Topology t = topo(J, K, M, N, P, 1, 0.1);
    const Ranks r{m, n, p};
    const std::size_t xs_sz = static_cast<std::size_t>(M) * N * P * t.links();
    const std::size_t a_sz = static_cast<std::size_t>(M) * m * t.users(), b_sz = static_cast<std::size_t>(N) * n * J,
                      c_sz = static_cast<std::size_t>(P) * p * t.links(), g_sz = static_cast<std::size_t>(m) * n * p * t.links();
    return for_groups(ngroups, nthreads, err, len, [&](std::int64_t g) {
        std::vector<Tensor3> xs;
        for (int l = 0; l < t.links(); ++l)
            xs.push_back(load_t(cp(X) + g * xs_sz + static_cast<std::size_t>(l) * M * N * P, M, N, P));
        FactorSet init, fs;
        if (initA) load_factor_set(init, t, r, cp(initA) + g * a_sz, cp(initB) + g * b_sz, cp(initC) + g * c_sz, nullptr);
        Trace tr = alternating_solve(t, xs, r, sweeps, initA ? &init : nullptr, pooled != 0, early_stop != 0, fs);
        for (int u = 0; u < t.users(); ++u) store_mat(fs.rx[u], cp(A) + g * a_sz + static_cast<std::size_t>(u) * M * m);
        for (int k = 0; k < J; ++k) store_mat(fs.tx[k], cp(B) + g * b_sz + static_cast<std::size_t>(k) * N * n);
        for (int l = 0; l < t.links(); ++l) {
            store_mat(fs.delay[l], cp(C) + g * c_sz + static_cast<std::size_t>(l) * P * p);
            std::copy(fs.cores[l].a.begin(), fs.cores[l].a.end(), cp(G) + g * g_sz + static_cast<std::size_t>(l) * m * n * p);
        }
        for (int s = 0; s <= sweeps; ++s)
            trace[g * (sweeps + 1) + s] = tr.objective[std::min<std::size_t>(s, tr.objective.size() - 1)];
        iters[g] = tr.iterations_run;
        double e = 0;
        for (auto& x : xs) e += squared_norm(x);
        energy[g] = e;
    });
}

// objective f and projection energy g for given factors (one group).
int orc_objective(int J, int K, int M, int N, int P, int m, int n, int p, const double* X, const double* A,
                  const double* B, const double* C, double* f, double* gproj, char* err, int len) {
    return guarded(err, len, [&] {
        const Topology t = topo(J, K, M, N, P, 1, 0.1);
        const Ranks r{m, n, p};
        std::vector<Tensor3> xs;
        for (int l = 0; l < t.links(); ++l) xs.push_back(load_t(cp(X) + static_cast<std::size_t>(l) * M * N * P, M, N, P));
        FactorSet fs;
        load_factor_set(fs, t, r, cp(A), cp(B), cp(C), nullptr);
        *f = objective_value(t, xs, fs);
        *gproj = projection_energy(t, xs, fs);
    });
}

// which: 0 rx (a=i,b=j), 1 tx (a=k), 2 delay (a=k,b=i,c=j)
int orc_update_gram(int which, int J, int K, int M, int N, int P, int m, int n, int p, const double* X,
                    const double* A, const double* B, const double* C, int a, int b, int c, double* out, char* err,
                    int len) {
    return guarded(err, len, [&] {
        const Topology t = topo(J, K, M, N, P, 1, 0.1);
        const Ranks r{m, n, p};
        std::vector<Tensor3> xs;
        for (int l = 0; l < t.links(); ++l) xs.push_back(load_t(cp(X) + static_cast<std::size_t>(l) * M * N * P, M, N, P));
        FactorSet fs;
        load_factor_set(fs, t, r, cp(A), cp(B), cp(C), nullptr);
        Mat gm = which == 0 ? rx_update_gram(t, xs, fs, a, b) : which == 1 ? tx_update_gram(t, xs, fs, a)
                                                                           : delay_update_gram(t, xs, fs, a, b, c);
        store_mat(gm, cp(out));
    });
}

// Compressed SINR over F coefficient grids per group.
// coeffs: [ngroups][F][links][P] complex; sinr/signal: [ngroups][F][users][L];
// ledger (nullable): 6 int64 summed over everything.
int orc_sinr_compressed(int J, int K, int P, int m, int n, int p, int L, double sigma, int scope, long long ngroups,
                        const double* C, const double* G, const double* coeffs, long long F, int nthreads,
                        double* sinr, double* signal, long long* ledger, char* err, int len) {
    const Topology t = topo(J, K, m, n, P, L, sigma);
    const Ranks r{m, n, p};
    const std::size_t c_sz = static_cast<std::size_t>(P) * p * t.links(), g_sz = static_cast<std::size_t>(m) * n * p * t.links();
    std::vector<Ledger> lg(static_cast<std::size_t>(ngroups));
    int rc = for_groups(ngroups, nthreads, err, len, [&](std::int64_t g) {
        FactorSet fs;
        fs.J = J; fs.K = K; fs.ranks = r;
        fs.delay.resize(t.links());
        fs.cores.resize(t.links());
        for (int l = 0; l < t.links(); ++l) {
            fs.delay[l] = load_mat(cp(C) + g * c_sz + static_cast<std::size_t>(l) * P * p, P, p);
            fs.cores[l] = load_t(cp(G) + g * g_sz + static_cast<std::size_t>(l) * m * n * p, m, n, p);
        }
        for (std::int64_t f = 0; f < F; ++f) {
            std::vector<std::vector<Cplx>> cs(t.links());
            for (int l = 0; l < t.links(); ++l) {
                const Cplx* src = cp(coeffs) + ((g * F + f) * t.links() + l) * static_cast<std::size_t>(P);
                cs[l].assign(src, src + P);
            }
            SinrOut o = run_compressed_pipeline(t, fs, cs, static_cast<Scope>(scope));
            const std::size_t off = static_cast<std::size_t>((g * F + f) * t.users() * L);
            std::copy(o.sinr.begin(), o.sinr.end(), sinr + off);
            std::copy(o.signal.begin(), o.signal.end(), signal + off);
            Ledger& a = lg[g];
            a.reconstruct += o.ledger.reconstruct; a.precoder += o.ledger.precoder; a.covariance += o.ledger.covariance;
            a.inverse += o.ledger.inverse; a.filter += o.ledger.filter; a.sinr += o.ledger.sinr;
        }
    });
    if (ledger) {
        std::fill(ledger, ledger + 6, 0);
        for (auto& l : lg) add_ledger(reinterpret_cast<std::int64_t*>(ledger), l);
    }
    return rc;
}

// Full-size SINR (comparator path) over F coefficient grids per group.
int orc_sinr_full(int J, int K, int M, int N, int P, int L, double sigma, int scope, long long ngroups,
                  const double* X, const double* coeffs, long long F, int nthreads, double* sinr, double* signal,
                  long long* ledger, char* err, int len) {
    const Topology t = topo(J, K, M, N, P, L, sigma);
    const std::size_t xs_sz = static_cast<std::size_t>(M) * N * P * t.links();
    std::vector<Ledger> lg(static_cast<std::size_t>(ngroups));
    int rc = for_groups(ngroups, nthreads, err, len, [&](std::int64_t g) {
        t.validate();
        std::vector<Tensor3> xs;
        for (int l = 0; l < t.links(); ++l)
            xs.push_back(load_t(cp(X) + g * xs_sz + static_cast<std::size_t>(l) * M * N * P, M, N, P));
        for (std::int64_t f = 0; f < F; ++f) {
            std::vector<std::vector<Cplx>> cs(t.links());
            for (int l = 0; l < t.links(); ++l) {
                const Cplx* src = cp(coeffs) + ((g * F + f) * t.links() + l) * static_cast<std::size_t>(P);
                cs[l].assign(src, src + P);
            }
            SinrOut o = run_full_pipeline(t, xs, cs, static_cast<Scope>(scope));
            const std::size_t off = static_cast<std::size_t>((g * F + f) * t.users() * L);
            std::copy(o.sinr.begin(), o.sinr.end(), sinr + off);
            std::copy(o.signal.begin(), o.signal.end(), signal + off);
            Ledger& a = lg[g];
            a.reconstruct += o.ledger.reconstruct; a.precoder += o.ledger.precoder; a.covariance += o.ledger.covariance;
            a.inverse += o.ledger.inverse; a.filter += o.ledger.filter; a.sinr += o.ledger.sinr;
        }
    });
    if (ledger) {
        std::fill(ledger, ledger + 6, 0);
        for (auto& l : lg) add_ledger(reinterpret_cast<std::int64_t*>(ledger), l);
    }
    return rc;
}

// Full pipeline on explicitly given assembled channels h[links] (M x N each).
int orc_evaluate_assembled(int J, int K, int M, int N, int L, double sigma, int scope, const double* H, double* sinr,
                           double* signal, char* err, int len) {
    return guarded(err, len, [&] {
        Topology t = topo(J, K, M, N, 1, L, sigma);
        std::vector<Mat> h;
        for (int l = 0; l < t.links(); ++l) h.push_back(load_mat(cp(H) + static_cast<std::size_t>(l) * M * N, M, N));
        SinrOut o = evaluate_assembled(t, h, static_cast<Scope>(scope), Ledger{});
        std::copy(o.sinr.begin(), o.sinr.end(), sinr);
        std::copy(o.signal.begin(), o.signal.end(), signal);
    });
}

}  // extern "C"
