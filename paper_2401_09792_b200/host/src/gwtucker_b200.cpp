// gwt:: drop-in API over the B200 C ABI (include/gwt_b200.h).
//
// Every numerical hot-path call (mode products, eigensolvers, the groupwise
// solver, compressed assembly and the SINR pipeline) runs on the GPU through
// the C ABI; this file only packs/unpacks the reference's value types and
// rethrows the reference's exceptions (std::invalid_argument /
// std::runtime_error with the same message text). There is no CPU fallback:
// without a CUDA device every GPU-backed call throws.
#include <chrono>
#include <cmath>
#include <limits>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "../../../include/gwt_b200.h"
#include "gwtucker/channel.hpp"
#include "gwtucker/decompose.hpp"
#include "gwtucker/linalg.hpp"
#include "gwtucker/sinr.hpp"
#include "gwtucker/tensor.hpp"

namespace gwt {

// decompose.cpp:42-56
const char* model_name(ModelKind model) {
    switch (model) {
        case ModelKind::individual: return "individual";
        case ModelKind::shared: return "shared";
        case ModelKind::groupwise: return "groupwise";
    }
    return "unknown";
}

ModelKind model_from_name(const std::string& name) {
    static const std::pair<const char*, ModelKind> known[] = {
        {"individual", ModelKind::individual}, {"shared", ModelKind::shared}, {"groupwise", ModelKind::groupwise}};
    for (const auto& k : known)
        if (name == k.first) return k.second;
    throw std::invalid_argument("unknown model '" + name + "' (expected individual, shared or groupwise)");
}

namespace {

struct Ctx {
    gwt_ctx* h = nullptr;
    Ctx() {
        const char* d = std::getenv("GWT_DEVICE");
        const int rc = gwt_ctx_create(&h, d ? std::atoi(d) : 0);
        if (rc != GWT_OK)
            throw std::runtime_error("gwt: no CUDA device available (the B200 backend has no CPU fallback)");
    }
    ~Ctx() { gwt_ctx_destroy(h); }
};

gwt_ctx* ctx() {
    thread_local Ctx c;  // one context per host thread
    return c.h;
}

void check(int rc) {
    if (rc == GWT_OK) return;
    const std::string msg = gwt_last_error(ctx());
    if (rc == GWT_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

gwt_topology ctopo(const SystemTopology& t) {
    return gwt_topology{t.num_cells, t.users_per_cell, t.rx_antennas, t.tx_antennas, t.num_taps, t.num_streams,
                        t.noise_std};
}

std::int64_t i64(Index v) { return static_cast<std::int64_t>(v); }

}  // namespace

// ---------------------------------------------------------------- Matrix
Matrix Matrix::Identity(Index rows, Index cols) {
    Matrix m(rows, cols);
    for (Index i = 0; i < std::min(rows, cols); ++i) m(i, i) = 1.0;
    return m;
}
Matrix Matrix::adjoint() const {
    Matrix o(c_, r_);
    for (Index j = 0; j < c_; ++j)
        for (Index i = 0; i < r_; ++i) o(j, i) = std::conj((*this)(i, j));
    return o;
}
Matrix Matrix::transpose() const {
    Matrix o(c_, r_);
    for (Index j = 0; j < c_; ++j)
        for (Index i = 0; i < r_; ++i) o(j, i) = (*this)(i, j);
    return o;
}
Matrix Matrix::conjugate() const {
    Matrix o(*this);
    for (auto& v : o.a_) v = std::conj(v);
    return o;
}
Matrix Matrix::col(Index j) const {
    Matrix o(r_, 1);
    for (Index i = 0; i < r_; ++i) o(i, 0) = (*this)(i, j);
    return o;
}
Matrix Matrix::leftCols(Index n) const {
    Matrix o(r_, n);
    std::copy(a_.begin(), a_.begin() + r_ * n, o.a_.begin());
    return o;
}
void Matrix::setCol(Index j, const Matrix& v) {
    for (Index i = 0; i < r_; ++i) (*this)(i, j) = v.a_[static_cast<std::size_t>(i)];
}
double Matrix::squaredNorm() const {
    double s = 0;
    for (const auto& v : a_) s += std::norm(v);
    return s;
}
double Matrix::norm() const { return std::sqrt(squaredNorm()); }
bool Matrix::allFinite() const {
    for (const auto& v : a_)
        if (!std::isfinite(v.real()) || !std::isfinite(v.imag())) return false;
    return true;
}
Matrix Matrix::operator*(const Matrix& o) const {
    if (c_ != o.r_) throw std::invalid_argument("Matrix: product shape mismatch");
    Matrix z(r_, o.c_);
    for (Index j = 0; j < o.c_; ++j)
        for (Index k = 0; k < c_; ++k) {
            const Cplx b = o(k, j);
            for (Index i = 0; i < r_; ++i) z(i, j) += (*this)(i, k) * b;
        }
    return z;
}
Matrix Matrix::operator+(const Matrix& o) const { Matrix z(*this); z += o; return z; }
Matrix Matrix::operator-(const Matrix& o) const { Matrix z(*this); z -= o; return z; }
Matrix& Matrix::operator+=(const Matrix& o) {
    for (std::size_t i = 0; i < a_.size(); ++i) a_[i] += o.a_[i];
    return *this;
}
Matrix& Matrix::operator-=(const Matrix& o) {
    for (std::size_t i = 0; i < a_.size(); ++i) a_[i] -= o.a_[i];
    return *this;
}
Matrix operator*(const Cplx& s, const Matrix& m) {
    Matrix z(m);
    for (auto& v : z.a_) v *= s;
    return z;
}
Vector::Vector(const Matrix& m) : Matrix(m.rows() * m.cols(), 1) {
    std::copy(m.data(), m.data() + m.size(), a_.begin());
}

// ---------------------------------------------------------------- Tensor3 (tensor.cpp)
Tensor3::Tensor3(int d1, int d2, int d3) : d1_(d1), d2_(d2), d3_(d3) {
    if (d1 <= 0 || d2 <= 0 || d3 <= 0)
        throw std::invalid_argument("Tensor3: dims must be positive, got (" + std::to_string(d1) + "," +
                                    std::to_string(d2) + "," + std::to_string(d3) + ")");
    data_.assign(static_cast<std::size_t>(d1) * d2 * d3, Cplx(0, 0));
}
int Tensor3::dim(int mode) const {
    switch (mode) {
        case 1: return d1_;
        case 2: return d2_;
        case 3: return d3_;
        default: throw std::invalid_argument("Tensor3::dim: mode must be 1, 2 or 3, got " + std::to_string(mode));
    }
}
Matrix Tensor3::mode1_view() const {
    Matrix m(d1_, static_cast<Index>(d2_) * d3_);
    std::copy(data_.begin(), data_.end(), m.data());
    return m;
}
Matrix Tensor3::slice_view(int i3) const {
    Matrix m(d1_, d2_);
    std::copy(data_.begin() + static_cast<std::size_t>(d1_) * d2_ * i3,
              data_.begin() + static_cast<std::size_t>(d1_) * d2_ * (i3 + 1), m.data());
    return m;
}
void Tensor3::setZero() { std::fill(data_.begin(), data_.end(), Cplx(0, 0)); }

Matrix matricize(const Tensor3& x, int mode) {
    const int d1 = x.dim1(), d2 = x.dim2(), d3 = x.dim3();
    if (mode == 1) return x.mode1_view();
    if (mode == 2) {
        Matrix m(d2, static_cast<Index>(d1) * d3);
        for (int i3 = 0; i3 < d3; ++i3)
            for (int i2 = 0; i2 < d2; ++i2)
                for (int i1 = 0; i1 < d1; ++i1) m(i2, i1 + static_cast<Index>(d1) * i3) = x(i1, i2, i3);
        return m;
    }
    if (mode == 3) {
        Matrix m(d3, static_cast<Index>(d1) * d2);
        for (int i3 = 0; i3 < d3; ++i3)
            for (int i2 = 0; i2 < d2; ++i2)
                for (int i1 = 0; i1 < d1; ++i1) m(i3, i1 + static_cast<Index>(d1) * i2) = x(i1, i2, i3);
        return m;
    }
    throw std::invalid_argument("matricize: mode must be 1, 2 or 3, got " + std::to_string(mode));
}

Tensor3 dematricize(const Matrix& m, int mode, const std::array<int, 3>& dims) {
    const int d1 = dims[0], d2 = dims[1], d3 = dims[2];
    Tensor3 x(d1, d2, d3);
    auto bad = [&](int md) {
        throw std::invalid_argument("dematricize: matrix shape does not match mode-" + std::to_string(md) + " dims");
    };
    if (mode == 1) {
        if (m.rows() != d1 || m.cols() != static_cast<Index>(d2) * d3) bad(1);
        std::copy(m.data(), m.data() + m.size(), x.data());
        return x;
    }
    if (mode == 2) {
        if (m.rows() != d2 || m.cols() != static_cast<Index>(d1) * d3) bad(2);
        for (int i3 = 0; i3 < d3; ++i3)
            for (int i2 = 0; i2 < d2; ++i2)
                for (int i1 = 0; i1 < d1; ++i1) x(i1, i2, i3) = m(i2, i1 + static_cast<Index>(d1) * i3);
        return x;
    }
    if (mode == 3) {
        if (m.rows() != d3 || m.cols() != static_cast<Index>(d1) * d2) bad(3);
        for (int i3 = 0; i3 < d3; ++i3)
            for (int i2 = 0; i2 < d2; ++i2)
                for (int i1 = 0; i1 < d1; ++i1) x(i1, i2, i3) = m(i3, i1 + static_cast<Index>(d1) * i2);
        return x;
    }
    throw std::invalid_argument("dematricize: mode must be 1, 2 or 3, got " + std::to_string(mode));
}

Tensor3 mode_product(const Tensor3& x, const Matrix& u, int mode) {
    if (mode < 1 || mode > 3)
        throw std::invalid_argument("mode_product: mode must be 1, 2 or 3, got " + std::to_string(mode));
    if (u.cols() != x.dim(mode))
        throw std::invalid_argument("mode_product: matrix has " + std::to_string(u.cols()) + " cols but tensor mode " +
                                    std::to_string(mode) + " has size " + std::to_string(x.dim(mode)));
    std::array<int, 3> od = x.dims();
    od[mode - 1] = static_cast<int>(u.rows());
    Tensor3 y(od[0], od[1], od[2]);
    check(gwt_mode_product(ctx(), GWT_C128, GWT_MEM_HOST, 1, x.dim1(), x.dim2(), x.dim3(), x.data(),
                           static_cast<int32_t>(u.rows()), u.data(), mode, y.data()));
    return y;
}

Matrix contract_mode3(const Tensor3& x, const Vector& coeff) {
    if (coeff.size() != x.dim3())
        throw std::invalid_argument("contract_mode3: coefficient length " + std::to_string(coeff.size()) +
                                    " does not match mode-3 size " + std::to_string(x.dim3()));
    Matrix ch(1, coeff.size());  // c^H
    for (Index q = 0; q < coeff.size(); ++q) ch(0, q) = std::conj(coeff(q));
    Tensor3 y = mode_product(x, ch, 3);
    Matrix h(x.dim1(), x.dim2());
    std::copy(y.data(), y.data() + h.size(), h.data());
    return h;
}

Cplx inner(const Tensor3& x, const Tensor3& y) {
    if (!x.same_dims(y)) throw std::invalid_argument("inner: tensor dims differ");
    Cplx acc(0, 0);
    for (std::size_t i = 0; i < x.size(); ++i) acc += x.data()[i] * std::conj(y.data()[i]);
    return acc;
}
double squared_norm(const Tensor3& x) {
    double s = 0;
    for (std::size_t i = 0; i < x.size(); ++i) s += std::norm(x.data()[i]);
    return s;
}
double frobenius_norm(const Tensor3& x) { return std::sqrt(squared_norm(x)); }

// ---------------------------------------------------------------- linalg
void phase_normalize_columns(Matrix& u) {
    for (Index c = 0; c < u.cols(); ++c) {
        Index best = 0;
        double bm = 0.0;
        for (Index r = 0; r < u.rows(); ++r)
            if (std::abs(u(r, c)) > bm) { bm = std::abs(u(r, c)); best = r; }
        if (bm > 0.0) {
            const Cplx f = std::conj(u(best, c)) / bm;
            for (Index r = 0; r < u.rows(); ++r) u(r, c) *= f;
        }
    }
}

static Matrix leading_with_values(const Matrix& h, int count, RealVector* vals) {
    if (h.rows() != h.cols()) throw std::invalid_argument("leading_eigenvectors: matrix is not square");
    if (count < 1 || count > h.rows())
        throw std::invalid_argument("leading_eigenvectors: count " + std::to_string(count) + " out of range for size " +
                                    std::to_string(h.rows()));
    Matrix out(h.rows(), count);
    RealVector ev(static_cast<std::size_t>(count));
    check(gwt_leading_eigenvectors(ctx(), static_cast<int32_t>(h.rows()), count, 1, GWT_C128, GWT_MEM_HOST, h.data(),
                                   out.data(), ev.data()));
    if (vals) *vals = ev;
    return out;
}

Matrix leading_eigenvectors(const Matrix& hermitian, int count) { return leading_with_values(hermitian, count, nullptr); }

TruncatedSvd truncated_svd(const Matrix& a, int count) {
    const Index mr = std::min(a.rows(), a.cols());
    if (count < 1 || count > mr)
        throw std::invalid_argument("truncated_svd: count " + std::to_string(count) + " out of range for " +
                                    std::to_string(a.rows()) + "x" + std::to_string(a.cols()) + " matrix");
    TruncatedSvd s;
    RealVector lam;
    const bool wide = a.rows() <= a.cols();
    const Matrix g = wide ? Matrix(a * a.adjoint()) : Matrix(a.adjoint() * a);
    Matrix e = leading_with_values(g, count, &lam);
    s.singular_values.resize(static_cast<std::size_t>(count));
    for (int c = 0; c < count; ++c) s.singular_values[c] = std::sqrt(std::max(lam[c], 0.0));
    Matrix other = wide ? Matrix(a.adjoint() * e) : Matrix(a * e);
    for (int c = 0; c < count; ++c) {
        const double sv = s.singular_values[c];
        for (Index r = 0; r < other.rows(); ++r) other(r, c) = sv > 0 ? other(r, c) / sv : Cplx(0, 0);
    }
    s.u = wide ? e : other;
    s.v = wide ? other : e;
    for (int c = 0; c < count; ++c) {  // phase from v, mirrored onto u (linalg.cpp:61-77)
        Index best = 0;
        double bm = 0.0;
        for (Index r = 0; r < s.v.rows(); ++r)
            if (std::abs(s.v(r, c)) > bm) { bm = std::abs(s.v(r, c)); best = r; }
        if (bm > 0.0) {
            const Cplx f = std::conj(s.v(best, c)) / bm;
            for (Index r = 0; r < s.v.rows(); ++r) s.v(r, c) *= f;
            for (Index r = 0; r < s.u.rows(); ++r) s.u(r, c) *= f;
        }
    }
    return s;
}

// ---------------------------------------------------------------- channel
void SystemTopology::validate() const {
    gwt_topology t = ctopo(*this);
    gwt_ranks r{1, 1, 1};
    gwt_ledger l;
    if (num_cells < 1) throw std::invalid_argument("topology: num_cells (J) must be >= 1");
    if (users_per_cell < 1) throw std::invalid_argument("topology: users_per_cell (K) must be >= 1");
    if (rx_antennas < 1) throw std::invalid_argument("topology: rx_antennas (M) must be >= 1");
    if (tx_antennas < 1) throw std::invalid_argument("topology: tx_antennas (N) must be >= 1");
    if (num_taps < 1) throw std::invalid_argument("topology: num_taps (P) must be >= 1");
    if (num_streams < 1) throw std::invalid_argument("topology: num_streams (L) must be >= 1");
    if (num_streams > std::min(rx_antennas, tx_antennas))
        throw std::invalid_argument("topology: num_streams (L) must satisfy L <= min(M, N)");
    if (!(noise_std > 0.0)) throw std::invalid_argument("topology: noise_std (sigma) must be > 0");
    (void)gwt_flop_estimate(&t, &r, 1, &l);
}

double ChannelSet::total_squared_norm() const {
    double acc = 0;
    for (const auto& x : tensors) acc += squared_norm(x);
    return acc;
}

Matrix assemble_channel_full(const Tensor3& x, const Vector& coeff, FlopLedger* ledger) {
    Matrix h = contract_mode3(x, coeff);
    if (ledger) ledger->reconstruct += static_cast<std::int64_t>(x.dim1()) * x.dim2() * x.dim3();
    return h;
}

Matrix assemble_channel_compressed(const Tensor3& core, const Matrix& delay_factor, const Vector& coeff,
                                   FlopLedger* ledger) {
    if (delay_factor.rows() != coeff.size())
        throw std::invalid_argument("assemble_channel_compressed: delay factor has " +
                                    std::to_string(delay_factor.rows()) + " rows but coefficient length is " +
                                    std::to_string(coeff.size()));
    if (delay_factor.cols() != core.dim3())
        throw std::invalid_argument("assemble_channel_compressed: delay factor has " +
                                    std::to_string(delay_factor.cols()) + " cols but core mode-3 size is " +
                                    std::to_string(core.dim3()));
    gwt_topology t{1, 1, core.dim1(), core.dim2(), static_cast<int32_t>(coeff.size()), 1, 0.1};
    gwt_ranks r{core.dim1(), core.dim2(), core.dim3()};
    Matrix h(core.dim1(), core.dim2());
    check(gwt_assemble_compressed(ctx(), &t, &r, 1, GWT_C128, GWT_MEM_HOST, delay_factor.data(), core.data(), nullptr,
                                  nullptr, coeff.data(), 1, h.data()));
    if (ledger)
        ledger->reconstruct += static_cast<std::int64_t>(core.dim1()) * core.dim2() * core.dim3() +
                               i64(delay_factor.rows()) * delay_factor.cols();
    return h;
}

// ---------------------------------------------------------------- decompose
void CompressionRanks::validate_against(int d1, int d2, int d3) const {
    if (m < 1 || m > d1)
        throw std::invalid_argument("rank m = " + std::to_string(m) + " out of range for mode-1 size " + std::to_string(d1));
    if (n < 1 || n > d2)
        throw std::invalid_argument("rank n = " + std::to_string(n) + " out of range for mode-2 size " + std::to_string(d2));
    if (p < 1 || p > d3)
        throw std::invalid_argument("rank p = " + std::to_string(p) + " out of range for mode-3 size " + std::to_string(d3));
}

namespace {

void check_channel_dims(const ChannelSet& ch) {  // decompose.cpp:13-21
    const SystemTopology& t = ch.topology;
    if (static_cast<int>(ch.tensors.size()) != t.num_links())
        throw std::invalid_argument("channel set has " + std::to_string(ch.tensors.size()) +
                                    " tensors but topology expects " + std::to_string(t.num_links()));
    for (const auto& x : ch.tensors)
        if (x.dim1() != t.rx_antennas || x.dim2() != t.tx_antennas || x.dim3() != t.num_taps)
            throw std::invalid_argument("channel set: inconsistent tensor dims");
}

struct Packed {
    std::vector<Cplx> X, A, B, C, G;
    std::vector<double> trace, energy;
    std::vector<int32_t> iters;
};

// Solve `groups` channel sets on the device; init (optional) per group.
std::vector<std::pair<GroupwiseFactorSet, SolveTrace>> solve_groups(const std::vector<const ChannelSet*>& groups,
                                                                    const CompressionRanks& ranks, int sweeps,
                                                                    const std::vector<const GroupwiseFactorSet*>* init,
                                                                    bool pooled, bool early_stop) {
    const SystemTopology& t = groups[0]->topology;
    for (auto* g : groups) check_channel_dims(*g);
    ranks.validate_against(t.rx_antennas, t.tx_antennas, t.num_taps);
    if (sweeps < 0) throw std::invalid_argument("solve: sweeps must be >= 0");
    const int J = t.num_cells, K = t.users_per_cell, M = t.rx_antennas, N = t.tx_antennas, P = t.num_taps;
    const int users = J * K, links = J * J * K, m = ranks.m, n = ranks.n, p = ranks.p;
    const std::size_t ng = groups.size();
    Packed pk;
    const std::size_t xs = static_cast<std::size_t>(M) * N * P;
    pk.X.resize(ng * links * xs);
    for (std::size_t g = 0; g < ng; ++g)
        for (int l = 0; l < links; ++l)
            std::copy(groups[g]->tensors[l].data(), groups[g]->tensors[l].data() + xs, pk.X.begin() + (g * links + l) * xs);
    pk.A.resize(ng * users * M * m);
    pk.B.resize(ng * J * N * n);
    pk.C.resize(ng * links * P * p);
    pk.G.resize(ng * links * m * n * p);
    pk.trace.resize(ng * (sweeps + 1));
    pk.energy.resize(ng);
    pk.iters.resize(ng);
    uint32_t flags = (early_stop ? GWT_SOLVE_EARLY_STOP : 0u) | (pooled ? GWT_SOLVE_POOLED : 0u);
    if (init) {
        flags |= GWT_SOLVE_INIT;
        for (std::size_t g = 0; g < ng; ++g) {
            const GroupwiseFactorSet& in = *(*init)[g];
            if (in.num_cells != J || in.users_per_cell != K || in.ranks.m != m || in.ranks.n != n || in.ranks.p != p ||
                static_cast<int>(in.rx_factors.size()) != users || static_cast<int>(in.tx_factors.size()) != J ||
                static_cast<int>(in.delay_factors.size()) != links)
                throw std::invalid_argument("solver init: factor set shape does not match channels/ranks");
            for (int u = 0; u < users; ++u)
                std::copy(in.rx_factors[u].data(), in.rx_factors[u].data() + M * m, pk.A.begin() + (g * users + u) * M * m);
            for (int k = 0; k < J; ++k)
                std::copy(in.tx_factors[k].data(), in.tx_factors[k].data() + N * n, pk.B.begin() + (g * J + k) * N * n);
            for (int l = 0; l < links; ++l)
                std::copy(in.delay_factors[l].data(), in.delay_factors[l].data() + P * p,
                          pk.C.begin() + (g * links + l) * P * p);
        }
    }
    gwt_topology ct = ctopo(t);
    if (ct.num_streams < 1) ct.num_streams = 1;
    gwt_ranks cr{m, n, p};
    check(gwt_groupwise_solve(ctx(), &ct, &cr, static_cast<int64_t>(ng), GWT_C128, GWT_MEM_HOST, pk.X.data(), sweeps,
                              flags, pk.A.data(), pk.B.data(), pk.C.data(), pk.G.data(), pk.trace.data(),
                              pk.iters.data(), pk.energy.data()));
    std::vector<std::pair<GroupwiseFactorSet, SolveTrace>> out(ng);
    for (std::size_t g = 0; g < ng; ++g) {
        GroupwiseFactorSet& fs = out[g].first;
        fs.num_cells = J;
        fs.users_per_cell = K;
        fs.ranks = ranks;
        fs.rx_factors.assign(users, Matrix(M, m));
        fs.tx_factors.assign(J, Matrix(N, n));
        fs.delay_factors.assign(links, Matrix(P, p));
        fs.cores.assign(links, Tensor3(m, n, p));
        for (int u = 0; u < users; ++u)
            std::copy(pk.A.begin() + (g * users + u) * M * m, pk.A.begin() + (g * users + u + 1) * M * m,
                      fs.rx_factors[u].data());
        for (int k = 0; k < J; ++k)
            std::copy(pk.B.begin() + (g * J + k) * N * n, pk.B.begin() + (g * J + k + 1) * N * n, fs.tx_factors[k].data());
        for (int l = 0; l < links; ++l) {
            std::copy(pk.C.begin() + (g * links + l) * P * p, pk.C.begin() + (g * links + l + 1) * P * p,
                      fs.delay_factors[l].data());
            const std::size_t cs = static_cast<std::size_t>(m) * n * p;
            std::copy(pk.G.begin() + (g * links + l) * cs, pk.G.begin() + (g * links + l + 1) * cs, fs.cores[l].data());
        }
        SolveTrace& tr = out[g].second;
        tr.iterations_run = pk.iters[g];
        tr.objective.assign(pk.trace.begin() + g * (sweeps + 1), pk.trace.begin() + g * (sweeps + 1) + pk.iters[g] + 1);
    }
    return out;
}

ChannelSet single(const Tensor3& x) {
    ChannelSet c;
    c.topology.num_cells = 1;
    c.topology.users_per_cell = 1;
    c.topology.rx_antennas = x.dim1();
    c.topology.tx_antennas = x.dim2();
    c.topology.num_taps = x.dim3();
    c.topology.num_streams = 1;
    c.tensors.push_back(x);
    return c;
}

GroupwiseFactorSet as_set(const Matrix& rx, const Matrix& tx, const Matrix& delay) {
    GroupwiseFactorSet fs;
    fs.num_cells = 1;
    fs.users_per_cell = 1;
    fs.ranks = CompressionRanks{static_cast<int>(rx.cols()), static_cast<int>(tx.cols()), static_cast<int>(delay.cols())};
    fs.rx_factors = {rx};
    fs.tx_factors = {tx};
    fs.delay_factors = {delay};
    return fs;
}

// objective f and cores at fixed factors: one device solve with 0 sweeps from `init`
std::pair<GroupwiseFactorSet, SolveTrace> at_factors(const ChannelSet& ch, const GroupwiseFactorSet& fs) {
    std::vector<const ChannelSet*> g{&ch};
    std::vector<const GroupwiseFactorSet*> in{&fs};
    return std::move(solve_groups(g, fs.ranks, 0, &in, false, false)[0]);
}

}  // namespace

std::pair<GroupwiseFactorSet, SolveTrace> groupwise_solve(const ChannelSet& channels, const CompressionRanks& ranks,
                                                          int sweeps, const GroupwiseFactorSet* init) {
    std::vector<const ChannelSet*> g{&channels};
    std::vector<const GroupwiseFactorSet*> in{init};
    return std::move(solve_groups(g, ranks, sweeps, init ? &in : nullptr, false, true)[0]);
}

std::pair<GroupwiseFactorSet, SolveTrace> shared_solve(const ChannelSet& channels, const CompressionRanks& ranks,
                                                       int sweeps, const GroupwiseFactorSet* init) {
    std::vector<const ChannelSet*> g{&channels};
    std::vector<const GroupwiseFactorSet*> in{init};
    return std::move(solve_groups(g, ranks, sweeps, init ? &in : nullptr, true, true)[0]);
}

std::vector<std::pair<GroupwiseFactorSet, SolveTrace>> groupwise_solve_batched(const std::vector<ChannelSet>& groups,
                                                                               const CompressionRanks& ranks,
                                                                               int sweeps, bool early_stop) {
    if (groups.empty()) return {};
    std::vector<const ChannelSet*> g;
    for (const auto& c : groups) {
        if (c.topology.num_cells != groups[0].topology.num_cells ||
            c.topology.users_per_cell != groups[0].topology.users_per_cell)
            throw std::invalid_argument("groupwise_solve_batched: groups must share one topology");
        g.push_back(&c);
    }
    return solve_groups(g, ranks, sweeps, nullptr, false, early_stop);
}

IndividualResult individual_solve(const ChannelSet& channels, const CompressionRanks& ranks, int sweeps,
                                  const GroupwiseFactorSet* init) {
    check_channel_dims(channels);
    const SystemTopology& topo = channels.topology;
    ranks.validate_against(topo.rx_antennas, topo.tx_antennas, topo.num_taps);
    if (sweeps < 0) throw std::invalid_argument("solve: sweeps must be >= 0");
    const int links = topo.num_links();
    std::vector<ChannelSet> sets;
    std::vector<GroupwiseFactorSet> warm;
    sets.reserve(static_cast<std::size_t>(links));
    for (int k = 0; k < topo.num_cells; ++k)
        for (int i = 0; i < topo.num_cells; ++i)
            for (int j = 0; j < topo.users_per_cell; ++j) {
                sets.push_back(single(channels.tensor(k, i, j)));
                if (init) warm.push_back(as_set(init->rx(i, j), init->tx(k), init->delay(k, i, j)));
            }
    std::vector<const ChannelSet*> g;
    std::vector<const GroupwiseFactorSet*> in;
    for (std::size_t l = 0; l < sets.size(); ++l) {
        g.push_back(&sets[l]);
        if (init) in.push_back(&warm[l]);
    }
    auto solved = solve_groups(g, ranks, sweeps, init ? &in : nullptr, false, true);
    IndividualResult result;
    std::size_t longest = 1;
    for (auto& r : solved) {
        result.links.push_back(TuckerFactors{r.first.rx_factors[0], r.first.tx_factors[0], r.first.delay_factors[0],
                                             r.first.cores[0]});
        longest = std::max(longest, r.second.objective.size());
        result.trace.iterations_run = std::max(result.trace.iterations_run, r.second.iterations_run);
    }
    result.trace.objective.assign(longest, 0.0);
    for (auto& r : solved)
        for (std::size_t s2 = 0; s2 < longest; ++s2)
            result.trace.objective[s2] += r.second.objective[std::min(s2, r.second.objective.size() - 1)];
    return result;
}

TuckerFactors hosvd(const Tensor3& x, const CompressionRanks& ranks) {
    ranks.validate_against(x.dim1(), x.dim2(), x.dim3());
    auto r = groupwise_solve(single(x), ranks, 0);
    return TuckerFactors{r.first.rx_factors[0], r.first.tx_factors[0], r.first.delay_factors[0], r.first.cores[0]};
}

std::pair<TuckerFactors, SolveTrace> hooi(const Tensor3& x, const CompressionRanks& ranks, int sweeps,
                                          const TuckerFactors* init) {
    ranks.validate_against(x.dim1(), x.dim2(), x.dim3());
    if (sweeps < 0) throw std::invalid_argument("hooi: sweeps must be >= 0");
    if (init && (init->rx.rows() != x.dim1() || init->rx.cols() != ranks.m || init->tx.rows() != x.dim2() ||
                 init->tx.cols() != ranks.n || init->delay.rows() != x.dim3() || init->delay.cols() != ranks.p))
        throw std::invalid_argument("hooi: init factor shapes do not match tensor dims and ranks");
    GroupwiseFactorSet in;
    if (init) in = as_set(init->rx, init->tx, init->delay);
    auto r = groupwise_solve(single(x), ranks, sweeps, init ? &in : nullptr);
    return {TuckerFactors{r.first.rx_factors[0], r.first.tx_factors[0], r.first.delay_factors[0], r.first.cores[0]},
            r.second};
}

Tensor3 reconstruct(const TuckerFactors& f) {
    const int M = static_cast<int>(f.rx.rows()), N = static_cast<int>(f.tx.rows()), P = static_cast<int>(f.delay.rows());
    gwt_topology t{1, 1, M, N, P, 1, 0.1};
    gwt_ranks r{f.core.dim1(), f.core.dim2(), f.core.dim3()};
    Tensor3 x(M, N, P);
    check(gwt_reconstruct(ctx(), &t, &r, 1, GWT_C128, GWT_MEM_HOST, f.rx.data(), f.tx.data(), f.delay.data(),
                          f.core.data(), x.data()));
    return x;
}

double tucker_residual(const Tensor3& x, const Matrix& rx, const Matrix& tx, const Matrix& delay) {
    return at_factors(single(x), as_set(rx, tx, delay)).second.objective.front();
}

void compute_cores(const ChannelSet& channels, GroupwiseFactorSet& factors) {
    factors.cores = at_factors(channels, factors).first.cores;
}

double objective_value(const ChannelSet& channels, const GroupwiseFactorSet& factors) {
    return at_factors(channels, factors).second.objective.front();
}

double projection_energy(const ChannelSet& channels, const GroupwiseFactorSet& factors) {
    return channels.total_squared_norm() - objective_value(channels, factors);
}

// ---- single Gauss-Seidel factor updates (decompose.cpp:146-193)
Matrix rx_update_gram(const ChannelSet& channels, const GroupwiseFactorSet& factors, int i, int j) {
    const int dim = channels.topology.rx_antennas;
    Matrix gram(dim, dim);
    for (int k = 0; k < channels.topology.num_cells; ++k) {
        const Tensor3 t = mode_product(mode_product(channels.tensor(k, i, j), factors.tx(k).adjoint(), 2),
                                       factors.delay(k, i, j).adjoint(), 3);
        const Matrix w = matricize(t, 1);
        gram += w * w.adjoint();
    }
    return gram;
}

Matrix update_rx_factor(const ChannelSet& channels, const GroupwiseFactorSet& factors, int i, int j) {
    return leading_eigenvectors(rx_update_gram(channels, factors, i, j), factors.ranks.m);
}

Matrix tx_update_gram(const ChannelSet& channels, const GroupwiseFactorSet& factors, int k) {
    const int dim = channels.topology.tx_antennas;
    Matrix gram(dim, dim);
    for (int i = 0; i < channels.topology.num_cells; ++i)
        for (int j = 0; j < channels.topology.users_per_cell; ++j) {
            const Tensor3 t = mode_product(mode_product(channels.tensor(k, i, j), factors.rx(i, j).adjoint(), 1),
                                           factors.delay(k, i, j).adjoint(), 3);
            const Matrix w = matricize(t, 2);
            gram += w * w.adjoint();
        }
    return gram;
}

Matrix update_tx_factor(const ChannelSet& channels, const GroupwiseFactorSet& factors, int k) {
    return leading_eigenvectors(tx_update_gram(channels, factors, k), factors.ranks.n);
}

Matrix delay_update_gram(const ChannelSet& channels, const GroupwiseFactorSet& factors, int k, int i, int j) {
    const Tensor3 t = mode_product(mode_product(channels.tensor(k, i, j), factors.rx(i, j).adjoint(), 1),
                                   factors.tx(k).adjoint(), 2);
    const Matrix w = matricize(t, 3);
    return w * w.adjoint();
}

Matrix update_delay_factor(const ChannelSet& channels, const GroupwiseFactorSet& factors, int k, int i, int j) {
    return leading_eigenvectors(delay_update_gram(channels, factors, k, i, j), factors.ranks.p);
}

// ---------------------------------------------------------------- sinr
std::vector<std::pair<int, int>> scope_pairs(const SystemTopology& topology, InterferenceScope scope, int i, int j) {
    std::vector<std::pair<int, int>> pairs;  // sinr.cpp:47-62
    if (scope == InterferenceScope::full) {
        for (int k = 0; k < topology.num_cells; ++k)
            for (int l = 0; l < topology.users_per_cell; ++l) pairs.emplace_back(k, l);
        return pairs;
    }
    pairs.emplace_back(i, j);
    for (int k = 0; k < topology.num_cells; ++k)
        if (k != i) pairs.emplace_back(k, 0);
    return pairs;
}

// ---- single-system stages of the full-size path (sinr.cpp:67-138)
AssembledChannels assemble_all_full(const ChannelSet& channels, FlopLedger* ledger) {
    AssembledChannels out;
    out.topology = channels.topology;
    out.h.reserve(channels.tensors.size());
    for (std::size_t l = 0; l < channels.tensors.size(); ++l)
        out.h.push_back(assemble_channel_full(channels.tensors[l], channels.coeffs[l], ledger));
    return out;
}

Precoder precoder_full(const Matrix& h, int streams, FlopLedger* ledger) {
    if (streams > std::min(h.rows(), h.cols()))
        throw std::invalid_argument("precoder: stream count " + std::to_string(streams) + " exceeds min dimension of " +
                                    std::to_string(h.rows()) + "x" + std::to_string(h.cols()) + " channel");
    TruncatedSvd svd = truncated_svd(h, streams);
    if (ledger) ledger->precoder += i64(h.rows()) * h.cols() * streams;
    return {std::move(svd.v), std::move(svd.singular_values), std::move(svd.u)};
}

std::vector<Precoder> precoders_full(const AssembledChannels& assembled, FlopLedger* ledger) {
    const SystemTopology& topo = assembled.topology;
    std::vector<Precoder> out;
    out.reserve(static_cast<std::size_t>(topo.num_users()));
    for (int i = 0; i < topo.num_cells; ++i)
        for (int j = 0; j < topo.users_per_cell; ++j)
            out.push_back(precoder_full(assembled.at(i, i, j), topo.num_streams, ledger));
    return out;
}

Matrix covariance_full(const AssembledChannels& assembled, const std::vector<Precoder>& precoders,
                       InterferenceScope scope, int i, int j, FlopLedger* ledger) {
    const SystemTopology& topo = assembled.topology;
    const double sigma = topo.noise_std;
    Matrix q = (sigma * sigma) * Matrix::Identity(topo.rx_antennas, topo.rx_antennas);
    for (const auto& kl : scope_pairs(topo, scope, i, j)) {
        const std::size_t user = static_cast<std::size_t>(kl.first) * topo.users_per_cell + kl.second;
        if (user >= precoders.size()) throw std::invalid_argument("covariance: scope references missing precoder");
        const Matrix term = assembled.at(kl.first, i, j) * precoders[user].v;
        q += term * term.adjoint();
    }
    if (ledger) {
        const std::int64_t M = topo.rx_antennas, N = topo.tx_antennas, L = topo.num_streams;
        ledger->covariance += i64(topo.num_users()) * (M * N * L + M * M * L);
    }
    return q;
}

Matrix filter_full(const Matrix& q, const Matrix& h_serving, const Matrix& v_serving, FlopLedger* ledger) {
    if (!q.allFinite() || !h_serving.allFinite() || !v_serving.allFinite())
        throw std::invalid_argument("filter: non-finite input");
    const Matrix hv = h_serving * v_serving;
    Matrix w(q.rows(), hv.cols());
    int32_t status = 0;
    check(gwt_hpd_solve(ctx(), static_cast<int32_t>(q.rows()), static_cast<int32_t>(hv.cols()), 1, GWT_MEM_HOST,
                        q.data(), hv.data(), 0, w.data(), &status));
    if (status == 4) throw std::invalid_argument("filter: non-finite input");
    if (status != 0) throw std::runtime_error("filter: covariance is not positive definite");
    if (ledger) {
        const std::int64_t M = q.rows(), L = v_serving.cols();
        ledger->inverse += M * M * M;
        ledger->filter += M * M * L;
    }
    return w;
}

std::vector<StreamSinr> sinr_full(const Matrix& w, const Matrix& q, const Matrix& h_serving, const Matrix& v_serving,
                                  FlopLedger* ledger) {
    if (ledger) {
        const std::int64_t M = q.rows(), L = w.cols();
        ledger->sinr += L * (M * M + 2 * M);
    }
    return sinr_compressed(w, q, h_serving, v_serving, nullptr);  // same stream formula (stream_sinrs)
}

SinrReport evaluate_assembled(const AssembledChannels& assembled, InterferenceScope scope, FlopLedger initial) {
    const SystemTopology& topo = assembled.topology;
    SinrReport report;
    report.num_cells = topo.num_cells;
    report.users_per_cell = topo.users_per_cell;
    report.num_streams = topo.num_streams;
    report.ledger = initial;
    report.signal_power.resize(static_cast<std::size_t>(topo.num_users()) * topo.num_streams);
    report.sinr.resize(report.signal_power.size());
    const std::vector<Precoder> precoders = precoders_full(assembled, &report.ledger);
    for (int i = 0; i < topo.num_cells; ++i)
        for (int j = 0; j < topo.users_per_cell; ++j) {
            const Matrix& h = assembled.at(i, i, j);
            const Precoder& pre = precoders[static_cast<std::size_t>(report.user_index(i, j))];
            const Matrix q = covariance_full(assembled, precoders, scope, i, j, &report.ledger);
            const Matrix w = filter_full(q, h, pre.v, &report.ledger);
            const std::vector<StreamSinr> ss = sinr_full(w, q, h, pre.v, &report.ledger);
            for (int r = 0; r < topo.num_streams; ++r) {
                const std::size_t at = static_cast<std::size_t>(report.user_index(i, j)) * topo.num_streams + r;
                report.signal_power[at] = ss[static_cast<std::size_t>(r)].signal_power;
                report.sinr[at] = ss[static_cast<std::size_t>(r)].sinr;
            }
        }
    return report;
}

SinrReport run_reconstructed_pipeline(const SystemTopology& topology, const std::vector<TuckerFactors>& links,
                                      const std::vector<Vector>& coeffs, InterferenceScope scope) {
    if (links.size() != coeffs.size() || static_cast<int>(links.size()) != topology.num_links())
        throw std::invalid_argument("run_reconstructed_pipeline: grid sizes do not match topology");
    const auto t0 = std::chrono::steady_clock::now();
    FlopLedger ledger;
    AssembledChannels assembled;
    assembled.topology = topology;
    assembled.h.reserve(links.size());
    for (std::size_t l = 0; l < links.size(); ++l) {
        const TuckerFactors& f = links[l];
        const Matrix h_small = assemble_channel_compressed(f.core, f.delay, coeffs[l], &ledger);
        assembled.h.push_back(f.rx * h_small * f.tx.transpose());  // Tucker mode-2 convention: B^T
        const std::int64_t M = f.rx.rows(), m = f.rx.cols(), n = f.tx.cols(), N = f.tx.rows();
        ledger.reconstruct += M * m * n + M * n * N;
    }
    SinrReport report = evaluate_assembled(assembled, scope, ledger);
    report.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return report;
}

// ---- single-system stages of the compressed path (sinr.cpp:162-254)
Precoder precoder_compressed(const Matrix& h_small, int streams, FlopLedger* ledger) {
    if (streams > std::min(h_small.rows(), h_small.cols()))
        throw std::invalid_argument("precoder: stream count " + std::to_string(streams) +
                                    " exceeds compressed channel size " + std::to_string(h_small.rows()) + "x" +
                                    std::to_string(h_small.cols()) + " (ranks chosen below stream count)");
    TruncatedSvd svd = truncated_svd(h_small, streams);  // device eigensolver on the Gram
    if (ledger) ledger->precoder += i64(h_small.rows()) * h_small.cols() * streams;
    return {std::move(svd.v), std::move(svd.singular_values), std::move(svd.u)};
}

std::vector<Precoder> precoders_compressed(const CompressedChannels& compressed, FlopLedger* ledger) {
    const SystemTopology& topo = compressed.topology;
    std::vector<Precoder> out;
    out.reserve(static_cast<std::size_t>(topo.num_users()));
    for (int i = 0; i < topo.num_cells; ++i)
        for (int j = 0; j < topo.users_per_cell; ++j)
            out.push_back(precoder_compressed(compressed.at(i, i, j), topo.num_streams, ledger));
    return out;
}

Matrix covariance_compressed(const CompressedChannels& compressed, const std::vector<Precoder>& precoders,
                             InterferenceScope scope, int i, int j, FlopLedger* ledger) {
    const SystemTopology& topo = compressed.topology;
    const double sigma = topo.noise_std;
    const int m = compressed.ranks.m;
    Matrix q = (sigma * sigma) * Matrix::Identity(m, m);
    for (const auto& kl : scope_pairs(topo, scope, i, j)) {
        const std::size_t user = static_cast<std::size_t>(kl.first) * topo.users_per_cell + kl.second;
        if (user >= precoders.size()) throw std::invalid_argument("covariance: scope references missing precoder");
        const Matrix term = compressed.at(kl.first, i, j) * precoders[user].v;
        q += term * term.adjoint();
    }
    if (ledger) {
        const std::int64_t mm = m, n = compressed.ranks.n, L = topo.num_streams;
        ledger->covariance += i64(topo.num_users()) * (mm * n * L + mm * mm * L);
    }
    return q;
}

WoodburyInverse woodbury_inverse_apply(const Matrix& q_small, double sigma, FlopLedger* ledger) {
    if (!(sigma > 0.0)) throw std::invalid_argument("woodbury_inverse_apply: sigma must be > 0");
    if (!q_small.allFinite()) throw std::invalid_argument("woodbury_inverse_apply: non-finite input");
    const Index m = q_small.rows();
    WoodburyInverse out;
    out.t = Matrix(m, m);
    int32_t status = 0;
    const Matrix rhs = q_small - (sigma * sigma) * Matrix::Identity(m, m);
    check(gwt_hpd_solve(ctx(), static_cast<int32_t>(m), static_cast<int32_t>(m), 1, GWT_MEM_HOST, q_small.data(),
                        rhs.data(), 1, out.t.data(), &status));
    if (status == 1) throw std::runtime_error("woodbury_inverse_apply: covariance is numerically singular");
    if (status == 2)
        throw std::runtime_error("woodbury_inverse_apply: covariance is numerically singular "
                                 "(condition estimate above 1e14)");
    if (status == 4) throw std::invalid_argument("woodbury_inverse_apply: non-finite input");
    out.inv_sigma_sq = 1.0 / (sigma * sigma);
    if (ledger) ledger->inverse += 2 * i64(m) * m * m;
    return out;
}

Matrix filter_compressed(const WoodburyInverse& inverse, const Matrix& h_serving, const Matrix& v_serving,
                         FlopLedger* ledger) {
    if (!h_serving.allFinite() || !v_serving.allFinite())
        throw std::invalid_argument("filter_compressed: non-finite input");
    const Matrix hv = h_serving * v_serving;
    Matrix w = inverse.inv_sigma_sq * (hv - inverse.t * hv);
    if (ledger) {
        const std::int64_t m = inverse.t.rows(), L = v_serving.cols();
        ledger->filter += m * m * L + m * L;
    }
    return w;
}

std::vector<StreamSinr> sinr_compressed(const Matrix& w_small, const Matrix& q_small, const Matrix& h_serving,
                                        const Matrix& v_serving, FlopLedger* ledger) {
    const Matrix hv = h_serving * v_serving;
    if (ledger) {
        const std::int64_t m = q_small.rows(), L = w_small.cols();
        ledger->sinr += L * (m * m + 2 * m);
    }
    const int streams = static_cast<int>(w_small.cols());  // stream_sinrs (sinr.cpp:28-43)
    std::vector<StreamSinr> out(static_cast<std::size_t>(streams));
    const Matrix qw = q_small * w_small;
    for (int r = 0; r < streams; ++r) {
        Cplx amp(0, 0), wqw(0, 0);
        for (Index a = 0; a < w_small.rows(); ++a) {
            amp += std::conj(w_small(a, r)) * hv(a, r);
            wqw += std::conj(w_small(a, r)) * qw(a, r);
        }
        const double sp = std::norm(amp);
        double denom = std::real(wqw) - sp;
        if (denom <= -1e-12)
            throw std::runtime_error("sinr: interference-plus-noise power is negative for stream " + std::to_string(r) +
                                     " (numerically invalid configuration)");
        denom = std::max(denom, std::numeric_limits<double>::min());
        out[static_cast<std::size_t>(r)].signal_power = sp;
        out[static_cast<std::size_t>(r)].sinr = sp / denom;
    }
    return out;
}

namespace {

void pack_compressed(const GroupwiseFactorSet& f, std::vector<Cplx>& C, std::vector<Cplx>& G, int& P) {
    const int links = static_cast<int>(f.cores.size());
    P = links ? static_cast<int>(f.delay_factors[0].rows()) : 0;
    const int m = f.ranks.m, n = f.ranks.n, p = f.ranks.p;
    C.resize(static_cast<std::size_t>(links) * P * p);
    G.resize(static_cast<std::size_t>(links) * m * n * p);
    for (int l = 0; l < links; ++l) {
        if (f.delay_factors[l].rows() != P || f.delay_factors[l].cols() != p || f.cores[l].dim3() != p)
            throw std::invalid_argument("assemble_channel_compressed: delay factor has " +
                                        std::to_string(f.delay_factors[l].cols()) + " cols but core mode-3 size is " +
                                        std::to_string(f.cores[l].dim3()));
        std::copy(f.delay_factors[l].data(), f.delay_factors[l].data() + P * p, C.begin() + static_cast<std::size_t>(l) * P * p);
        std::copy(f.cores[l].data(), f.cores[l].data() + m * n * p, G.begin() + static_cast<std::size_t>(l) * m * n * p);
    }
}

// per-item status of the batched kernels -> the reference's exception text (sinr.cpp:28-43, 205-227); code 3
// carries the first failing stream in bits 8+; code 5 (rank-deficient anchor precoder) raises nothing, as in
// the reference
std::string item_error(int st, bool& runtime) {
    runtime = (st & 0xFF) != 4;
    switch (st & 0xFF) {
        case 1: return "woodbury_inverse_apply: covariance is numerically singular";
        case 2: return "woodbury_inverse_apply: covariance is numerically singular (condition estimate above 1e14)";
        case 3:
            return "sinr: interference-plus-noise power is negative for stream " + std::to_string(st >> 8) +
                   " (numerically invalid configuration)";
        case 4: return "woodbury_inverse_apply: non-finite input";
        default: return std::string();
    }
}

}  // namespace

CompressedChannels assemble_all_compressed(const SystemTopology& topology, const GroupwiseFactorSet& factors,
                                           const std::vector<Vector>& coeffs, FlopLedger* ledger) {
    if (coeffs.size() != factors.cores.size())
        throw std::invalid_argument("assemble_all_compressed: coefficient grid does not match cores");
    std::vector<Cplx> C, G;
    int P = 0;
    pack_compressed(factors, C, G, P);
    const int links = static_cast<int>(factors.cores.size());
    std::vector<Cplx> co(static_cast<std::size_t>(links) * P);
    for (int l = 0; l < links; ++l) {
        if (coeffs[l].size() != P)
            throw std::invalid_argument("assemble_channel_compressed: delay factor has " + std::to_string(P) +
                                        " rows but coefficient length is " + std::to_string(coeffs[l].size()));
        std::copy(coeffs[l].data(), coeffs[l].data() + P, co.begin() + static_cast<std::size_t>(l) * P);
    }
    gwt_topology t = ctopo(topology);
    t.num_taps = P;
    gwt_ranks r{factors.ranks.m, factors.ranks.n, factors.ranks.p};
    const int m = r.m, n = r.n;
    std::vector<Cplx> H(static_cast<std::size_t>(links) * m * n);
    check(gwt_assemble_compressed(ctx(), &t, &r, 1, GWT_C128, GWT_MEM_HOST, C.data(), G.data(), nullptr, nullptr,
                                  co.data(), 1, H.data()));
    CompressedChannels out;
    out.topology = topology;
    out.ranks = factors.ranks;
    for (int l = 0; l < links; ++l) {
        Matrix h(m, n);
        std::copy(H.begin() + static_cast<std::size_t>(l) * m * n, H.begin() + static_cast<std::size_t>(l + 1) * m * n,
                  h.data());
        out.h.push_back(std::move(h));
        if (ledger) ledger->reconstruct += static_cast<std::int64_t>(m) * n * r.p + static_cast<std::int64_t>(P) * r.p;
    }
    return out;
}

std::vector<SinrReport> run_compressed_pipeline_batched(const SystemTopology& topology,
                                                        const GroupwiseFactorSet& factors,
                                                        const std::vector<std::vector<Vector>>& grids,
                                                        InterferenceScope scope) {
    const auto t0 = std::chrono::steady_clock::now();
    const int links = static_cast<int>(factors.cores.size());
    for (const auto& g : grids)
        if (static_cast<int>(g.size()) != links)
            throw std::invalid_argument("assemble_all_compressed: coefficient grid does not match cores");
    std::vector<Cplx> C, G;
    int P = 0;
    pack_compressed(factors, C, G, P);
    const std::size_t F = grids.size();
    std::vector<Cplx> co(F * links * P);
    for (std::size_t f = 0; f < F; ++f)
        for (int l = 0; l < links; ++l) {
            if (grids[f][l].size() != P)
                throw std::invalid_argument("assemble_channel_compressed: delay factor has " + std::to_string(P) +
                                            " rows but coefficient length is " + std::to_string(grids[f][l].size()));
            std::copy(grids[f][l].data(), grids[f][l].data() + P, co.begin() + (f * links + l) * P);
        }
    gwt_topology t = ctopo(topology);
    t.num_taps = P;
    gwt_ranks r{factors.ranks.m, factors.ranks.n, factors.ranks.p};
    const int users = topology.num_users(), L = topology.num_streams;
    std::vector<double> sinr(F * users * L), sig(F * users * L);
    std::vector<int32_t> st(F * users);
    gwt_ledger led{};
    check(gwt_sinr_compressed_coeffs(ctx(), &t, &r, 1, GWT_C128, GWT_MEM_HOST, C.data(), G.data(), co.data(),
                                     static_cast<int64_t>(F),
                                     scope == InterferenceScope::full ? GWT_SCOPE_FULL : GWT_SCOPE_PAPER, sinr.data(),
                                     sig.data(), st.data(), &led));
    for (std::size_t i = 0; i < st.size(); ++i) {  // first failure in reference order (grid, then i, then j)
        bool runtime = false;
        const std::string msg = item_error(st[i], runtime);
        if (!msg.empty()) {
            if (runtime) throw std::runtime_error(msg);
            throw std::invalid_argument(msg);
        }
    }
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::vector<SinrReport> out(F);
    for (std::size_t f = 0; f < F; ++f) {
        SinrReport& rep = out[f];
        rep.num_cells = topology.num_cells;
        rep.users_per_cell = topology.users_per_cell;
        rep.num_streams = L;
        rep.sinr.assign(sinr.begin() + f * users * L, sinr.begin() + (f + 1) * users * L);
        rep.signal_power.assign(sig.begin() + f * users * L, sig.begin() + (f + 1) * users * L);
        rep.ledger = FlopLedger{led.reconstruct / static_cast<std::int64_t>(F), led.precoder / static_cast<std::int64_t>(F),
                                led.covariance / static_cast<std::int64_t>(F), led.inverse / static_cast<std::int64_t>(F),
                                led.filter / static_cast<std::int64_t>(F), led.sinr / static_cast<std::int64_t>(F)};
        rep.seconds = secs / static_cast<double>(F);
    }
    return out;
}

SinrReport run_compressed_pipeline(const SystemTopology& topology, const GroupwiseFactorSet& factors,
                                   const std::vector<Vector>& coeffs, InterferenceScope scope) {
    if (coeffs.size() != factors.cores.size())
        throw std::invalid_argument("assemble_all_compressed: coefficient grid does not match cores");
    return run_compressed_pipeline_batched(topology, factors, {coeffs}, scope).front();
}

SinrReport run_full_pipeline(const ChannelSet& channels, InterferenceScope scope) {
    const auto t0 = std::chrono::steady_clock::now();
    const SystemTopology& topology = channels.topology;
    check_channel_dims(channels);
    const int links = topology.num_links(), M = topology.rx_antennas, N = topology.tx_antennas,
              P = topology.num_taps;
    if (static_cast<int>(channels.coeffs.size()) != links)
        throw std::invalid_argument("assemble_all_full: coefficient count does not match links");
    std::vector<Cplx> X(static_cast<std::size_t>(links) * M * N * P), co(static_cast<std::size_t>(links) * P);
    for (int l = 0; l < links; ++l) {
        std::copy(channels.tensors[l].data(), channels.tensors[l].data() + static_cast<std::size_t>(M) * N * P,
                  X.begin() + static_cast<std::size_t>(l) * M * N * P);
        if (channels.coeffs[l].size() != P)
            throw std::invalid_argument("assemble_channel_full: coefficient length " +
                                        std::to_string(channels.coeffs[l].size()) + " does not match mode-3 size " +
                                        std::to_string(P));
        std::copy(channels.coeffs[l].data(), channels.coeffs[l].data() + P, co.begin() + static_cast<std::size_t>(l) * P);
    }
    gwt_topology t = ctopo(topology);
    const int users = topology.num_users(), L = topology.num_streams;
    std::vector<double> sinr(static_cast<std::size_t>(users) * L), sig(static_cast<std::size_t>(users) * L);
    std::vector<int32_t> st(static_cast<std::size_t>(users));
    gwt_ledger led{};
    check(gwt_sinr_full(ctx(), &t, 1, GWT_C128, GWT_MEM_HOST, X.data(), nullptr, nullptr, co.data(), 1,
                        scope == InterferenceScope::full ? GWT_SCOPE_FULL : GWT_SCOPE_PAPER, sinr.data(), sig.data(),
                        st.data(), &led));
    for (std::size_t i = 0; i < st.size(); ++i) {
        bool runtime = false;
        const std::string msg = item_error(st[i], runtime);
        if (!msg.empty()) {
            if (runtime) throw std::runtime_error(msg);
            throw std::invalid_argument(msg);
        }
    }
    SinrReport rep;
    rep.num_cells = topology.num_cells;
    rep.users_per_cell = topology.users_per_cell;
    rep.num_streams = L;
    rep.sinr = std::move(sinr);
    rep.signal_power = std::move(sig);
    rep.ledger = FlopLedger{led.reconstruct, led.precoder, led.covariance, led.inverse, led.filter, led.sinr};
    rep.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return rep;
}

FlopLedger flop_estimate(const SystemTopology& topology, const CompressionRanks& ranks, PipelinePath path) {
    topology.validate();
    ranks.validate_against(topology.rx_antennas, topology.tx_antennas, topology.num_taps);
    gwt_topology t = ctopo(topology);
    gwt_ranks r{ranks.m, ranks.n, ranks.p};
    gwt_ledger l{};
    if (gwt_flop_estimate(&t, &r, path == PipelinePath::full ? 0 : 1, &l) != GWT_OK)
        throw std::invalid_argument("flop_estimate: invalid topology or ranks");
    return FlopLedger{l.reconstruct, l.precoder, l.covariance, l.inverse, l.filter, l.sinr};
}

}  // namespace gwt
