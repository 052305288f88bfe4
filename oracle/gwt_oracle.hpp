// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Eigen-free CPU restatement of the reference library `gwtucker`
// (/root/reference/proj/src/{tensor,linalg,channel,decompose,sinr}.cpp) in
// complex<double>. It exists to CHECK the B200 product path and to be timed as
// the CPU baseline; only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load it. The product
// (paper_2401_09792_b200/) never links or calls it.
//
// Parity pinning (round 2): against the REFERENCE ITSELF. oracle/_ref/libgwtref.so
// is the reference's own proj/src/{tensor,linalg,channel,decompose,sinr,archive,
// metrics}.cpp compiled unchanged from /root/reference against an in-repo
// Eigen-subset shim (oracle/eigen_shim, recipe oracle/Makefile `ref`);
// tests/test_ref.py holds this restatement to it on the reference generator's desk
// systems and BASELINE C1: solver traces within 1e-12 of the energy with equal
// iteration counts, factor subspaces within 1e-8, compressed-pipeline SINR within
// 1e-12 and full-pipeline SINR within 1e-10, equal flop ledgers, identical
// archive bytes. Also (a) the reference's own known-answer tests and identities,
// restated in tests/test_oracle.py, and (b) LAPACK (numpy/scipy) cross-checks of
// the dense kernels, with golden fixtures under tests/golden/.
#pragma once

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

using Cplx = std::complex<double>;

// Column-major dense complex matrix (the subset of Eigen::MatrixXcd the
// reference uses).
struct Mat {
    int r = 0, c = 0;
    std::vector<Cplx> a;
    Mat() = default;
    Mat(int rows, int cols) : r(rows), c(cols), a(static_cast<std::size_t>(rows) * cols, Cplx(0, 0)) {}
    Cplx& operator()(int i, int j) { return a[static_cast<std::size_t>(i) + static_cast<std::size_t>(r) * j]; }
    const Cplx& operator()(int i, int j) const { return a[static_cast<std::size_t>(i) + static_cast<std::size_t>(r) * j]; }
    static Mat identity(int n) {
        Mat m(n, n);
        for (int i = 0; i < n; ++i) m(i, i) = 1.0;
        return m;
    }
};

Mat operator*(const Mat& x, const Mat& y);
Mat adjoint(const Mat& x);
Mat transpose(const Mat& x);
double sq_norm(const Mat& x);

// Tensor3, mode-1-fastest: (i1,i2,i3) at i1 + d1*(i2 + d2*i3)
// (reference proj/include/gwtucker/tensor.hpp:15-39).
struct Tensor3 {
    int d1 = 0, d2 = 0, d3 = 0;
    std::vector<Cplx> a;
    Tensor3() = default;
    Tensor3(int x, int y, int z);
    Cplx& operator()(int i, int j, int k) { return a[i + static_cast<std::size_t>(d1) * (j + static_cast<std::size_t>(d2) * k)]; }
    const Cplx& operator()(int i, int j, int k) const { return a[i + static_cast<std::size_t>(d1) * (j + static_cast<std::size_t>(d2) * k)]; }
    int dim(int mode) const;
};

Mat matricize(const Tensor3& x, int mode);                         // tensor.cpp:36-60
Tensor3 dematricize(const Mat& m, int mode, int d1, int d2, int d3);  // tensor.cpp:62-93
Tensor3 mode_product(const Tensor3& x, const Mat& u, int mode);    // tensor.cpp:95-114
Mat contract_mode3(const Tensor3& x, const std::vector<Cplx>& c);  // tensor.cpp:116-124
double squared_norm(const Tensor3& x);                             // tensor.cpp:137-143

// linalg.cpp
void phase_normalize_columns(Mat& u);                 // linalg.cpp:11-25
struct Eig { std::vector<double> values; Mat vectors; };  // ascending, like Eigen
Eig hermitian_eig(const Mat& h);                      // Householder + implicit QL
Mat leading_eigenvectors(const Mat& h, int count);    // linalg.cpp:27-45
struct Svd { Mat u; std::vector<double> s; Mat v; };
Svd truncated_svd(const Mat& a, int count);           // linalg.cpp:47-79
bool llt(const Mat& q, Mat& l);                       // lower Cholesky; false if not PD

struct Topology {
    int J = 0, K = 0, M = 0, N = 0, P = 0, L = 0;
    double sigma = 0.1;
    int users() const { return J * K; }
    int links() const { return J * J * K; }
    int link(int k, int i, int j) const { return (k * J + i) * K + j; }
    void validate() const;  // channel.cpp:13-27 (SystemTopology::validate)
};
enum Scope { kScopeFull = 0, kScopePaper = 1 };

struct Ranks { int m = 0, n = 0, p = 0; void validate_against(int d1, int d2, int d3) const; };

struct FactorSet {   // decompose.hpp:48-68
    int J = 0, K = 0;
    Ranks ranks;
    std::vector<Mat> rx, tx, delay;
    std::vector<Tensor3> cores;
};
struct Trace { std::vector<double> objective; int iterations_run = 0; };

struct Ledger { std::int64_t reconstruct = 0, precoder = 0, covariance = 0, inverse = 0, filter = 0, sinr = 0; };

// decompose.cpp
FactorSet initial_factors(const Topology& t, const std::vector<Tensor3>& xs, const Ranks& r, bool pooled);
Trace alternating_solve(const Topology& t, const std::vector<Tensor3>& xs, const Ranks& r, int sweeps,
                        const FactorSet* init, bool pooled, bool early_stop, FactorSet& out);
double objective_value(const Topology& t, const std::vector<Tensor3>& xs, const FactorSet& fs);
double projection_energy(const Topology& t, const std::vector<Tensor3>& xs, const FactorSet& fs);
Tensor3 project_core(const Tensor3& x, const Mat& rx, const Mat& tx, const Mat& delay);
Tensor3 reconstruct(const Tensor3& core, const Mat& rx, const Mat& tx, const Mat& delay);
Mat rx_update_gram(const Topology& t, const std::vector<Tensor3>& xs, const FactorSet& fs, int i, int j);
Mat tx_update_gram(const Topology& t, const std::vector<Tensor3>& xs, const FactorSet& fs, int k);
Mat delay_update_gram(const Topology& t, const std::vector<Tensor3>& xs, const FactorSet& fs, int k, int i, int j);
struct Hosvd { Mat rx, tx, delay; Tensor3 core; };
Hosvd hosvd(const Tensor3& x, const Ranks& r);
Trace hooi(const Tensor3& x, const Ranks& r, int sweeps, const Hosvd* init, Hosvd& out);

// sinr.cpp (per-user outputs user-major, stream inner)
struct SinrOut { std::vector<double> sinr, signal; Ledger ledger; };
SinrOut run_compressed_pipeline(const Topology& t, const FactorSet& fs,
                                const std::vector<std::vector<Cplx>>& coeffs, Scope scope);
SinrOut run_full_pipeline(const Topology& t, const std::vector<Tensor3>& xs,
                          const std::vector<std::vector<Cplx>>& coeffs, Scope scope);
SinrOut evaluate_assembled(const Topology& t, const std::vector<Mat>& h, Scope scope, Ledger initial);
std::vector<std::pair<int, int>> scope_pairs(const Topology& t, Scope scope, int i, int j);
Mat assemble_channel_compressed(const Tensor3& core, const Mat& delay, const std::vector<Cplx>& c, Ledger* l);

// reference generator (channel.cpp:13-180), restated for the reference's own test cases
struct GenParams { int rays = 4; double tap_decay = 0.7, rician = 10.0, coeff_decay = 0.8; };
void generate_reference_set(const Topology& t, const GenParams& gp, std::uint64_t seed,
                            std::vector<Tensor3>& xs, std::vector<std::vector<Cplx>>& coeffs);

}  // namespace orc
