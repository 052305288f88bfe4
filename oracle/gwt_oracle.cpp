// ORACLE — TEST INFRASTRUCTURE ONLY. See gwt_oracle.hpp for the contract.
// Every function cites the reference file:line it restates
// (paths relative to /root/reference/proj).
#include "gwt_oracle.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <numbers>
#include <numeric>
#include <random>

namespace orc {

// ---------------------------------------------------------------------------
// dense helpers

Mat operator*(const Mat& x, const Mat& y) {
    if (x.c != y.r) throw std::invalid_argument("oracle: matmul shape mismatch");
    Mat z(x.r, y.c);
    for (int j = 0; j < y.c; ++j)
        for (int k = 0; k < x.c; ++k) {
            const Cplx b = y(k, j);
            if (b == Cplx(0, 0)) continue;
            const Cplx* xa = &x.a[static_cast<std::size_t>(x.r) * k];
            Cplx* za = &z.a[static_cast<std::size_t>(z.r) * j];
            for (int i = 0; i < x.r; ++i) za[i] += xa[i] * b;
        }
    return z;
}

Mat adjoint(const Mat& x) {
    Mat y(x.c, x.r);
    for (int j = 0; j < x.c; ++j)
        for (int i = 0; i < x.r; ++i) y(j, i) = std::conj(x(i, j));
    return y;
}

Mat transpose(const Mat& x) {
    Mat y(x.c, x.r);
    for (int j = 0; j < x.c; ++j)
        for (int i = 0; i < x.r; ++i) y(j, i) = x(i, j);
    return y;
}

double sq_norm(const Mat& x) {
    double s = 0;
    for (const Cplx& v : x.a) s += std::norm(v);
    return s;
}

static bool all_finite(const Mat& m) {
    for (const Cplx& v : m.a)
        if (!std::isfinite(v.real()) || !std::isfinite(v.imag())) return false;
    return true;
}

// ---------------------------------------------------------------------------
// tensor.cpp

Tensor3::Tensor3(int x, int y, int z) : d1(x), d2(y), d3(z) {
    if (x <= 0 || y <= 0 || z <= 0)  // tensor.cpp:8-13
        throw std::invalid_argument("Tensor3: dims must be positive, got (" + std::to_string(x) + "," +
                                    std::to_string(y) + "," + std::to_string(z) + ")");
    a.assign(static_cast<std::size_t>(x) * y * z, Cplx(0, 0));
}

int Tensor3::dim(int mode) const {  // tensor.cpp:15-22
    switch (mode) {
        case 1: return d1;
        case 2: return d2;
        case 3: return d3;
        default: throw std::invalid_argument("Tensor3::dim: mode must be 1, 2 or 3, got " + std::to_string(mode));
    }
}

Mat matricize(const Tensor3& x, int mode) {  // tensor.cpp:36-60
    const int d1 = x.d1, d2 = x.d2, d3 = x.d3;
    if (mode == 1) {
        Mat m(d1, d2 * d3);
        m.a = x.a;
        return m;
    }
    if (mode == 2) {
        Mat m(d2, d1 * d3);
        for (int i3 = 0; i3 < d3; ++i3)
            for (int i2 = 0; i2 < d2; ++i2)
                for (int i1 = 0; i1 < d1; ++i1) m(i2, i1 + d1 * i3) = x(i1, i2, i3);
        return m;
    }
    if (mode == 3) {
        Mat m(d3, d1 * d2);
        for (int i3 = 0; i3 < d3; ++i3)
            for (int i2 = 0; i2 < d2; ++i2)
                for (int i1 = 0; i1 < d1; ++i1) m(i3, i1 + d1 * i2) = x(i1, i2, i3);
        return m;
    }
    throw std::invalid_argument("matricize: mode must be 1, 2 or 3, got " + std::to_string(mode));
}

Tensor3 dematricize(const Mat& m, int mode, int d1, int d2, int d3) {  // tensor.cpp:62-93
    Tensor3 x(d1, d2, d3);
    if (mode == 1) {
        if (m.r != d1 || m.c != d2 * d3) throw std::invalid_argument("dematricize: matrix shape does not match mode-1 dims");
        x.a = m.a;
        return x;
    }
    if (mode == 2) {
        if (m.r != d2 || m.c != d1 * d3) throw std::invalid_argument("dematricize: matrix shape does not match mode-2 dims");
        for (int i3 = 0; i3 < d3; ++i3)
            for (int i2 = 0; i2 < d2; ++i2)
                for (int i1 = 0; i1 < d1; ++i1) x(i1, i2, i3) = m(i2, i1 + d1 * i3);
        return x;
    }
    if (mode == 3) {
        if (m.r != d3 || m.c != d1 * d2) throw std::invalid_argument("dematricize: matrix shape does not match mode-3 dims");
        for (int i3 = 0; i3 < d3; ++i3)
            for (int i2 = 0; i2 < d2; ++i2)
                for (int i1 = 0; i1 < d1; ++i1) x(i1, i2, i3) = m(i3, i1 + d1 * i2);
        return x;
    }
    throw std::invalid_argument("dematricize: mode must be 1, 2 or 3, got " + std::to_string(mode));
}

Tensor3 mode_product(const Tensor3& x, const Mat& u, int mode) {  // tensor.cpp:95-114
    if (mode < 1 || mode > 3)
        throw std::invalid_argument("mode_product: mode must be 1, 2 or 3, got " + std::to_string(mode));
    if (u.c != x.dim(mode))
        throw std::invalid_argument("mode_product: matrix has " + std::to_string(u.c) + " cols but tensor mode " +
                                    std::to_string(mode) + " has size " + std::to_string(x.dim(mode)));
    int o1 = x.d1, o2 = x.d2, o3 = x.d3;
    (mode == 1 ? o1 : mode == 2 ? o2 : o3) = u.r;
    Tensor3 y(o1, o2, o3);
    // Direct index form of U * X_(mode) (same sums as the reference's GEMM on
    // the unfolding, without the explicit copies).
    if (mode == 1) {
        for (int i3 = 0; i3 < x.d3; ++i3)
            for (int i2 = 0; i2 < x.d2; ++i2)
                for (int k = 0; k < x.d1; ++k) {
                    const Cplx v = x(k, i2, i3);
                    for (int r = 0; r < u.r; ++r) y(r, i2, i3) += u(r, k) * v;
                }
    } else if (mode == 2) {
        for (int i3 = 0; i3 < x.d3; ++i3)
            for (int k = 0; k < x.d2; ++k)
                for (int r = 0; r < u.r; ++r) {
                    const Cplx w = u(r, k);
                    for (int i1 = 0; i1 < x.d1; ++i1) y(i1, r, i3) += w * x(i1, k, i3);
                }
    } else {
        for (int k = 0; k < x.d3; ++k)
            for (int r = 0; r < u.r; ++r) {
                const Cplx w = u(r, k);
                const Cplx* xs = &x.a[static_cast<std::size_t>(x.d1) * x.d2 * k];
                Cplx* ys = &y.a[static_cast<std::size_t>(y.d1) * y.d2 * r];
                for (std::size_t e = 0; e < static_cast<std::size_t>(x.d1) * x.d2; ++e) ys[e] += w * xs[e];
            }
    }
    return y;
}

Mat contract_mode3(const Tensor3& x, const std::vector<Cplx>& c) {  // tensor.cpp:116-124
    if (static_cast<int>(c.size()) != x.d3)
        throw std::invalid_argument("contract_mode3: coefficient length " + std::to_string(c.size()) +
                                    " does not match mode-3 size " + std::to_string(x.d3));
    Mat h(x.d1, x.d2);
    for (int i3 = 0; i3 < x.d3; ++i3) {
        const Cplx w = std::conj(c[i3]);
        for (int i2 = 0; i2 < x.d2; ++i2)
            for (int i1 = 0; i1 < x.d1; ++i1) h(i1, i2) += w * x(i1, i2, i3);
    }
    return h;
}

double squared_norm(const Tensor3& x) {  // tensor.cpp:137-143
    double s = 0;
    for (const Cplx& v : x.a) s += std::norm(v);
    return s;
}

// ---------------------------------------------------------------------------
// linalg.cpp

void phase_normalize_columns(Mat& u) {  // linalg.cpp:11-25
    for (int c = 0; c < u.c; ++c) {
        int best = 0;
        double best_mag = 0.0;
        for (int r = 0; r < u.r; ++r) {
            const double mag = std::abs(u(r, c));
            if (mag > best_mag) { best_mag = mag; best = r; }
        }
        if (best_mag > 0.0) {
            const Cplx f = std::conj(u(best, c)) / best_mag;
            for (int r = 0; r < u.r; ++r) u(r, c) *= f;
        }
    }
}

// Hermitian eigendecomposition with the algorithm family of Eigen's
// SelfAdjointEigenSolver (called at linalg.cpp:34): Householder reduction to
// Hermitian tridiagonal form, a diagonal phase similarity to a real symmetric
// tridiagonal, then implicit-shift QL with the rotations accumulated into the
// eigenvector matrix. Eigenvalues ascending.
Eig hermitian_eig(const Mat& h) {
    const int n = h.r;
    if (h.r != h.c) throw std::invalid_argument("leading_eigenvectors: matrix is not square");
    Mat a = h;
    // Hermitian part (the reference only ever feeds exact Hermitian Grams).
    for (int j = 0; j < n; ++j) {
        a(j, j) = Cplx(a(j, j).real(), 0.0);
        for (int i = j + 1; i < n; ++i) a(j, i) = std::conj(a(i, j));
    }
    Mat q = Mat::identity(n);
    std::vector<Cplx> v(n), p(n), w(n);
    for (int k = 0; k + 2 < n; ++k) {
        double tail2 = 0;
        for (int i = k + 2; i < n; ++i) tail2 += std::norm(a(i, k));
        if (tail2 == 0.0) continue;  // already tridiagonal in this column
        const double xnorm2 = tail2 + std::norm(a(k + 1, k));
        const double xnorm = std::sqrt(xnorm2);
        const Cplx x0 = a(k + 1, k);
        const Cplx ph = std::abs(x0) > 0 ? x0 / std::abs(x0) : Cplx(1, 0);
        const Cplx alpha = -ph * xnorm;
        const int len = n - k - 1;
        for (int i = 0; i < len; ++i) v[i] = a(k + 1 + i, k);
        v[0] -= alpha;
        double vn2 = 0;
        for (int i = 0; i < len; ++i) vn2 += std::norm(v[i]);
        const double tau = 2.0 / vn2;
        // p = tau * B v, B = trailing block
        for (int i = 0; i < len; ++i) {
            Cplx s = 0;
            for (int jj = 0; jj < len; ++jj) s += a(k + 1 + i, k + 1 + jj) * v[jj];
            p[i] = tau * s;
        }
        Cplx vp = 0;
        for (int i = 0; i < len; ++i) vp += std::conj(v[i]) * p[i];
        const Cplx kk = 0.5 * tau * vp;
        for (int i = 0; i < len; ++i) w[i] = p[i] - kk * v[i];
        for (int jj = 0; jj < len; ++jj)
            for (int i = 0; i < len; ++i)
                a(k + 1 + i, k + 1 + jj) -= v[i] * std::conj(w[jj]) + w[i] * std::conj(v[jj]);
        a(k + 1, k) = alpha;
        a(k, k + 1) = std::conj(alpha);
        for (int i = k + 2; i < n; ++i) { a(i, k) = 0; a(k, i) = 0; }
        // q <- q * H,  H = I - tau v v^H acting on rows/cols k+1..n-1
        for (int r = 0; r < n; ++r) {
            Cplx s = 0;
            for (int i = 0; i < len; ++i) s += q(r, k + 1 + i) * v[i];
            s *= tau;
            for (int i = 0; i < len; ++i) q(r, k + 1 + i) -= s * std::conj(v[i]);
        }
    }
    std::vector<double> d(n), e(n, 0.0);
    for (int i = 0; i < n; ++i) d[i] = a(i, i).real();
    // phase similarity D^H T D with real non-negative sub-diagonal
    std::vector<Cplx> delta(n, Cplx(1, 0));
    for (int i = 0; i + 1 < n; ++i) {
        const Cplx sub = a(i + 1, i);
        const double mag = std::abs(sub);
        e[i] = mag;
        delta[i + 1] = mag > 0 ? delta[i] * sub / mag : delta[i];
    }
    Mat z(n, n);  // z = q * D, then QL rotations applied on the right
    for (int j = 0; j < n; ++j)
        for (int r = 0; r < n; ++r) z(r, j) = q(r, j) * delta[j];
    // implicit-shift QL on (d, e), e[i] = T(i+1, i)
    const double eps = std::numeric_limits<double>::epsilon();
    double f = 0.0, tst1 = 0.0;
    for (int l = 0; l < n; ++l) {
        tst1 = std::max(tst1, std::abs(d[l]) + std::abs(e[l]));
        int m = l;
        while (m < n) {
            if (std::abs(e[m]) <= eps * tst1) break;
            ++m;
        }
        if (m == n) m = n - 1;
        if (m > l) {
            int iter = 0;
            do {
                if (++iter > 300) throw std::runtime_error("leading_eigenvectors: eigendecomposition failed");
                double g = d[l];
                double pp = (d[l + 1] - g) / (2.0 * e[l]);
                double r = std::hypot(pp, 1.0);
                if (pp < 0) r = -r;
                d[l] = e[l] / (pp + r);
                d[l + 1] = e[l] * (pp + r);
                const double dl1 = d[l + 1];
                double hh = g - d[l];
                for (int i = l + 2; i < n; ++i) d[i] -= hh;
                f += hh;
                pp = d[m];
                double c = 1.0, c2 = 1.0, c3 = 1.0, s = 0.0, s2 = 0.0;
                const double el1 = e[l + 1];
                for (int i = m - 1; i >= l; --i) {
                    c3 = c2;
                    c2 = c;
                    s2 = s;
                    g = c * e[i];
                    hh = c * pp;
                    r = std::hypot(pp, e[i]);
                    e[i + 1] = s * r;
                    s = e[i] / r;
                    c = pp / r;
                    pp = c * d[i] - s * g;
                    d[i + 1] = hh + s * (c * g + s * d[i]);
                    for (int k = 0; k < n; ++k) {
                        const Cplx t = z(k, i + 1);
                        z(k, i + 1) = s * z(k, i) + c * t;
                        z(k, i) = c * z(k, i) - s * t;
                    }
                }
                pp = -s * s2 * c3 * el1 * e[l] / dl1;
                e[l] = s * pp;
                d[l] = c * pp;
            } while (std::abs(e[l]) > eps * tst1);
        }
        d[l] += f;
        e[l] = 0.0;
    }
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return d[x] < d[y]; });
    Eig out;
    out.values.resize(n);
    out.vectors = Mat(n, n);
    for (int j = 0; j < n; ++j) {
        out.values[j] = d[order[j]];
        for (int r = 0; r < n; ++r) out.vectors(r, j) = z(r, order[j]);
    }
    return out;
}

Mat leading_eigenvectors(const Mat& h, int count) {  // linalg.cpp:27-45
    if (h.r != h.c) throw std::invalid_argument("leading_eigenvectors: matrix is not square");
    if (count < 1 || count > h.r)
        throw std::invalid_argument("leading_eigenvectors: count " + std::to_string(count) + " out of range for size " +
                                    std::to_string(h.r));
    Eig es = hermitian_eig(h);
    const int n = h.r;
    Mat out(n, count);
    for (int c = 0; c < count; ++c)
        for (int r = 0; r < n; ++r) out(r, c) = es.vectors(r, n - 1 - c);
    phase_normalize_columns(out);
    return out;
}

// One-sided (Hestenes) Jacobi on a tall matrix: t (r x c, r >= c) -> t V has
// orthogonal columns. Returns W = t V and V.
static void hestenes(Mat& w, Mat& v) {
    const int c = w.c, r = w.r;
    v = Mat::identity(c);
    for (int sweep = 0; sweep < 80; ++sweep) {
        bool rotated = false;
        for (int p = 0; p < c; ++p)
            for (int q = p + 1; q < c; ++q) {
                double alpha = 0, beta = 0;
                Cplx gamma = 0;
                for (int i = 0; i < r; ++i) {
                    alpha += std::norm(w(i, p));
                    beta += std::norm(w(i, q));
                    gamma += std::conj(w(i, p)) * w(i, q);
                }
                const double g = std::abs(gamma);
                if (g == 0.0 || g <= 1e-15 * std::sqrt(alpha * beta)) continue;
                rotated = true;
                const Cplx ph = std::conj(gamma / g);  // e^{-i phi}
                const double zeta = (beta - alpha) / (2.0 * g);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double cs = 1.0 / std::sqrt(1.0 + t * t);
                const double sn = cs * t;
                for (int i = 0; i < r; ++i) {
                    const Cplx x = w(i, p), y = ph * w(i, q);
                    w(i, p) = cs * x - sn * y;
                    w(i, q) = sn * x + cs * y;
                }
                for (int i = 0; i < c; ++i) {
                    const Cplx x = v(i, p), y = ph * v(i, q);
                    v(i, p) = cs * x - sn * y;
                    v(i, q) = sn * x + cs * y;
                }
            }
        if (!rotated) break;
    }
}

// Thin SVD with the leading `count` triplets; phase from v mirrored onto u
// (linalg.cpp:47-79). Singular vectors of distinct singular values agree with
// Eigen's JacobiSVD up to the phase that the convention then fixes.
Svd truncated_svd(const Mat& a, int count) {
    const int max_rank = std::min(a.r, a.c);
    if (count < 1 || count > max_rank)
        throw std::invalid_argument("truncated_svd: count " + std::to_string(count) + " out of range for " +
                                    std::to_string(a.r) + "x" + std::to_string(a.c) + " matrix");
    const bool tall = a.r >= a.c;
    Mat w = tall ? a : adjoint(a);
    Mat vv;
    hestenes(w, vv);
    const int k = w.c;
    std::vector<double> s(k);
    for (int j = 0; j < k; ++j) {
        double nn = 0;
        for (int i = 0; i < w.r; ++i) nn += std::norm(w(i, j));
        s[j] = std::sqrt(nn);
    }
    std::vector<int> order(k);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return s[x] > s[y]; });
    // tall: a = W S^-1 * S * V^H -> U = W/s, V = vv.  wide: a^H = U' S V'^H -> U = V' = vv, V = W/s
    Svd out;
    out.s.resize(count);
    const int ur = a.r, vr = a.c;
    out.u = Mat(ur, count);
    out.v = Mat(vr, count);
    for (int c = 0; c < count; ++c) {
        const int j = order[c];
        out.s[c] = s[j];
        Mat& left = tall ? out.u : out.v;  // normalised W columns
        Mat& right = tall ? out.v : out.u; // accumulated rotations
        for (int i = 0; i < w.r; ++i) left(i, c) = s[j] > 0 ? w(i, j) / s[j] : Cplx(i == c ? 1.0 : 0.0, 0.0);
        for (int i = 0; i < vv.r; ++i) right(i, c) = vv(i, j);
    }
    for (int c = 0; c < count; ++c) {  // linalg.cpp:61-77
        int best = 0;
        double best_mag = 0.0;
        for (int r = 0; r < out.v.r; ++r) {
            const double mag = std::abs(out.v(r, c));
            if (mag > best_mag) { best_mag = mag; best = r; }
        }
        if (best_mag > 0.0) {
            const Cplx f = std::conj(out.v(best, c)) / best_mag;
            for (int r = 0; r < out.v.r; ++r) out.v(r, c) *= f;
            for (int r = 0; r < out.u.r; ++r) out.u(r, c) *= f;
        }
    }
    return out;
}

bool llt(const Mat& q, Mat& l) {  // Eigen::LLT (sinr.cpp:122,210), lower factor
    const int n = q.r;
    l = Mat(n, n);
    for (int j = 0; j < n; ++j) {
        double djj = q(j, j).real();
        for (int k = 0; k < j; ++k) djj -= std::norm(l(j, k));
        if (!(djj > 0.0) || !std::isfinite(djj)) return false;
        const double ljj = std::sqrt(djj);
        l(j, j) = ljj;
        for (int i = j + 1; i < n; ++i) {
            Cplx s = q(i, j);
            for (int k = 0; k < j; ++k) s -= l(i, k) * std::conj(l(j, k));
            l(i, j) = s / ljj;
        }
    }
    return true;
}

// Solve (L L^H) X = B
static Mat llt_solve(const Mat& l, const Mat& b) {
    const int n = l.r;
    Mat x = b;
    for (int col = 0; col < b.c; ++col) {
        for (int i = 0; i < n; ++i) {
            Cplx s = x(i, col);
            for (int k = 0; k < i; ++k) s -= l(i, k) * x(k, col);
            x(i, col) = s / l(i, i);
        }
        for (int i = n - 1; i >= 0; --i) {
            Cplx s = x(i, col);
            for (int k = i + 1; k < n; ++k) s -= std::conj(l(k, i)) * x(k, col);
            x(i, col) = s / l(i, i);
        }
    }
    return x;
}

// ---------------------------------------------------------------------------
// channel.cpp

void Topology::validate() const {  // channel.cpp SystemTopology::validate
    if (J < 1) throw std::invalid_argument("topology: num_cells (J) must be >= 1");
    if (K < 1) throw std::invalid_argument("topology: users_per_cell (K) must be >= 1");
    if (M < 1) throw std::invalid_argument("topology: rx_antennas (M) must be >= 1");
    if (N < 1) throw std::invalid_argument("topology: tx_antennas (N) must be >= 1");
    if (P < 1) throw std::invalid_argument("topology: num_taps (P) must be >= 1");
    if (L < 1) throw std::invalid_argument("topology: num_streams (L) must be >= 1");
    if (L > std::min(M, N)) throw std::invalid_argument("topology: num_streams (L) must satisfy L <= min(M, N)");
    if (!(sigma > 0.0)) throw std::invalid_argument("topology: noise_std (sigma) must be > 0");
}

namespace {
std::uint64_t mix64(std::uint64_t x) {  // channel.cpp:13-18
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
std::uint64_t link_seed(std::uint64_t master, int k, int i, int j) {  // channel.cpp:20-26
    std::uint64_t s = master;
    s = mix64(s ^ (static_cast<std::uint64_t>(k) + 1));
    s = mix64(s ^ (static_cast<std::uint64_t>(i) + 1));
    s = mix64(s ^ (static_cast<std::uint64_t>(j) + 1));
    return s;
}
class LinkRng {  // channel.cpp:31-58
public:
    explicit LinkRng(std::uint64_t seed) : eng_(seed) {}
    double uniform01() { return (static_cast<double>(eng_() >> 11) + 0.5) * 0x1.0p-53; }
    double gaussian() {
        if (have_) { have_ = false; return spare_; }
        const double u1 = uniform01(), u2 = uniform01();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 2.0 * std::numbers::pi * u2;
        spare_ = r * std::sin(a);
        have_ = true;
        return r * std::cos(a);
    }
private:
    std::mt19937_64 eng_;
    bool have_ = false;
    double spare_ = 0.0;
};
std::vector<Cplx> steering(int count, double angle) {  // channel.cpp:60-66
    std::vector<Cplx> a(count);
    const double step = std::numbers::pi * std::sin(angle);
    for (int q = 0; q < count; ++q) a[q] = std::polar(1.0, step * q);
    return a;
}
Cplx draw_cn(LinkRng& rng) {  // channel.cpp:98-102
    const double re = rng.gaussian();
    const double im = rng.gaussian();
    return Cplx(re, im) * std::numbers::sqrt2 / 2.0;
}
constexpr double kClusterSpread = 0.25;
double angle_center(std::uint64_t master, std::uint64_t tag, int index) {  // channel.cpp:110-113
    LinkRng rng(mix64(master ^ mix64(tag + static_cast<std::uint64_t>(index) + 1)));
    return (rng.uniform01() - 0.5) * 2.0;
}
}  // namespace

void generate_reference_set(const Topology& t, const GenParams& gp, std::uint64_t seed,
                            std::vector<Tensor3>& xs, std::vector<std::vector<Cplx>>& coeffs) {
    // channel.cpp:115-180
    t.validate();
    xs.clear();
    coeffs.clear();
    constexpr std::uint64_t kUserTag = 0x75736572u, kBaseTag = 0x62617365u;
    for (int k = 0; k < t.J; ++k)
        for (int i = 0; i < t.J; ++i)
            for (int j = 0; j < t.K; ++j) {
                LinkRng rng(link_seed(seed, k, i, j));
                const double rxc = angle_center(seed, kUserTag, i * t.K + j);
                const double txc = angle_center(seed, kBaseTag, k);
                Tensor3 x(t.M, t.N, t.P);
                for (int l = 0; l < t.P; ++l) {
                    const bool los = (l == 0);
                    const int rays = los ? std::min(gp.rays, 2) : gp.rays;
                    Mat slice(t.M, t.N);
                    for (int r = 0; r < rays; ++r) {
                        const double theta = rxc + (rng.uniform01() - 0.5) * 2.0 * kClusterSpread;
                        const double phi = txc + (rng.uniform01() - 0.5) * 2.0 * kClusterSpread;
                        Cplx gain = draw_cn(rng);
                        if (los && r == 0)
                            gain = std::sqrt(gp.rician) * std::polar(1.0, 2.0 * std::numbers::pi * rng.uniform01());
                        const auto ar = steering(t.M, theta), at = steering(t.N, phi);
                        for (int b = 0; b < t.N; ++b)
                            for (int a = 0; a < t.M; ++a) slice(a, b) += gain * (ar[a] * std::conj(at[b]));
                    }
                    const double target = std::pow(gp.tap_decay, l) * t.M * t.N;
                    const double actual = sq_norm(slice);
                    const double sc = actual > 0 ? std::sqrt(target / actual) : 1.0;
                    for (int b = 0; b < t.N; ++b)
                        for (int a = 0; a < t.M; ++a) x(a, b, l) = slice(a, b) * (actual > 0 ? sc : 1.0);
                }
                std::vector<Cplx> c(t.P);
                double nn = 0;
                for (int l = 0; l < t.P; ++l) {
                    c[l] = draw_cn(rng) * std::sqrt(std::pow(gp.coeff_decay, l));
                    nn += std::norm(c[l]);
                }
                const double norm = std::sqrt(nn);
                if (norm > 0.0)
                    for (auto& v : c) v *= std::sqrt(static_cast<double>(t.P)) / norm;
                xs.push_back(std::move(x));
                coeffs.push_back(std::move(c));
            }
}

Mat assemble_channel_compressed(const Tensor3& core, const Mat& delay, const std::vector<Cplx>& c, Ledger* l) {
    // channel.cpp:189-208
    if (delay.r != static_cast<int>(c.size()))
        throw std::invalid_argument("assemble_channel_compressed: delay factor has " + std::to_string(delay.r) +
                                    " rows but coefficient length is " + std::to_string(c.size()));
    if (delay.c != core.d3)
        throw std::invalid_argument("assemble_channel_compressed: delay factor has " + std::to_string(delay.c) +
                                    " cols but core mode-3 size is " + std::to_string(core.d3));
    std::vector<Cplx> d(delay.c, Cplx(0, 0));  // d = C^H c
    for (int q = 0; q < delay.c; ++q)
        for (int r = 0; r < delay.r; ++r) d[q] += std::conj(delay(r, q)) * c[r];
    Mat h = contract_mode3(core, d);
    if (l) l->reconstruct += static_cast<std::int64_t>(core.d1) * core.d2 * core.d3 + static_cast<std::int64_t>(delay.r) * delay.c;
    return h;
}

// ---------------------------------------------------------------------------
// decompose.cpp

void Ranks::validate_against(int d1, int d2, int d3) const {  // decompose.cpp:58-68
    if (m < 1 || m > d1) throw std::invalid_argument("rank m = " + std::to_string(m) + " out of range for mode-1 size " + std::to_string(d1));
    if (n < 1 || n > d2) throw std::invalid_argument("rank n = " + std::to_string(n) + " out of range for mode-2 size " + std::to_string(d2));
    if (p < 1 || p > d3) throw std::invalid_argument("rank p = " + std::to_string(p) + " out of range for mode-3 size " + std::to_string(d3));
}

static Mat gram(const Mat& w) {  // w * w^H
    Mat g(w.r, w.r);
    for (int k = 0; k < w.c; ++k)
        for (int j = 0; j < w.r; ++j) {
            const Cplx b = std::conj(w(j, k));
            for (int i = 0; i < w.r; ++i) g(i, j) += w(i, k) * b;
        }
    return g;
}

static void add_to(Mat& a, const Mat& b) {
    for (std::size_t i = 0; i < a.a.size(); ++i) a.a[i] += b.a[i];
}

Tensor3 project_core(const Tensor3& x, const Mat& rx, const Mat& tx, const Mat& delay) {  // decompose.cpp:23-26
    return mode_product(mode_product(mode_product(x, adjoint(rx), 1), adjoint(tx), 2), adjoint(delay), 3);
}

Tensor3 reconstruct(const Tensor3& core, const Mat& rx, const Mat& tx, const Mat& delay) {  // decompose.cpp:139-141
    return mode_product(mode_product(mode_product(core, rx, 1), tx, 2), delay, 3);
}

static double residual_for(const Tensor3& x, const Mat& rx, const Mat& tx, const Mat& delay) {  // decompose.cpp:31-38
    Tensor3 core = project_core(x, rx, tx, delay);
    Tensor3 xh = reconstruct(core, rx, tx, delay);
    double acc = 0.0;
    for (std::size_t i = 0; i < x.a.size(); ++i) acc += std::norm(x.a[i] - xh.a[i]);
    return acc;
}

Hosvd hosvd(const Tensor3& x, const Ranks& r) {  // decompose.cpp:73-91
    r.validate_against(x.d1, x.d2, x.d3);
    Hosvd f;
    f.rx = leading_eigenvectors(gram(matricize(x, 1)), r.m);
    f.tx = leading_eigenvectors(gram(matricize(x, 2)), r.n);
    f.delay = leading_eigenvectors(gram(matricize(x, 3)), r.p);
    f.core = project_core(x, f.rx, f.tx, f.delay);
    return f;
}

Trace hooi(const Tensor3& x, const Ranks& r, int sweeps, const Hosvd* init, Hosvd& f) {  // decompose.cpp:97-137
    r.validate_against(x.d1, x.d2, x.d3);
    if (sweeps < 0) throw std::invalid_argument("hooi: sweeps must be >= 0");
    f = init ? *init : hosvd(x, r);
    const double energy = squared_norm(x);
    Trace tr;
    tr.objective.push_back(residual_for(x, f.rx, f.tx, f.delay));
    for (int s = 0; s < sweeps; ++s) {
        f.rx = leading_eigenvectors(gram(matricize(mode_product(mode_product(x, adjoint(f.tx), 2), adjoint(f.delay), 3), 1)), r.m);
        f.tx = leading_eigenvectors(gram(matricize(mode_product(mode_product(x, adjoint(f.rx), 1), adjoint(f.delay), 3), 2)), r.n);
        f.delay = leading_eigenvectors(gram(matricize(mode_product(mode_product(x, adjoint(f.rx), 1), adjoint(f.tx), 2), 3)), r.p);
        const double obj = residual_for(x, f.rx, f.tx, f.delay);
        const double dec = tr.objective.back() - obj;
        tr.objective.push_back(obj);
        tr.iterations_run = s + 1;
        if (dec < 1e-10 * energy) break;
    }
    f.core = project_core(x, f.rx, f.tx, f.delay);
    return tr;
}

Mat rx_update_gram(const Topology& t, const std::vector<Tensor3>& xs, const FactorSet& fs, int i, int j) {
    // decompose.cpp:146-157
    Mat g(t.M, t.M);
    for (int k = 0; k < t.J; ++k) {
        const Tensor3& x = xs[t.link(k, i, j)];
        Tensor3 w = mode_product(mode_product(x, adjoint(fs.tx[k]), 2), adjoint(fs.delay[t.link(k, i, j)]), 3);
        add_to(g, gram(matricize(w, 1)));
    }
    return g;
}

Mat tx_update_gram(const Topology& t, const std::vector<Tensor3>& xs, const FactorSet& fs, int k) {
    // decompose.cpp:163-175
    Mat g(t.N, t.N);
    for (int i = 0; i < t.J; ++i)
        for (int j = 0; j < t.K; ++j) {
            const Tensor3& x = xs[t.link(k, i, j)];
            Tensor3 w = mode_product(mode_product(x, adjoint(fs.rx[i * t.K + j]), 1), adjoint(fs.delay[t.link(k, i, j)]), 3);
            add_to(g, gram(matricize(w, 2)));
        }
    return g;
}

Mat delay_update_gram(const Topology& t, const std::vector<Tensor3>& xs, const FactorSet& fs, int k, int i, int j) {
    // decompose.cpp:181-188
    const Tensor3& x = xs[t.link(k, i, j)];
    Tensor3 w = mode_product(mode_product(x, adjoint(fs.rx[i * t.K + j]), 1), adjoint(fs.tx[k]), 2);
    return gram(matricize(w, 3));
}

double objective_value(const Topology& t, const std::vector<Tensor3>& xs, const FactorSet& fs) {  // decompose.cpp:217-226
    double f = 0.0;
    for (int k = 0; k < t.J; ++k)
        for (int i = 0; i < t.J; ++i)
            for (int j = 0; j < t.K; ++j)
                f += residual_for(xs[t.link(k, i, j)], fs.rx[i * t.K + j], fs.tx[k], fs.delay[t.link(k, i, j)]);
    return f;
}

double projection_energy(const Topology& t, const std::vector<Tensor3>& xs, const FactorSet& fs) {  // decompose.cpp:206-215
    double g = 0.0;
    for (int k = 0; k < t.J; ++k)
        for (int i = 0; i < t.J; ++i)
            for (int j = 0; j < t.K; ++j)
                g += squared_norm(project_core(xs[t.link(k, i, j)], fs.rx[i * t.K + j], fs.tx[k], fs.delay[t.link(k, i, j)]));
    return g;
}

FactorSet initial_factors(const Topology& t, const std::vector<Tensor3>& xs, const Ranks& r, bool pooled) {
    // decompose.cpp:248-300
    FactorSet fs;
    fs.J = t.J;
    fs.K = t.K;
    fs.ranks = r;
    fs.rx.resize(t.users());
    fs.tx.resize(t.J);
    fs.delay.resize(t.links());
    if (pooled) {
        Mat g(t.M, t.M);
        for (const Tensor3& x : xs) add_to(g, gram(matricize(x, 1)));
        Mat sh = leading_eigenvectors(g, r.m);
        for (Mat& f : fs.rx) f = sh;
    } else {
        for (int i = 0; i < t.J; ++i)
            for (int j = 0; j < t.K; ++j) {
                Mat g(t.M, t.M);
                for (int k = 0; k < t.J; ++k) add_to(g, gram(matricize(xs[t.link(k, i, j)], 1)));
                fs.rx[i * t.K + j] = leading_eigenvectors(g, r.m);
            }
    }
    if (pooled) {
        Mat g(t.N, t.N);
        for (const Tensor3& x : xs) add_to(g, gram(matricize(x, 2)));
        Mat sh = leading_eigenvectors(g, r.n);
        for (Mat& f : fs.tx) f = sh;
    } else {
        for (int k = 0; k < t.J; ++k) {
            Mat g(t.N, t.N);
            for (int i = 0; i < t.J; ++i)
                for (int j = 0; j < t.K; ++j) add_to(g, gram(matricize(xs[t.link(k, i, j)], 2)));
            fs.tx[k] = leading_eigenvectors(g, r.n);
        }
    }
    for (int l = 0; l < t.links(); ++l) fs.delay[l] = leading_eigenvectors(gram(matricize(xs[l], 3)), r.p);
    return fs;
}

Trace alternating_solve(const Topology& t, const std::vector<Tensor3>& xs, const Ranks& r, int sweeps,
                        const FactorSet* init, bool pooled, bool early_stop, FactorSet& fs) {
    // decompose.cpp:309-373 (check_channel_dims :13-21, check_init_shape :302-307)
    if (static_cast<int>(xs.size()) != t.links())
        throw std::invalid_argument("channel set has " + std::to_string(xs.size()) + " tensors but topology expects " +
                                    std::to_string(t.links()));
    for (const Tensor3& x : xs)
        if (x.d1 != t.M || x.d2 != t.N || x.d3 != t.P) throw std::invalid_argument("channel set: inconsistent tensor dims");
    r.validate_against(t.M, t.N, t.P);
    if (sweeps < 0) throw std::invalid_argument("solve: sweeps must be >= 0");
    if (init && (init->J != t.J || init->K != t.K || init->ranks.m != r.m || init->ranks.n != r.n || init->ranks.p != r.p))
        throw std::invalid_argument("solver init: factor set shape does not match channels/ranks");
    fs = init ? *init : initial_factors(t, xs, r, pooled);
    double energy = 0.0;
    for (const Tensor3& x : xs) energy += squared_norm(x);
    Trace tr;
    tr.objective.push_back(objective_value(t, xs, fs));
    for (int s = 0; s < sweeps; ++s) {
        if (pooled) {
            Mat g(t.M, t.M);
            for (int i = 0; i < t.J; ++i)
                for (int j = 0; j < t.K; ++j) add_to(g, rx_update_gram(t, xs, fs, i, j));
            Mat sh = leading_eigenvectors(g, r.m);
            for (Mat& f : fs.rx) f = sh;
        } else {
            std::vector<Mat> fresh(t.users());
            for (int i = 0; i < t.J; ++i)
                for (int j = 0; j < t.K; ++j) fresh[i * t.K + j] = leading_eigenvectors(rx_update_gram(t, xs, fs, i, j), r.m);
            fs.rx = std::move(fresh);
        }
        if (pooled) {
            Mat g(t.N, t.N);
            for (int k = 0; k < t.J; ++k) add_to(g, tx_update_gram(t, xs, fs, k));
            Mat sh = leading_eigenvectors(g, r.n);
            for (Mat& f : fs.tx) f = sh;
        } else {
            std::vector<Mat> fresh(t.J);
            for (int k = 0; k < t.J; ++k) fresh[k] = leading_eigenvectors(tx_update_gram(t, xs, fs, k), r.n);
            fs.tx = std::move(fresh);
        }
        for (int k = 0; k < t.J; ++k)
            for (int i = 0; i < t.J; ++i)
                for (int j = 0; j < t.K; ++j)
                    fs.delay[t.link(k, i, j)] = leading_eigenvectors(delay_update_gram(t, xs, fs, k, i, j), r.p);
        const double obj = objective_value(t, xs, fs);
        const double dec = tr.objective.back() - obj;
        tr.objective.push_back(obj);
        tr.iterations_run = s + 1;
        if (early_stop && dec < 1e-10 * energy) break;
    }
    fs.cores.resize(t.links());  // compute_cores decompose.cpp:195-204
    for (int k = 0; k < t.J; ++k)
        for (int i = 0; i < t.J; ++i)
            for (int j = 0; j < t.K; ++j)
                fs.cores[t.link(k, i, j)] = project_core(xs[t.link(k, i, j)], fs.rx[i * t.K + j], fs.tx[k], fs.delay[t.link(k, i, j)]);
    return tr;
}

// ---------------------------------------------------------------------------
// sinr.cpp

namespace {
void check_finite(const Mat& m, const char* what) {  // sinr.cpp:23-26
    if (!all_finite(m)) throw std::invalid_argument(std::string(what) + ": non-finite input");
}

void stream_sinrs(const Mat& w, const Mat& q, const Mat& hv, double* sinr, double* sig) {  // sinr.cpp:28-43
    const int streams = w.c;
    for (int r = 0; r < streams; ++r) {
        Cplx amp = 0;
        for (int i = 0; i < w.r; ++i) amp += std::conj(w(i, r)) * hv(i, r);
        const double s = std::norm(amp);
        Cplx wqw = 0;
        for (int i = 0; i < w.r; ++i) {
            Cplx qw = 0;
            for (int k = 0; k < w.r; ++k) qw += q(i, k) * w(k, r);
            wqw += std::conj(w(i, r)) * qw;
        }
        double denom = wqw.real() - s;
        if (denom <= -1e-12)
            throw std::runtime_error("sinr: interference-plus-noise power is negative for stream " + std::to_string(r) +
                                     " (numerically invalid configuration)");
        denom = std::max(denom, std::numeric_limits<double>::min());
        sig[r] = s;
        sinr[r] = s / denom;
    }
}

struct Precoder { Mat v; std::vector<double> s; Mat u; };

Precoder precoder(const Mat& h, int streams, bool compressed, Ledger* l) {  // sinr.cpp:76-85, 162-172
    if (streams > std::min(h.r, h.c)) {
        if (compressed)
            throw std::invalid_argument("precoder: stream count " + std::to_string(streams) + " exceeds compressed channel size " +
                                        std::to_string(h.r) + "x" + std::to_string(h.c) + " (ranks chosen below stream count)");
        throw std::invalid_argument("precoder: stream count " + std::to_string(streams) + " exceeds min dimension of " +
                                    std::to_string(h.r) + "x" + std::to_string(h.c) + " channel");
    }
    Svd s = truncated_svd(h, streams);
    if (l) l->precoder += static_cast<std::int64_t>(h.r) * h.c * streams;
    return {std::move(s.v), std::move(s.s), std::move(s.u)};
}

Mat covariance(const Topology& t, const std::vector<Mat>& h, const std::vector<Precoder>& pre, Scope scope, int i, int j,
               int dim) {  // sinr.cpp:97-114 / 184-203
    Mat q = Mat::identity(dim);
    for (auto& v : q.a) v *= t.sigma * t.sigma;
    for (const auto& [k, l] : scope_pairs(t, scope, i, j)) {
        const std::size_t user = static_cast<std::size_t>(k) * t.K + l;
        if (user >= pre.size()) throw std::invalid_argument("covariance: scope references missing precoder");
        Mat term = h[t.link(k, i, j)] * pre[user].v;
        add_to(q, gram(term));
    }
    return q;
}
}  // namespace

std::vector<std::pair<int, int>> scope_pairs(const Topology& t, Scope scope, int i, int j) {  // sinr.cpp:47-62
    std::vector<std::pair<int, int>> pairs;
    if (scope == kScopeFull) {
        for (int k = 0; k < t.J; ++k)
            for (int l = 0; l < t.K; ++l) pairs.emplace_back(k, l);
        return pairs;
    }
    pairs.emplace_back(i, j);
    for (int k = 0; k < t.J; ++k)
        if (k != i) pairs.emplace_back(k, 0);
    return pairs;
}

SinrOut evaluate_assembled(const Topology& t, const std::vector<Mat>& h, Scope scope, Ledger initial) {
    // sinr.cpp:259-285 (full path: precoder_full, covariance_full, filter_full, sinr_full)
    SinrOut out;
    out.ledger = initial;
    out.sinr.assign(static_cast<std::size_t>(t.users()) * t.L, 0.0);
    out.signal.assign(out.sinr.size(), 0.0);
    std::vector<Precoder> pre;
    for (int i = 0; i < t.J; ++i)
        for (int j = 0; j < t.K; ++j) pre.push_back(precoder(h[t.link(i, i, j)], t.L, false, &out.ledger));
    const std::int64_t M = h[0].r, N = h[0].c, L = t.L;
    for (int i = 0; i < t.J; ++i)
        for (int j = 0; j < t.K; ++j) {
            const Mat& hs = h[t.link(i, i, j)];
            const Precoder& p = pre[i * t.K + j];
            Mat q = covariance(t, h, pre, scope, i, j, hs.r);
            out.ledger.covariance += static_cast<std::int64_t>(t.users()) * (M * N * L + M * M * L);
            check_finite(q, "filter");
            check_finite(hs, "filter");
            check_finite(p.v, "filter");
            Mat hv = hs * p.v;
            Mat l;
            if (!llt(q, l)) throw std::runtime_error("filter: covariance is not positive definite");
            Mat w = llt_solve(l, hv);
            out.ledger.inverse += M * M * M;
            out.ledger.filter += M * M * L;
            out.ledger.sinr += L * (M * M + 2 * M);
            stream_sinrs(w, q, hv, &out.sinr[(i * t.K + j) * t.L], &out.signal[(i * t.K + j) * t.L]);
        }
    return out;
}

SinrOut run_full_pipeline(const Topology& t, const std::vector<Tensor3>& xs,
                          const std::vector<std::vector<Cplx>>& coeffs, Scope scope) {  // sinr.cpp:287-294
    Ledger lg;
    std::vector<Mat> h;
    for (std::size_t l = 0; l < xs.size(); ++l) {
        h.push_back(contract_mode3(xs[l], coeffs[l]));
        lg.reconstruct += static_cast<std::int64_t>(xs[l].d1) * xs[l].d2 * xs[l].d3;
    }
    return evaluate_assembled(t, h, scope, lg);
}

SinrOut run_compressed_pipeline(const Topology& t, const FactorSet& fs,
                                const std::vector<std::vector<Cplx>>& coeffs, Scope scope) {  // sinr.cpp:296-326
    if (coeffs.size() != fs.cores.size())
        throw std::invalid_argument("assemble_all_compressed: coefficient grid does not match cores");
    SinrOut out;
    out.sinr.assign(static_cast<std::size_t>(t.users()) * t.L, 0.0);
    out.signal.assign(out.sinr.size(), 0.0);
    std::vector<Mat> h;
    for (std::size_t l = 0; l < fs.cores.size(); ++l)
        h.push_back(assemble_channel_compressed(fs.cores[l], fs.delay[l], coeffs[l], &out.ledger));
    std::vector<Precoder> pre;
    for (int i = 0; i < t.J; ++i)
        for (int j = 0; j < t.K; ++j) pre.push_back(precoder(h[t.link(i, i, j)], t.L, true, &out.ledger));
    const double sigma = t.sigma;
    const std::int64_t m = fs.ranks.m, n = fs.ranks.n, L = t.L;
    for (int i = 0; i < t.J; ++i)
        for (int j = 0; j < t.K; ++j) {
            const Mat& hs = h[t.link(i, i, j)];
            const Precoder& p = pre[i * t.K + j];
            Mat q = covariance(t, h, pre, scope, i, j, fs.ranks.m);
            out.ledger.covariance += static_cast<std::int64_t>(t.users()) * (m * n * L + m * m * L);
            // woodbury_inverse_apply sinr.cpp:205-227
            if (!(sigma > 0.0)) throw std::invalid_argument("woodbury_inverse_apply: sigma must be > 0");
            check_finite(q, "woodbury_inverse_apply");
            Mat l;
            if (!llt(q, l)) throw std::runtime_error("woodbury_inverse_apply: covariance is numerically singular");
            double dmax = 0, dmin = std::numeric_limits<double>::infinity();
            for (int d = 0; d < l.r; ++d) { dmax = std::max(dmax, l(d, d).real()); dmin = std::min(dmin, l(d, d).real()); }
            const double ratio = dmax / dmin;
            if (ratio * ratio > 1e14)
                throw std::runtime_error("woodbury_inverse_apply: covariance is numerically singular (condition estimate above 1e14)");
            Mat qs = q;
            for (int d = 0; d < qs.r; ++d) qs(d, d) -= sigma * sigma;
            Mat tt = llt_solve(l, qs);
            const double inv_s2 = 1.0 / (sigma * sigma);
            out.ledger.inverse += 2 * m * m * m;
            // filter_compressed sinr.cpp:229-240
            check_finite(hs, "filter_compressed");
            check_finite(p.v, "filter_compressed");
            Mat hv = hs * p.v;
            Mat thv = tt * hv;
            Mat w = hv;
            for (std::size_t e = 0; e < w.a.size(); ++e) w.a[e] = inv_s2 * (hv.a[e] - thv.a[e]);
            out.ledger.filter += m * m * L + m * L;
            out.ledger.sinr += L * (m * m + 2 * m);  // sinr_compressed sinr.cpp:242-254
            stream_sinrs(w, q, hv, &out.sinr[(i * t.K + j) * t.L], &out.signal[(i * t.K + j) * t.L]);
        }
    return out;
}

}  // namespace orc
