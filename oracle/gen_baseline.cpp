// ORACLE — TEST INFRASTRUCTURE ONLY. The BASELINE.json channel generator
// restated on the oracle's side, so that bench.py's CPU
// reference arm and the tests produce their inputs without loading the product
// library. Built with -ffp-contract=off: the values must be bit-identical to
// the product's generator (tests/test_oracle.py::test_baseline_generator_bit_identical).
//
// Per link (group g, base k, cell i, user j) one portable RNG stream: the
// reference's mix64 / link_seed / LinkRng (proj/src/channel.cpp:13-58) with the
// group folded into the master seed. Per tap q, in draw order: theta, phi ~
// U(-pi/3, pi/3); a_q = sqrt(p_q) * CN(0,1) (Box-Muller pair, channel.cpp:98-102);
// tau_q ~ U(0, max_delay); p_q = exp(-decay q) / sum. X(:,:,q) = a_q a_r(theta)
// a_t(phi)^H with the ULA steering of channel.cpp:60-66.
#include <cmath>
#include <complex>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

namespace {

using Cplx = std::complex<double>;

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
        if (have_) {
            have_ = false;
            return spare_;
        }
        const double u1 = uniform01(), u2 = uniform01();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 2.0 * M_PI * u2;
        spare_ = r * std::sin(a);
        have_ = true;
        return r * std::cos(a);
    }

private:
    std::mt19937_64 eng_;
    bool have_ = false;
    double spare_ = 0.0;
};

constexpr std::uint64_t kGroupTag = 0x67726f7570ULL;  // "group"

}  // namespace

// X: [ngroups][links][P][N][M] interleaved (binary64 when c64 == 0, binary32 otherwise); tau [ngroups][links][P].
extern "C" int orc_generate_baseline(int J, int K, int M, int N, int P, long long group0, long long ngroups,
                                     unsigned long long seed, double pdp_decay, double max_delay, int c64, void* X,
                                     double* tau, int nthreads) {
    if (J < 1 || K < 1 || M < 1 || N < 1 || P < 1 || ngroups < 0 || !(max_delay >= 0.0)) return 1;
    const int links = J * J * K;
    std::vector<double> pdp(P);
    double tot = 0.0;
    for (int q = 0; q < P; ++q) tot += (pdp[q] = std::exp(-pdp_decay * q));
    for (auto& v : pdp) v /= tot;
    const std::size_t tsz = static_cast<std::size_t>(M) * N * P;
    auto link = [&](long long gl) {
        const long long g = gl / links;
        const int l = static_cast<int>(gl % links);
        const int k = l / (J * K), i = (l / K) % J, j = l % K;  // link = (k J + i) K + j (channel.hpp:53-56)
        const std::uint64_t master = mix64(seed ^ mix64(kGroupTag + static_cast<std::uint64_t>(group0 + g) + 1));
        LinkRng rng(link_seed(master, k, i, j));
        std::vector<Cplx> ar(M), atc(N);
        for (int q = 0; q < P; ++q) {
            const double theta = (rng.uniform01() * 2.0 - 1.0) * (M_PI / 3.0);
            const double phi = (rng.uniform01() * 2.0 - 1.0) * (M_PI / 3.0);
            const double re = rng.gaussian(), im = rng.gaussian();
            const Cplx a = Cplx(re, im) * (std::sqrt(pdp[q]) * M_SQRT1_2);
            tau[gl * P + q] = rng.uniform01() * max_delay;
            const double sr = M_PI * std::sin(theta), st = M_PI * std::sin(phi);
            for (int x = 0; x < M; ++x) ar[x] = std::polar(1.0, sr * x);
            for (int y = 0; y < N; ++y) atc[y] = std::polar(1.0, -st * y);  // conj of the tx steering entry
            for (int y = 0; y < N; ++y) {
                const Cplx ay = a * atc[y];
                for (int x = 0; x < M; ++x) {
                    const Cplx v = ar[x] * ay;
                    const std::size_t e = static_cast<std::size_t>(gl) * tsz + x + static_cast<std::size_t>(M) * (y + static_cast<std::size_t>(N) * q);
                    if (c64) {
                        static_cast<float*>(X)[2 * e] = static_cast<float>(v.real());
                        static_cast<float*>(X)[2 * e + 1] = static_cast<float>(v.imag());
                    } else {
                        static_cast<double*>(X)[2 * e] = v.real();
                        static_cast<double*>(X)[2 * e + 1] = v.imag();
                    }
                }
            }
        }
    };
    const long long total = ngroups * links;
    const int nt = std::max(1, std::min<int>(nthreads, static_cast<int>(std::min<long long>(total, 256))));
    std::vector<std::thread> th;
    for (int w = 0; w < nt; ++w)
        th.emplace_back([&, w] {
            for (long long gl = w; gl < total; gl += nt) link(gl);
        });
    for (auto& t : th) t.join();
    return 0;
}
