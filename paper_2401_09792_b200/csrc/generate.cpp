// Seeded synthetic channel sets of BASELINE.json. Input
// synthesis for benches and tests; not part of the measured hot path.
//
// Per link (group g, base k, cell i, user j) a portable RNG stream is derived
// with the reference's seed mixer (proj/src/channel.cpp:13-58: mix64,
// link_seed, mt19937_64 + hand-rolled uniform/Box-Muller so streams are
// platform-independent), with the group folded into the master seed. For each
// tap q: theta, phi ~ U(-pi/3, pi/3); a_q = sqrt(p_q) * CN(0,1);
// p_q = exp(-decay*q) / sum; tau_q ~ U(0, max_delay);
// X(:,:,q) = a_q * a_r(theta) a_t(phi)^H with ULA half-wavelength steering
// e^{j pi q' sin(angle)} (channel.cpp:60-66).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

#include "../../include/gwt_b200.h"

namespace {

std::uint64_t mix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

struct Stream {
    std::mt19937_64 eng;
    bool have = false;
    double spare = 0.0;
    explicit Stream(std::uint64_t s) : eng(s) {}
    double u01() { return (static_cast<double>(eng() >> 11) + 0.5) * 0x1.0p-53; }
    double gauss() {
        if (have) {
            have = false;
            return spare;
        }
        const double u1 = u01(), u2 = u01();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 2.0 * M_PI * u2;
        spare = r * std::sin(a);
        have = true;
        return r * std::cos(a);
    }
};

constexpr std::uint64_t kGroupTag = 0x67726f7570ULL;  // "group"

}  // namespace

extern "C" int gwt_generate_channels(const gwt_topology* topo, int64_t group0, int64_t ngroups, uint64_t seed,
                                     double pdp_decay, double max_delay, gwt_dtype dtype, void* X, double* tau,
                                     int32_t nthreads) {
    if (!topo || ngroups < 0 || !(max_delay >= 0.0)) return GWT_INVALID_ARGUMENT;
    const int J = topo->num_cells, K = topo->users_per_cell, M = topo->rx_antennas, N = topo->tx_antennas,
              P = topo->num_taps;
    if (J < 1 || K < 1 || M < 1 || N < 1 || P < 1) return GWT_INVALID_ARGUMENT;
    const int links = J * J * K;
    const std::size_t tsz = static_cast<std::size_t>(M) * N * P;
    std::vector<double> pdp(P);
    double tot = 0.0;
    for (int q = 0; q < P; ++q) tot += (pdp[q] = std::exp(-pdp_decay * q));
    for (auto& v : pdp) v /= tot;
    auto one_link = [&](int64_t gl) {
        const int64_t g = gl / links;
        const int l = static_cast<int>(gl % links);
        const int k = l / (J * K), i = (l / K) % J, j = l % K;
        std::uint64_t s = mix64(seed ^ mix64(kGroupTag + static_cast<std::uint64_t>(group0 + g) + 1));
        s = mix64(s ^ (static_cast<std::uint64_t>(k) + 1));
        s = mix64(s ^ (static_cast<std::uint64_t>(i) + 1));
        s = mix64(s ^ (static_cast<std::uint64_t>(j) + 1));
        Stream rng(s);
        std::vector<std::complex<double>> ar(M), at(N);
        for (int q = 0; q < P; ++q) {
            const double theta = (rng.u01() * 2.0 - 1.0) * (M_PI / 3.0);
            const double phi = (rng.u01() * 2.0 - 1.0) * (M_PI / 3.0);
            const double re = rng.gauss(), im = rng.gauss();
            const std::complex<double> a = std::complex<double>(re, im) * (std::sqrt(pdp[q]) * M_SQRT1_2);
            const double d = rng.u01() * max_delay;
            tau[gl * P + q] = d;
            const double st = M_PI * std::sin(theta), sp = M_PI * std::sin(phi);
            for (int x = 0; x < M; ++x) ar[x] = std::polar(1.0, st * x);
            for (int y = 0; y < N; ++y) at[y] = std::polar(1.0, -sp * y);  // conj(a_t)
            for (int y = 0; y < N; ++y) {
                const std::complex<double> ay = a * at[y];
                for (int x = 0; x < M; ++x) {
                    const std::complex<double> v = ar[x] * ay;
                    const std::size_t at_idx = static_cast<std::size_t>(gl) * tsz + x + static_cast<std::size_t>(M) * (y + static_cast<std::size_t>(N) * q);
                    if (dtype == GWT_C64) {
                        float* p = static_cast<float*>(X) + 2 * at_idx;
                        p[0] = static_cast<float>(v.real());
                        p[1] = static_cast<float>(v.imag());
                    } else {
                        double* p = static_cast<double*>(X) + 2 * at_idx;
                        p[0] = v.real();
                        p[1] = v.imag();
                    }
                }
            }
        }
    };
    const int64_t total = ngroups * links;
    const int nt = std::max(1, std::min<int>(nthreads, static_cast<int>(std::min<int64_t>(total, 256))));
    std::atomic<int64_t> next{0};
    auto worker = [&] {
        for (;;) {
            const int64_t gl = next.fetch_add(1);
            if (gl >= total) break;
            one_link(gl);
        }
    };
    if (nt == 1) {
        worker();
    } else {
        std::vector<std::thread> th;
        for (int i = 0; i < nt; ++i) th.emplace_back(worker);
        for (auto& t : th) t.join();
    }
    return GWT_OK;
}
