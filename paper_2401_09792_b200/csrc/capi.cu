// extern "C" boundary (include/gwt_b200.h) and host-side orchestration of the
// B200 kernels. Validation mirrors the reference's exception texts
// (proj/src/{decompose,sinr,channel}.cpp); no exception crosses the ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gwt_b200.h"
#include "kernels.cuh"

using namespace gwtk;

namespace {

struct GwtError {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw GwtError{code, msg}; }
[[noreturn]] void invalid(const std::string& msg) { fail(GWT_INVALID_ARGUMENT, msg); }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(GWT_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

// Tuning switches, read from the environment ONCE when the context is created (INTEGRATION.md lists them)
struct GwtOptions {
    int64_t ws_bytes = int64_t(16) << 30;  // GWT_WS_BYTES: workspace budget for Tucker intermediates
    int solve_lanes = 4;                   // GWT_SOLVE_LANES
    bool solve_side = true;                // GWT_SOLVE_NO_SIDE unset
    bool poll = true;                      // GWT_NO_POLL unset
    int eig64_min_d = 1 << 30;             // GWT_EIG64_MIN_D
    bool gram_tc = true;                   // GWT_GRAM_TC != 0
    int sinr_path = 0;                     // GWT_SINR_PATH: 0 auto, 1 tc, 2 users, 3 pg
    int64_t sinr_chunk_bytes = int64_t(2) << 30;  // GWT_SINR_CHUNK_BYTES
    int sinr_pipeline = 0;                 // GWT_SINR_PIPELINE: host-path group chunks (0: 8 on the tensor-core path, else 4)
    int sinr_dev_lanes = 0;                // GWT_SINR_DEV_LANES (0: by path)
    int sinr_lanes = 0;                    // GWT_SINR_LANES: host-path compute lanes (0: by path)
    bool sinr_copy_streams = true;         // GWT_SINR_COPY_STREAMS != 0
    bool pg_small = false;                 // GWT_PG_SMALL: m > 4 tensor path -> the 8-lanes Jacobi solver
    void read() {
        auto num = [](const char* k, int64_t& v) { if (const char* e = std::getenv(k)) v = std::strtoll(e, nullptr, 10); };
        auto inum = [](const char* k, int& v) { if (const char* e = std::getenv(k)) v = std::atoi(e); };
        num("GWT_WS_BYTES", ws_bytes);
        inum("GWT_SOLVE_LANES", solve_lanes);
        solve_side = !std::getenv("GWT_SOLVE_NO_SIDE");
        poll = !std::getenv("GWT_NO_POLL");
        inum("GWT_EIG64_MIN_D", eig64_min_d);
        if (const char* e = std::getenv("GWT_GRAM_TC")) gram_tc = std::atoi(e) != 0;
        if (const char* e = std::getenv("GWT_SINR_PATH"))
            sinr_path = !std::strcmp(e, "tc") ? 1 : !std::strcmp(e, "users") ? 2 : !std::strcmp(e, "pg") ? 3 : 0;
        num("GWT_SINR_CHUNK_BYTES", sinr_chunk_bytes);
        inum("GWT_SINR_PIPELINE", sinr_pipeline);
        inum("GWT_SINR_DEV_LANES", sinr_dev_lanes);
        inum("GWT_SINR_LANES", sinr_lanes);
        if (const char* e = std::getenv("GWT_SINR_COPY_STREAMS")) sinr_copy_streams = std::atoi(e) != 0;
        pg_small = std::getenv("GWT_PG_SMALL") != nullptr;
    }
};

struct gwt_ctx {
    int device = 0;
    GwtOptions opt;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    std::string last_error;
    int64_t launches = 0;
    struct Slot {
        void* p = nullptr;
        size_t bytes = 0;
    };
    std::vector<Slot> slots = std::vector<Slot>(40);
    cudaEvent_t ev[16] = {};
    int* pinned[8] = {};  // per solver lane: early-stop count read back without a blocking copy
    // host-buffer SINR pipeline: dedicated copy streams and per-chunk events (sinr_impl)
    cudaStream_t cp_h2d = nullptr, cp_d2h = nullptr;
    std::vector<cudaEvent_t> chev;
    cudaEvent_t chunk_event(size_t i) {
        while (chev.size() <= i) {
            cudaEvent_t e;
            ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
            chev.push_back(e);
        }
        return chev[i];
    }
    void copy_streams() {
        if (!cp_h2d) ck(cudaStreamCreateWithFlags(&cp_h2d, cudaStreamNonBlocking), "cudaStreamCreate");
        if (!cp_d2h) ck(cudaStreamCreateWithFlags(&cp_d2h, cudaStreamNonBlocking), "cudaStreamCreate");
    }
    // per solver lane: side stream + events for the objective tail of a sweep (SolveLane::sweep)
    cudaStream_t side[8] = {};
    cudaEvent_t side_ev[8][4] = {};
    cudaStream_t side_stream(int lane) {
        if (!side[lane]) {
            ck(cudaStreamCreateWithFlags(&side[lane], cudaStreamNonBlocking), "cudaStreamCreate");
            for (auto& e : side_ev[lane]) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        }
        return side[lane];
    }
    int* pin(int lane) {
        if (!pinned[lane]) ck(cudaMallocHost(&pinned[lane], 64), "cudaMallocHost");
        return pinned[lane];
    }
    double stage_ms[8] = {};
    // extra solver lanes (stream + workspace) that run group sub-chunks concurrently with lane 0 (ctx->stream)
    struct Lane {
        cudaStream_t st = nullptr;
        cudaEvent_t ev = nullptr;
        std::vector<Slot> slots = std::vector<Slot>(40);
    };
    std::vector<Lane> lanes;

    void* ws(int slot, size_t bytes) { return ws_in(slots, slot, bytes); }
    void* lws(int lane, int slot, size_t bytes) { return lane == 0 ? ws(slot, bytes) : ws_in(lanes[lane - 1].slots, slot, bytes); }
    void* ws_in(std::vector<Slot>& v, int slot, size_t bytes) {
        Slot& s = v[slot];
        if (bytes == 0) bytes = 16;
        if (s.bytes < bytes) {
            if (s.p) ck(cudaFree(s.p), "cudaFree");
            s.p = nullptr;
            s.bytes = 0;
            ck(cudaMalloc(&s.p, bytes), "cudaMalloc(workspace)");
            s.bytes = bytes;
        }
        return s.p;
    }
    void launched(cudaError_t e, int n = 1) {
        ck(e, "kernel launch");
        launches += n;
    }
};

namespace {

// workspace slots
enum {
    WS_X = 0, WS_A, WS_B, WS_C, WS_G, WS_Y1, WS_W, WS_W2, WS_Z, WS_Z2, WS_GRAM, WS_EIGA, WS_EIGZ, WS_EIGX, WS_POOL,
    WS_ENERGY, WS_CAPT, WS_TRACE, WS_FAIL, WS_FROZEN, WS_TAU, WS_FREQ, WS_COEF, WS_H, WS_PG, WS_EG, WS_SINR, WS_SIG,
    WS_STATUS, WS_MISC, WS_PART, WS_GPART, WS_STOP, WS_EIG64, WS_BREADY, WS_EREADY
};


template <class F>
int guarded(gwt_ctx* ctx, F&& f) {
    if (!ctx) return GWT_INVALID_ARGUMENT;
    try {
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        f();
        ctx->last_error.clear();
        return GWT_OK;
    } catch (const GwtError& e) {
        ctx->last_error = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        ctx->last_error = e.what();
        return GWT_RUNTIME_ERROR;
    }
}

void validate_topology(const gwt_topology& t) {  // SystemTopology::validate (channel.cpp)
    if (t.num_cells < 1) invalid("topology: num_cells (J) must be >= 1");
    if (t.users_per_cell < 1) invalid("topology: users_per_cell (K) must be >= 1");
    if (t.rx_antennas < 1) invalid("topology: rx_antennas (M) must be >= 1");
    if (t.tx_antennas < 1) invalid("topology: tx_antennas (N) must be >= 1");
    if (t.num_taps < 1) invalid("topology: num_taps (P) must be >= 1");
    if (t.num_streams < 1) invalid("topology: num_streams (L) must be >= 1");
    if (t.num_streams > std::min(t.rx_antennas, t.tx_antennas))
        invalid("topology: num_streams (L) must satisfy L <= min(M, N)");
    if (!(t.noise_std > 0.0)) invalid("topology: noise_std (sigma) must be > 0");
}

void validate_ranks(const gwt_ranks& r, int d1, int d2, int d3) {  // decompose.cpp:58-68
    if (r.m < 1 || r.m > d1)
        invalid("rank m = " + std::to_string(r.m) + " out of range for mode-1 size " + std::to_string(d1));
    if (r.n < 1 || r.n > d2)
        invalid("rank n = " + std::to_string(r.n) + " out of range for mode-2 size " + std::to_string(d2));
    if (r.p < 1 || r.p > d3)
        invalid("rank p = " + std::to_string(r.p) + " out of range for mode-3 size " + std::to_string(d3));
}

Topo mk_topo(const gwt_topology& t, const gwt_ranks& r) {
    Topo o;
    o.J = t.num_cells; o.K = t.users_per_cell; o.M = t.rx_antennas; o.N = t.tx_antennas; o.P = t.num_taps;
    o.m = r.m; o.n = r.n; o.p = r.p; o.L = t.num_streams;
    return o;
}

struct Timer {
    gwt_ctx* ctx;
    int n = 0;
    explicit Timer(gwt_ctx* c) : ctx(c) {
        for (auto& e : ctx->ev)
            if (!e) ck(cudaEventCreate(&e), "cudaEventCreate");
    }
    void mark(int i) { ck(cudaEventRecord(ctx->ev[i], ctx->stream), "cudaEventRecord"); }
    float between(int a, int b) {
        float ms = 0;
        cudaEventElapsedTime(&ms, ctx->ev[a], ctx->ev[b]);
        return ms;
    }
};

size_t csize(gwt_dtype dt) { return dt == GWT_C64 ? 8 : 16; }

// ---------------------------------------------------------------------------
// Tucker solve on device pointers for one sub-chunk of groups on one solver lane (stream +
// workspace). The driver interleaves the lanes sweep by sweep, so the latency-bound eigensolver
// launches of one lane overlap the bandwidth-bound contractions of the others.
template <class T>
struct SolveLane {
    using Cx = cplx_t<T>;
    gwt_ctx* ctx = nullptr;
    int lane = 0;
    cudaStream_t st = nullptr;
    Topo t{};
    int64_t G = 0;
    const void* X = nullptr;
    int sweeps = 0;
    unsigned flags = 0;
    void *A = nullptr, *B = nullptr, *Cf = nullptr, *Gc = nullptr;
    double *trace_d = nullptr, *energy = nullptr;
    // workspace
    void *Y1, *W, *W2, *Z, *Z2, *gram, *gpart, *pool;
    size_t gpart_bytes = 0;
    double2* eA;
    double* eZ;
    double2* eX;
    double *capt, *part;
    int* failp;
    int hfail = 0;
    GemmDesc dZ{}, dZ2{}, dG{}, dY1{}, dW{}, dW2{};
    int rx_kind = 0, tx_kind = 0, rx_copies = 0, tx_copies = 0;
    // early stop (decompose.cpp:363-368), decided on the device (k_stop_freeze)
    bool early = false;
    std::vector<int> iters;
    char* frozen = nullptr;
    int* stopd = nullptr;  // [G flags][G iterations_run][count]
    int* hcount = nullptr;  // pinned copy of the stopped count
    cudaEvent_t sev[3] = {};
    bool done = false;
    // fixed-sweep mode: the objective tail (core, ||core||^2, trace entry) of sweep s runs on a side
    // stream; nothing on the next sweep's rx -> tx path reads its inputs' successors, only that
    // sweep's Z2 = Z x2 B^H rewrite (and the delay update after it) must wait for it
    cudaStream_t side = nullptr;
    cudaEvent_t evc = nullptr, evo = nullptr, eva = nullptr, evz = nullptr;
    bool tail_pending = false;
    size_t a_sz = 0, b_sz = 0, c_sz = 0, g_sz = 0;

    void* ws(int slot, size_t bytes) { return ctx->lws(lane, slot, bytes); }
    void gemm(const GemmDesc& d, const void* in, const void* U, void* out) {
        ctx->launched(launch_cgemm<T>(t, d, G, in, U, out, st));
    }
    void gram_eig(const GramDesc& d, const void* V, int D, int count, void* out_factor, int copies, bool delay = false) {
        // copies > 0: pooled (one set per group) broadcast to `copies` factors
        const int users = t.users(), links = t.links();
        const int sets = d.set_kind == FI_USER ? users : d.set_kind == FI_BASE ? t.J : d.set_kind == FI_LINK ? links : 1;
        ctx->launched(launch_gram<T>(t, d, G, sets, V, gram, gpart, gpart_bytes, st, ctx->opt.gram_tc));
        void* dst = copies > 0 ? pool : out_factor;
        const int64_t batch = G * sets;
        if (sizeof(T) == 4 && D > 8 && (D >= ctx->opt.eig64_min_d || (delay && D >= 64))) {
            // c64 Gram decomposed in binary64: the delay Gram carries the power-delay profile's graded
            // spectrum (p_q ~ e^-0.3q: 1e-3 at the 24th of 64 taps), and the fp32 Householder's eps32 ||A||
            // backward error moves its trailing kept eigenvectors (C4: NMSE +1.3e-6 vs the oracle; 6e-8 in
            // binary64). GWT_EIG64_MIN_D forces binary64 for every mode with D >= the value.
            double2* g64 = (double2*)ws(WS_EIG64, 16 * batch * ((int64_t)D * D + (int64_t)D * count));
            double2* o64 = g64 + batch * D * D;
            ctx->launched(launch_cplx_widen(gram, g64, batch * D * D, st));
            ctx->launched(launch_heev_topk<double>(D, count, batch, g64, o64, nullptr, eA, eZ, eX, failp, st));
            ctx->launched(launch_cplx_narrow(o64, dst, batch * D * count, st));
        } else {
            ctx->launched(launch_heev_topk<T>(D, count, batch, gram, dst, nullptr, eA, eZ, eX, failp, st));
            // fp32 eigensolvers: restore orthonormality in binary64 (k_orth.cu); D <= 8 is solved in binary64
            if (sizeof(T) == 4 && D > 8) ctx->launched(launch_orth_cholqr(D, count, batch, dst, st));
        }
        if (copies > 0) ctx->launched(launch_broadcast<T>(pool, out_factor, (int64_t)D * count, copies, G, st));
    }
    void objective(int slot) {
        gemm(dZ, X, A, Z);
        gemm(dZ2, Z, B, Z2);
        gemm(dG, Z2, Cf, Gc);
        ctx->launched(launch_group_sqnorm<T>(Gc, (int64_t)t.links() * t.m * t.n * t.p, G, capt, part, st));
        ctx->launched(launch_objective(G, energy, capt, trace_d, sweeps + 1, slot, st));
    }

    // allocations, ||X||^2, initial factors (decompose.cpp:248-300) and the sweep-0 objective
    void begin() {
        const size_t cs = sizeof(Cx);
        const int links = t.links(), users = t.users();
        const int64_t MNP = (int64_t)t.M * t.N * t.P;
        const bool pooled = flags & GWT_SOLVE_POOLED;
        early = flags & GWT_SOLVE_EARLY_STOP;
        Y1 = ws(WS_Y1, cs * G * links * t.M * t.N * t.p);
        W = ws(WS_W, cs * G * links * t.M * t.n * t.p);
        W2 = ws(WS_W2, cs * G * links * t.m * t.N * t.p);
        Z = ws(WS_Z, cs * G * links * t.m * t.N * t.P);
        Z2 = ws(WS_Z2, cs * G * links * t.m * t.n * t.P);
        const int64_t gram_elems = std::max({(int64_t)G * users * t.M * t.M, (int64_t)G * t.J * t.N * t.N,
                                             (int64_t)G * links * t.P * t.P});
        gram = ws(WS_GRAM, cs * gram_elems);
        gpart_bytes = std::min<size_t>(cs * gram_elems * 8, size_t(256) << 20);  // K-split partials
        gpart = ws(WS_GPART, gpart_bytes);
        const int64_t eig_a = std::max({(int64_t)G * users * heev_ws_a_elems(t.M),
                                        (int64_t)G * t.J * heev_ws_a_elems(t.N), (int64_t)G * links * heev_ws_a_elems(t.P)});
        const int64_t eig_z = std::max({(int64_t)G * users * heev_ws_z_elems(t.M, t.m),
                                        (int64_t)G * t.J * heev_ws_z_elems(t.N, t.n),
                                        (int64_t)G * links * heev_ws_z_elems(t.P, t.p)});
        const int64_t eig_x = std::max({(int64_t)G * users * t.M * t.m, (int64_t)G * t.J * t.N * t.n,
                                        (int64_t)G * links * t.P * t.p});
        eA = (double2*)ws(WS_EIGA, 16 * eig_a);
        eZ = (double*)ws(WS_EIGZ, 8 * eig_z);
        eX = (double2*)ws(WS_EIGX, 16 * eig_x);
        pool = ws(WS_POOL, cs * G * std::max(t.M * t.m, t.N * t.n));
        capt = (double*)ws(WS_CAPT, 8 * G);
        failp = (int*)ws(WS_FAIL, 4);
        part = (double*)ws(WS_PART, 8 * G * kSqnormMaxBlocks);
        ck(cudaMemsetAsync(failp, 0, 4, st), "memset");
        // mode-product descriptors
        dZ.R = t.N * t.P; dZ.S = 1; dZ.Kd = t.M; dZ.Cols = t.m;  // Z = X x1 A^H  (m x N x P)
        dZ.in_item = MNP; dZ.rs_in = t.M; dZ.s_in = 0; dZ.ks_in = 1;
        dZ.out_item = (int64_t)t.m * t.N * t.P; dZ.rs_out = t.m; dZ.s_out = 0; dZ.cs_out = 1; dZ.fkind = FI_USER;
        dZ2.R = t.m; dZ2.S = t.P; dZ2.Kd = t.N; dZ2.Cols = t.n;  // Z2 = Z x2 B^H (m x n x P)
        dZ2.in_item = (int64_t)t.m * t.N * t.P; dZ2.rs_in = 1; dZ2.s_in = (int64_t)t.m * t.N; dZ2.ks_in = t.m;
        dZ2.out_item = (int64_t)t.m * t.n * t.P; dZ2.rs_out = 1; dZ2.s_out = (int64_t)t.m * t.n; dZ2.cs_out = t.m;
        dZ2.fkind = FI_BASE;
        dG.R = t.m * t.n; dG.S = 1; dG.Kd = t.P; dG.Cols = t.p;  // core = Z2 x3 C^H (m x n x p)
        dG.in_item = (int64_t)t.m * t.n * t.P; dG.rs_in = 1; dG.s_in = 0; dG.ks_in = (int64_t)t.m * t.n;
        dG.out_item = (int64_t)t.m * t.n * t.p; dG.rs_out = 1; dG.s_out = 0; dG.cs_out = (int64_t)t.m * t.n;
        dG.fkind = FI_LINK;
        dY1.R = t.M * t.N; dY1.S = 1; dY1.Kd = t.P; dY1.Cols = t.p;  // Y1 = X x3 C^H (M x N x p)
        dY1.in_item = MNP; dY1.rs_in = 1; dY1.s_in = 0; dY1.ks_in = (int64_t)t.M * t.N;
        dY1.out_item = (int64_t)t.M * t.N * t.p; dY1.rs_out = 1; dY1.s_out = 0; dY1.cs_out = (int64_t)t.M * t.N;
        dY1.fkind = FI_LINK;
        dW.R = t.M; dW.S = t.p; dW.Kd = t.N; dW.Cols = t.n;  // W = Y1 x2 B^H (M x n x p)
        dW.in_item = (int64_t)t.M * t.N * t.p; dW.rs_in = 1; dW.s_in = (int64_t)t.M * t.N; dW.ks_in = t.M;
        dW.out_item = (int64_t)t.M * t.n * t.p; dW.rs_out = 1; dW.s_out = (int64_t)t.M * t.n; dW.cs_out = t.M;
        dW.fkind = FI_BASE;
        dW2.R = t.N * t.p; dW2.S = 1; dW2.Kd = t.M; dW2.Cols = t.m;  // W2 = Y1 x1 A^H (m x N x p)
        dW2.in_item = (int64_t)t.M * t.N * t.p; dW2.rs_in = t.M; dW2.s_in = 0; dW2.ks_in = 1;
        dW2.out_item = (int64_t)t.m * t.N * t.p; dW2.rs_out = t.m; dW2.s_out = 0; dW2.cs_out = 1; dW2.fkind = FI_USER;
        rx_kind = pooled ? FI_GROUP : FI_USER;
        tx_kind = pooled ? FI_GROUP : FI_BASE;
        rx_copies = pooled ? users : 0;
        tx_copies = pooled ? t.J : 0;

        ctx->launched(launch_group_sqnorm<T>(X, links * MNP, G, energy, part, st));
        if (!(flags & GWT_SOLVE_INIT)) {
            GramDesc g1{t.M, t.N * t.P, 1, MNP, 1, t.M, 0, rx_kind};
            gram_eig(g1, X, t.M, t.m, A, rx_copies);
            GramDesc g2{t.N, t.M, t.P, MNP, t.M, 1, (int64_t)t.M * t.N, tx_kind};
            gram_eig(g2, X, t.N, t.n, B, tx_copies);
            GramDesc g3{t.P, t.M * t.N, 1, MNP, (int64_t)t.M * t.N, 1, 0, FI_LINK};
            gram_eig(g3, X, t.P, t.p, Cf, 0, true);
        }
        objective(0);
        a_sz = cs * users * t.M * t.m;
        b_sz = cs * t.J * t.N * t.n;
        c_sz = cs * links * t.P * t.p;
        g_sz = cs * links * t.m * t.n * t.p;
        if (early) {
            frozen = (char*)ws(WS_FROZEN, (a_sz + b_sz + c_sz + g_sz) * G);
            stopd = (int*)ws(WS_STOP, 4 * (2 * G + 1));
            ck(cudaMemsetAsync(stopd, 0, 4 * (2 * G + 1), st), "memset");
            hcount = ctx->pin(lane);
            *hcount = 0;
            for (auto& e : sev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        }
        iters.assign(G, sweeps);
        done = false;
        tail_pending = false;
        side = nullptr;
        if (!early && sweeps > 0 && ctx->opt.solve_side) {
            side = ctx->side_stream(lane);
            evc = ctx->side_ev[lane][0];
            evo = ctx->side_ev[lane][1];
            eva = ctx->side_ev[lane][2];
            evz = ctx->side_ev[lane][3];
        }
    }

    // enqueue one alternating sweep (decompose.cpp:330-370): rx, tx, delay factors, then cores + objective
    void sweep(int s) {
        gemm(dY1, X, Cf, Y1);
        gemm(dW, Y1, B, W);
        GramDesc grx{t.M, t.n * t.p, 1, (int64_t)t.M * t.n * t.p, 1, t.M, 0, rx_kind};
        gram_eig(grx, W, t.M, t.m, A, rx_copies);
        if (side) {  // Z = X x1 A^H needs only the new A: computed beside the tx update, behind the tail
            ck(cudaEventRecord(eva, st), "cudaEventRecord");
            ck(cudaStreamWaitEvent(side, eva, 0), "cudaStreamWaitEvent");
            ctx->launched(launch_cgemm<T>(t, dZ, G, X, A, Z, side));
            ck(cudaEventRecord(evz, side), "cudaEventRecord");
        }
        gemm(dW2, Y1, A, W2);
        GramDesc gtx{t.N, t.m, t.p, (int64_t)t.m * t.N * t.p, t.m, 1, (int64_t)t.m * t.N, tx_kind};
        gram_eig(gtx, W2, t.N, t.n, B, tx_copies);
        if (side) {  // Z ready, and the previous sweep's tail (which still read Z2 and C) done before it
            ck(cudaStreamWaitEvent(st, evz, 0), "cudaStreamWaitEvent");
            tail_pending = false;
        } else {
            gemm(dZ, X, A, Z);
        }
        if (tail_pending) {  // the previous sweep's tail still reads Z2 and C
            ck(cudaStreamWaitEvent(st, evo, 0), "cudaStreamWaitEvent");
            tail_pending = false;
        }
        gemm(dZ2, Z, B, Z2);
        GramDesc gd{t.P, t.m * t.n, 1, (int64_t)t.m * t.n * t.P, (int64_t)t.m * t.n, 1, 0, FI_LINK};
        gram_eig(gd, Z2, t.P, t.p, Cf, 0, true);
        if (side) {
            ck(cudaEventRecord(evc, st), "cudaEventRecord");
            ck(cudaStreamWaitEvent(side, evc, 0), "cudaStreamWaitEvent");
            ctx->launched(launch_cgemm<T>(t, dG, G, Z2, Cf, Gc, side));
            ctx->launched(launch_group_sqnorm<T>(Gc, (int64_t)t.links() * t.m * t.n * t.p, G, capt, part, side));
            ctx->launched(launch_objective(G, energy, capt, trace_d, sweeps + 1, s + 1, side));
            ck(cudaEventRecord(evo, side), "cudaEventRecord");
            tail_pending = true;
            return;
        }
        gemm(dG, Z2, Cf, Gc);
        ctx->launched(launch_group_sqnorm<T>(Gc, (int64_t)t.links() * t.m * t.n * t.p, G, capt, part, st));
        ctx->launched(launch_objective(G, energy, capt, trace_d, sweeps + 1, s + 1, st));
        if (early) {
            ctx->launched(launch_stop_freeze(G, trace_d, energy, sweeps + 1, s, stopd, A, B, Cf, Gc, frozen, a_sz, b_sz,
                                             c_sz, g_sz, st));
            ck(cudaMemcpyAsync(hcount, stopd + 2 * G, 4, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaEventRecord(sev[s % 3], st), "cudaEventRecord");
        }
    }

    // host side, early-stop mode: wait for sweep s to finish (the lane keeps the next sweep queued)
    // and retire the lane once every group in it has stopped
    void poll(int s) {
        ck(cudaEventSynchronize(sev[s % 3]), "cudaEventSynchronize");
        if (*hcount >= G) done = true;
    }

    void end() {
        if (tail_pending) {
            ck(cudaStreamWaitEvent(st, evo, 0), "cudaStreamWaitEvent");
            tail_pending = false;
        }
        if (early) {
            ctx->launched(launch_unfreeze(G, stopd, A, B, Cf, Gc, frozen, a_sz, b_sz, c_sz, g_sz, st));
            std::vector<int> h(2 * G);
            ck(cudaMemcpyAsync(h.data(), stopd, 8 * G, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaStreamSynchronize(st), "sync");
            for (int64_t g = 0; g < G; ++g) iters[g] = h[g] ? h[G + g] : sweeps;
            for (auto& e : sev) cudaEventDestroy(e);
        }
        ck(cudaMemcpyAsync(&hfail, failp, 4, cudaMemcpyDeviceToHost, st), "D2H");
    }
};

// Solve one chunk of G groups (device pointers) on up to ctx->opt.solve_lanes concurrent lanes.
template <class T>
void solve_chunk(gwt_ctx* ctx, const Topo& t, int64_t G, const void* X, int sweeps, unsigned flags, void* A, void* B,
                 void* Cf, void* Gc, double* trace_d, double* energy_d, std::vector<int>& iters, double* ms) {
    using Cx = cplx_t<T>;
    const size_t cs = sizeof(Cx);
    const int links = t.links(), users = t.users();
    const int64_t x_g = (int64_t)links * t.M * t.N * t.P, a_g = (int64_t)users * t.M * t.m,
                  b_g = (int64_t)t.J * t.N * t.n, c_g = (int64_t)links * t.P * t.p,
                  g_g = (int64_t)links * t.m * t.n * t.p;
    const int L = (int)std::min<int64_t>(std::max(1, std::min(8, ctx->opt.solve_lanes)), G);
    while ((int)ctx->lanes.size() < L - 1) {
        gwt_ctx::Lane ln;
        ck(cudaStreamCreateWithFlags(&ln.st, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaEventCreateWithFlags(&ln.ev, cudaEventDisableTiming), "cudaEventCreate");
        ctx->lanes.push_back(ln);
    }
    Timer tm(ctx);
    tm.mark(1);
    std::vector<SolveLane<T>> lanes(L);
    if (L > 1) {  // lanes 1.. start after everything already queued on ctx->stream
        ck(cudaEventRecord(ctx->ev[10], ctx->stream), "cudaEventRecord");
        for (int l = 1; l < L; ++l) ck(cudaStreamWaitEvent(ctx->lanes[l - 1].st, ctx->ev[10], 0), "cudaStreamWaitEvent");
    }
    int64_t g0 = 0;
    for (int l = 0; l < L; ++l) {
        SolveLane<T>& ln = lanes[l];
        const int64_t Gl = G / L + (l < G % L ? 1 : 0);
        ln.ctx = ctx;
        ln.lane = l;
        ln.st = l == 0 ? ctx->stream : ctx->lanes[l - 1].st;
        ln.t = t;
        ln.G = Gl;
        ln.X = (const char*)X + cs * g0 * x_g;
        ln.sweeps = sweeps;
        ln.flags = flags;
        ln.A = (char*)A + cs * g0 * a_g;
        ln.B = (char*)B + cs * g0 * b_g;
        ln.Cf = (char*)Cf + cs * g0 * c_g;
        ln.Gc = (char*)Gc + cs * g0 * g_g;
        ln.trace_d = trace_d + g0 * (sweeps + 1);
        ln.energy = energy_d + g0;
        g0 += Gl;
        ln.begin();
    }
    tm.mark(2);
    const bool early = flags & GWT_SOLVE_EARLY_STOP;
    // early stop is decided on the device; the host stays one sweep ahead of each lane (so the GPU
    // never idles on it) and stops enqueuing a lane once all its groups have stopped
    for (int s = 0; s < sweeps; ++s) {
        bool any = false;
        for (auto& ln : lanes)
            if (!ln.done) {
                ln.sweep(s);
                any = true;
            }
        if (!any) break;
        if (early && s >= 1 && ctx->opt.poll)
            for (auto& ln : lanes)
                if (!ln.done) ln.poll(s - 1);
    }
    for (auto& ln : lanes) ln.end();
    for (int l = 1; l < L; ++l) {  // ctx->stream waits for the other lanes
        ck(cudaEventRecord(ctx->lanes[l - 1].ev, ctx->lanes[l - 1].st), "cudaEventRecord");
        ck(cudaStreamWaitEvent(ctx->stream, ctx->lanes[l - 1].ev, 0), "cudaStreamWaitEvent");
    }
    tm.mark(3);
    ck(cudaStreamSynchronize(ctx->stream), "sync");
    iters.clear();
    for (auto& ln : lanes) {
        if (ln.hfail) fail(GWT_RUNTIME_ERROR, "leading_eigenvectors: eigendecomposition failed");
        iters.insert(iters.end(), ln.iters.begin(), ln.iters.end());
    }
    ms[0] += tm.between(1, 2);
    ms[1] += tm.between(2, 3);
}

template <class T>
void groupwise_solve_impl(gwt_ctx* ctx, const gwt_topology* topo, const gwt_ranks* ranks, int64_t ngroups,
                          gwt_mem mem, const void* X, int sweeps, unsigned flags, void* A, void* B, void* Cf,
                          void* Gc, double* trace, int32_t* iters, double* energy) {
    using Cx = cplx_t<T>;
    const size_t cs = sizeof(Cx);
    // reference checks: check_channel_dims, ranks.validate_against, sweeps >= 0 (decompose.cpp:314-318)
    gwt_topology tt = *topo;
    if (tt.num_streams < 1) tt.num_streams = 1;
    if (tt.num_cells < 1 || tt.users_per_cell < 1 || tt.rx_antennas < 1 || tt.tx_antennas < 1 || tt.num_taps < 1)
        invalid("channel set: inconsistent tensor dims");
    validate_ranks(*ranks, tt.rx_antennas, tt.tx_antennas, tt.num_taps);
    if (sweeps < 0) invalid("solve: sweeps must be >= 0");
    if (ngroups < 0) invalid("solve: ngroups must be >= 0");
    if (std::max({tt.rx_antennas, tt.tx_antennas, tt.num_taps}) > 256)
        invalid("solve: mode sizes above 256 are not supported by the batched eigensolver");
    if (ngroups == 0) return;
    const Topo t = mk_topo(tt, *ranks);
    const int links = t.links(), users = t.users();
    const int64_t x_g = (int64_t)links * t.M * t.N * t.P, a_g = (int64_t)users * t.M * t.m,
                  b_g = (int64_t)t.J * t.N * t.n, c_g = (int64_t)links * t.P * t.p,
                  g_g = (int64_t)links * t.m * t.n * t.p;
    // per-group workspace bytes -> group chunk
    const int64_t per_group = cs * (links * ((int64_t)t.M * t.N * t.p + (int64_t)t.M * t.n * t.p +
                                             (int64_t)t.m * t.N * t.p + (int64_t)t.m * t.N * t.P +
                                             (int64_t)t.m * t.n * t.P) +
                                    std::max({(int64_t)users * t.M * t.M, (int64_t)t.J * t.N * t.N,
                                              (int64_t)links * t.P * t.P}) * 3) +
                              (mem == GWT_MEM_HOST ? cs * (x_g + a_g + b_g + c_g + g_g) : 0);
    int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(ngroups, (int64_t)(ctx->opt.ws_bytes / std::max<int64_t>(per_group, 1))));
    double ms[2] = {0, 0};
    Timer tm(ctx);
    tm.mark(0);
    double h2d_ms = 0;
    for (int64_t g0 = 0; g0 < ngroups; g0 += chunk) {
        const int64_t G = std::min(chunk, ngroups - g0);
        const void* Xd;
        void *Ad, *Bd, *Cd, *Gd;
        double* trace_d = (double*)ctx->ws(WS_TRACE, 8 * G * (sweeps + 1));
        if (mem == GWT_MEM_HOST) {
            tm.mark(4);
            void* xb = ctx->ws(WS_X, cs * G * x_g);
            ck(cudaMemcpyAsync(xb, (const char*)X + cs * g0 * x_g, cs * G * x_g, cudaMemcpyHostToDevice, ctx->stream), "H2D X");
            Xd = xb;
            Ad = ctx->ws(WS_A, cs * G * a_g);
            Bd = ctx->ws(WS_B, cs * G * b_g);
            Cd = ctx->ws(WS_C, cs * G * c_g);
            Gd = ctx->ws(WS_G, cs * G * g_g);
            if (flags & GWT_SOLVE_INIT) {
                ck(cudaMemcpyAsync(Ad, (const char*)A + cs * g0 * a_g, cs * G * a_g, cudaMemcpyHostToDevice, ctx->stream), "H2D");
                ck(cudaMemcpyAsync(Bd, (const char*)B + cs * g0 * b_g, cs * G * b_g, cudaMemcpyHostToDevice, ctx->stream), "H2D");
                ck(cudaMemcpyAsync(Cd, (const char*)Cf + cs * g0 * c_g, cs * G * c_g, cudaMemcpyHostToDevice, ctx->stream), "H2D");
            }
            tm.mark(5);
            ck(cudaStreamSynchronize(ctx->stream), "sync");
            h2d_ms += tm.between(4, 5);
        } else {
            Xd = (const char*)X + cs * g0 * x_g;
            Ad = (char*)A + cs * g0 * a_g;
            Bd = (char*)B + cs * g0 * b_g;
            Cd = (char*)Cf + cs * g0 * c_g;
            Gd = (char*)Gc + cs * g0 * g_g;
        }
        std::vector<int> it;
        std::vector<double> th;
        double* en = (double*)ctx->ws(WS_ENERGY, 8 * G);
        solve_chunk<T>(ctx, t, G, Xd, sweeps, flags, Ad, Bd, Cd, Gd, trace_d, en, it, ms);
        // trace: entries after an early stop repeat the final objective
        th.resize((size_t)G * (sweeps + 1));
        ck(cudaMemcpy(th.data(), trace_d, 8 * th.size(), cudaMemcpyDeviceToHost), "D2H trace");
        for (int64_t g = 0; g < G; ++g)
            for (int s = it[g] + 1; s <= sweeps; ++s) th[g * (sweeps + 1) + s] = th[g * (sweeps + 1) + it[g]];
        std::vector<double> enh(G);
        ck(cudaMemcpy(enh.data(), en, 8 * G, cudaMemcpyDeviceToHost), "D2H energy");
        if (mem == GWT_MEM_HOST) {
            tm.mark(4);
            ck(cudaMemcpyAsync((char*)A + cs * g0 * a_g, Ad, cs * G * a_g, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
            ck(cudaMemcpyAsync((char*)B + cs * g0 * b_g, Bd, cs * G * b_g, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
            ck(cudaMemcpyAsync((char*)Cf + cs * g0 * c_g, Cd, cs * G * c_g, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
            ck(cudaMemcpyAsync((char*)Gc + cs * g0 * g_g, Gd, cs * G * g_g, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
            if (trace) std::memcpy(trace + g0 * (sweeps + 1), th.data(), 8 * th.size());
            if (iters) for (int64_t g = 0; g < G; ++g) iters[g0 + g] = it[g];
            if (energy) std::memcpy(energy + g0, enh.data(), 8 * G);
            tm.mark(5);
            ck(cudaStreamSynchronize(ctx->stream), "sync");
            h2d_ms += tm.between(4, 5);
        } else {
            if (trace) ck(cudaMemcpyAsync(trace + g0 * (sweeps + 1), th.data(), 8 * th.size(), cudaMemcpyHostToDevice, ctx->stream), "H2D");
            std::vector<int32_t> it32(it.begin(), it.end());
            if (iters) ck(cudaMemcpyAsync(iters + g0, it32.data(), 4 * G, cudaMemcpyHostToDevice, ctx->stream), "H2D");
            if (energy) ck(cudaMemcpyAsync(energy + g0, en, 8 * G, cudaMemcpyDeviceToDevice, ctx->stream), "D2D");
            ck(cudaStreamSynchronize(ctx->stream), "sync");
        }
    }
    tm.mark(6);
    ck(cudaStreamSynchronize(ctx->stream), "sync");
    std::fill(ctx->stage_ms, ctx->stage_ms + 8, 0.0);
    ctx->stage_ms[0] = tm.between(0, 6);
    ctx->stage_ms[1] = ms[0];
    ctx->stage_ms[2] = ms[1];
    ctx->stage_ms[7] = h2d_ms;
}

// ---------------------------------------------------------------------------
// compressed SINR
void validate_sinr(const gwt_topology& tp, const gwt_ranks& r, int scope) {
    // run_compressed_pipeline does not validate the topology; the first checks it meets are the
    // precoder's stream count (sinr.cpp:163-167) and woodbury_inverse_apply's sigma (:208-209)
    if (tp.num_cells < 1 || tp.users_per_cell < 1 || tp.num_taps < 1 || tp.num_streams < 1)
        invalid("topology: num_cells, users_per_cell, num_taps and num_streams must be >= 1");
    if (r.m < 1 || r.n < 1 || r.p < 1) invalid("ranks must be >= 1");
    if (scope != GWT_SCOPE_FULL && scope != GWT_SCOPE_PAPER) invalid("sinr: unknown interference scope");
    if (tp.num_streams > std::min(r.m, r.n))  // precoder_compressed (sinr.cpp:163-167)
        invalid("precoder: stream count " + std::to_string(tp.num_streams) + " exceeds compressed channel size " +
                std::to_string(r.m) + "x" + std::to_string(r.n) + " (ranks chosen below stream count)");
    if (!(tp.noise_std > 0.0)) invalid("woodbury_inverse_apply: sigma must be > 0");
    if (r.m > 8) invalid("sinr: compressed receive rank m > 8 is not supported by the B200 small-matrix kernel");
}

// Per-stage CUDA events recorded by sinr_device without a host wait (lanes stay asynchronous);
// resolved after the caller's final synchronisation.
struct StageEvents {
    std::vector<cudaEvent_t> evs;  // per lane call: boundaries
    std::vector<int> kind;         // interval i between evs[i] and evs[i+1] (within one call), -1 = call break
    void resolve(double& ms_r, double& ms_p, double& ms_s) {
        for (size_t i = 0; i < kind.size(); ++i) {
            if (kind[i] < 0) continue;
            float a = 0;
            cudaEventElapsedTime(&a, evs[i], evs[i + 1]);
            (kind[i] == 0 ? ms_r : kind[i] == 1 ? ms_p : ms_s) += a;
        }
        for (auto& ev : evs) cudaEventDestroy(ev);
        evs.clear();
        kind.clear();
    }
};

// the tensor-core rebuild + pair-Gram path (k_rgram.cu) for large cores (m n >= 256: C3, C4, C5); the small
// C2 cores (m n = 96) measured faster on the CUDA-core rebuild + pair-Gram kernels (0.54 vs 0.63 ms)
bool tc_sinr_shape(const gwt_ctx* ctx, const Topo& t) {
    return rgram_fits(t) && (ctx->opt.sinr_path == 1 || t.m * t.n >= 256);
}

// Generic device pipeline (any scope) for ngroups groups on device pointers, on solver/SINR lane
// `lane` (stream st + its workspace): rebuild -> pair Grams per subcarrier chunk, then ONE eig+MMSE
// launch per pair-Gram block. timing: per-stage CUDA events (host waits at the end).
template <class T>
void sinr_device(gwt_ctx* ctx, int lane, cudaStream_t st, const Topo& t, const gwt_topology* topo, int64_t ngroups,
                 const void* Cd, const void* Gd, const double* taud, const double* fd, const void* cod, int64_t F,
                 int scope, double* sd, double* sgd, int* std_, bool timing, double& ms_r, double& ms_p, double& ms_s,
                 StageEvents* deferred = nullptr) {
    using Cx = cplx_t<T>;
    const size_t cs = sizeof(Cx);
    const int links = t.links(), users = t.users();
    const int S = scope == GWT_SCOPE_PAPER ? t.J : t.J * t.K;
    const int path = ctx->opt.sinr_path;
    {
        // generic path (any scope): rebuild -> pair Grams per subcarrier chunk sized so H~ stays resident in
        // L2 between producer and consumer; then ONE eig+MMSE launch over all subcarriers (full occupancy)
        const int64_t per_f_h = (int64_t)cs * ngroups * links * t.m * t.n;
        // (measured on C2: L2-sized chunks are slower - fewer CTAs per launch - so default to 2 GiB)
        const int64_t chunk_bytes = ctx->opt.sinr_chunk_bytes;
        const int64_t Fc = std::max<int64_t>(1, std::min<int64_t>(F, chunk_bytes / std::max<int64_t>(per_f_h, 1)));
        // stage S: the per-user kernel (k_users.cu) for m > 4; for m <= 4 the pair-Gram route
        // (K2 + thread-per-user K3) measured faster (C2: 0.21 vs 0.31 ms). GWT_SINR_PATH=users|pg forces one.
        const bool force_users = path == 2, force_pg = path == 3;
        const bool users_path = scope == GWT_SCOPE_PAPER && sinr_users_fits(t, cs) && !force_pg && (t.m > 4 || force_users);
        // c64 paper scope, m in {4, 8}: rebuild fused with the pair Grams on the tensor cores (k_rgram.cu)
        const bool tc_path = sizeof(T) == 4 && scope == GWT_SCOPE_PAPER && !cod && tc_sinr_shape(ctx, t) && !force_users &&
                             !force_pg;
        if (tc_path) {
            const int64_t Ft = std::min<int64_t>(F, 256);
            double2* PGt = (double2*)ctx->lws(lane, WS_PG, 16 * ngroups * Ft * users * S * t.m * t.m);
            double* EGt = (double*)ctx->lws(lane, WS_EG, 8 * ngroups * Ft * users * (((t.L + 1) & ~1) + 2 * t.m * t.L));
            void* Bready = ctx->lws(lane, WS_BREADY, rgram_bready_bytes(t, ngroups));
            void* Eready = ctx->lws(lane, WS_EREADY, rgram_eready_bytes(t, ngroups, (int)Ft));
            std::vector<cudaEvent_t> evs_l;
            std::vector<int> kind_l;
            std::vector<cudaEvent_t>& evs = deferred ? deferred->evs : evs_l;
            std::vector<int>& kind = deferred ? deferred->kind : kind_l;
            if (deferred && !evs.empty()) kind.push_back(-1);
            auto rec = [&]() {
                if (!timing && !deferred) return;
                cudaEvent_t ev;
                ck(cudaEventCreate(&ev), "cudaEventCreate");
                ck(cudaEventRecord(ev, st), "event");
                evs.push_back(ev);
            };
            rec();
            ctx->launched(launch_rgram_prep(t, ngroups, Gd, Bready, st));
            rec();
            kind.push_back(0);
            for (int64_t f0 = 0; f0 < F; f0 += Ft) {
                const int fc = (int)std::min(Ft, F - f0);
                ctx->launched(launch_rgram(t, ngroups, fc, f0, 0, fc, Cd, taud, fd, Bready, Eready, PGt, st), 2);
                rec();
                kind.push_back(1);
                // m > 4: the per-user Householder/QL kernel in PG mode; m <= 4: the thread-per-user Jacobi kernel
                if (t.m > 4 && sinr_users_pg_fits(t) && !ctx->opt.pg_small)
                    ctx->launched(launch_sinr_users_pg(t, ngroups * fc, fc, F, f0, topo->noise_std, PGt, sd, sgd, std_, st));
                else
                    ctx->launched(launch_sinr_small(t, scope, S, ngroups * fc * users, topo->noise_std, fc, F, f0, PGt,
                                                    EGt, sd, sgd, std_, st));
                rec();
                kind.push_back(2);
            }
            if (timing && !deferred) {
                ck(cudaEventSynchronize(evs.back()), "sync");
                for (size_t q = 0; q < kind.size(); ++q) {
                    float a = 0;
                    cudaEventElapsedTime(&a, evs[q], evs[q + 1]);
                    (kind[q] == 0 ? ms_r : kind[q] == 1 ? ms_p : ms_s) += a;
                }
            }
            if (!deferred)
                for (auto& ev : evs) cudaEventDestroy(ev);
            return;
        }
        void* H = ctx->lws(lane, WS_H, cs * ngroups * Fc * links * t.m * t.n);
        // pair Grams for a block of Fs subcarriers: [g][Fs][users][S][m*m] (fp64), Fs bounded by ~2 GB
        const int64_t per_f_pg = (int64_t)ngroups * users * (16LL * S * t.m * t.m + 8LL * (((t.L + 1) & ~1) + 2 * t.m * t.L));
        const int64_t Fs = std::max<int64_t>(Fc, std::min<int64_t>(F, (int64_t)(2ll << 30) / std::max<int64_t>(per_f_pg, 1)) / Fc * Fc);
        double2* PG = users_path ? nullptr : (double2*)ctx->lws(lane, WS_PG, 16 * ngroups * std::min(Fs, F) * users * S * t.m * t.m);
        double* EG = users_path ? nullptr : (double*)ctx->lws(lane, WS_EG, 8 * ngroups * std::min(Fs, F) * users * (((t.L + 1) & ~1) + 2 * t.m * t.L));
        std::vector<cudaEvent_t> evs_local;
        std::vector<int> kind_local;  // 0 rebuild, 1 pair gram, 2 small, per interval
        std::vector<cudaEvent_t>& evs = deferred ? deferred->evs : evs_local;
        std::vector<int>& kind = deferred ? deferred->kind : kind_local;
        if (deferred && !evs.empty()) kind.push_back(-1);  // break between two calls' event chains
        auto rec = [&]() {
            if (!timing && !deferred) return;
            cudaEvent_t ev;
            ck(cudaEventCreate(&ev), "cudaEventCreate");
            ck(cudaEventRecord(ev, st), "event");
            evs.push_back(ev);
        };
        rec();
        if (users_path) {
            // paper scope: rebuild -> per-user solve (serving Gram, eig, anchor precoders, MMSE) per chunk
            for (int64_t f0 = 0; f0 < F; f0 += Fc) {
                const int fc = (int)std::min(Fc, F - f0);
                ctx->launched(launch_rebuild<T>(t, (int)ngroups, fc, f0, F, Cd, Gd, taud, fd, cod, H, st));
                rec();
                kind.push_back(0);
                ctx->launched(launch_sinr_users<T>(t, ngroups * fc, fc, F, f0, topo->noise_std, H, sd, sgd, std_, st));
                rec();
                kind.push_back(2);
            }
        }
        for (int64_t F0 = 0; !users_path && F0 < F; F0 += Fs) {
            const int64_t fs = std::min(Fs, F - F0);
            for (int64_t f0 = F0; f0 < F0 + fs; f0 += Fc) {
                const int fc = (int)std::min(Fc, F0 + fs - f0);
                ctx->launched(launch_rebuild<T>(t, (int)ngroups, fc, f0, F, Cd, Gd, taud, fd, cod, H, st));
                rec();
                kind.push_back(0);
                ctx->launched(launch_pair_gram<T>(t, scope, S, fc, (int)ngroups, f0 - F0, fs, H, PG, st));
                rec();
                kind.push_back(1);
            }
            ctx->launched(launch_sinr_small(t, scope, S, ngroups * fs * users, topo->noise_std, (int)fs, F, F0, PG, EG,
                                            sd, sgd, std_, st),
                          2);
            rec();
            kind.push_back(2);
        }
        if (timing && !deferred) {
            ck(cudaEventSynchronize(evs.back()), "sync");
            for (size_t i = 0; i < kind.size(); ++i) {
                float a = 0;
                cudaEventElapsedTime(&a, evs[i], evs[i + 1]);
                (kind[i] == 0 ? ms_r : kind[i] == 1 ? ms_p : ms_s) += a;
            }
        }
        if (!deferred)
            for (auto& ev : evs) cudaEventDestroy(ev);
    }
}

template <class T>
void sinr_impl(gwt_ctx* ctx, const gwt_topology* topo, const gwt_ranks* ranks, int64_t ngroups, gwt_mem mem,
               const void* Cf, const void* Gc, const double* tau, const double* freqs, const void* coeffs, int64_t F,
               int scope, double* sinr, double* signal, int32_t* status) {
    using Cx = cplx_t<T>;
    const size_t cs = sizeof(Cx);
    const Topo t = mk_topo(*topo, *ranks);
    cudaStream_t st = ctx->stream;
    const int links = t.links(), users = t.users();
    const int S = scope == GWT_SCOPE_PAPER ? t.J : t.J * t.K;
    const int64_t c_g = (int64_t)links * t.P * t.p, g_g = (int64_t)links * t.m * t.n * t.p;
    Timer tm(ctx);
    tm.mark(0);
    double copy_ms = 0;
    const void *Cd = Cf, *Gd = Gc, *cod = coeffs;
    const double *taud = tau, *fd = freqs;
    double *sd = sinr, *sgd = signal;
    int* std_ = (int*)status;
    const int64_t out_rows = ngroups * F * users;
    // two stream lanes overlap the CUDA-core rebuild of one group half with the Gram / eig stages of the
    // other; the tensor-core path keeps every SM busy with one lane (C4: 710 ms single lane vs 839 ms)
    const bool tc_shape = sizeof(T) == 4 && scope == GWT_SCOPE_PAPER && !coeffs && tc_sinr_shape(ctx, t);
    // host-buffer calls: group chunks through the copy / compute / copy engines; the exposed copies are the first
    // chunk's H2D and the last chunk's D2H (C4, 10.7 GB per step: 4 / 8 / 16 chunks 610 / 591 / 588 ms against
    // 557 ms device-resident)
    const int64_t nch = std::min<int64_t>(ngroups, ctx->opt.sinr_pipeline > 0 ? ctx->opt.sinr_pipeline : (tc_shape ? 8 : 4));
    const int64_t ndev = std::min<int64_t>(ngroups, ctx->opt.sinr_dev_lanes > 0 ? ctx->opt.sinr_dev_lanes : (tc_shape ? 1 : 2));
    if (mem == GWT_MEM_DEVICE && ndev > 1 && !coeffs) {
        // device-resident: group chunks on ndev stream lanes so the FP32-issue-bound rebuild of one
        // chunk overlaps the memory/fp64-bound Gram and small-matrix stages of the others
        while ((int)ctx->lanes.size() < ndev - 1) {
            gwt_ctx::Lane ln;
            ck(cudaStreamCreateWithFlags(&ln.st, cudaStreamNonBlocking), "cudaStreamCreate");
            ck(cudaEventCreateWithFlags(&ln.ev, cudaEventDisableTiming), "cudaEventCreate");
            ctx->lanes.push_back(ln);
        }
        auto lane_st = [&](int l) { return l == 0 ? ctx->stream : ctx->lanes[l - 1].st; };
        ck(cudaEventRecord(ctx->ev[10], ctx->stream), "cudaEventRecord");
        for (int l = 1; l < ndev; ++l) ck(cudaStreamWaitEvent(lane_st(l), ctx->ev[10], 0), "cudaStreamWaitEvent");
        const int64_t cg = (ngroups + ndev - 1) / ndev;
        double dr = 0, dp = 0, ds = 0;
        StageEvents sev;
        for (int64_t c = 0, g0 = 0; g0 < ngroups; ++c, g0 += cg) {
            const int l = (int)c;
            const int64_t G = std::min(cg, ngroups - g0);
            sinr_device<T>(ctx, l, lane_st(l), t, topo, G, (const char*)Cf + cs * g0 * c_g, (const char*)Gc + cs * g0 * g_g,
                           tau + g0 * links * t.P, freqs, nullptr, F, scope, sinr + g0 * F * users * t.L,
                           signal + g0 * F * users * t.L, status + g0 * F * users, false, dr, dp, ds, &sev);
        }
        for (int l = 1; l < ndev; ++l) {
            ck(cudaEventRecord(ctx->lanes[l - 1].ev, lane_st(l)), "cudaEventRecord");
            ck(cudaStreamWaitEvent(ctx->stream, ctx->lanes[l - 1].ev, 0), "cudaStreamWaitEvent");
        }
        tm.mark(6);
        ck(cudaStreamSynchronize(ctx->stream), "sync");
        sev.resolve(dr, dp, ds);
        std::fill(ctx->stage_ms, ctx->stage_ms + 8, 0.0);
        ctx->stage_ms[0] = tm.between(0, 6);
        // per-stage kernel time summed over the lanes (the lanes overlap, so the sum exceeds stage_ms[0])
        ctx->stage_ms[4] = dr;
        ctx->stage_ms[5] = dp;
        ctx->stage_ms[6] = ds;
        return;
    }
    if (mem == GWT_MEM_HOST && nch > 1 && ctx->opt.sinr_copy_streams) {
        // host buffers: group chunks flow through three engines — one H2D copy stream, NS compute lanes,
        // one D2H copy stream — chained by per-chunk events, so PCIe traffic in both directions overlaps
        // the kernels while the kernels keep the device-resident 2-lane concurrency (4 compute lanes of
        // the older scheme contended: 0.38 vs 0.36 ms device time on C2)
        const int NS = (int)std::min<int64_t>(ctx->opt.sinr_lanes > 0 ? ctx->opt.sinr_lanes : (tc_shape ? 1 : 2), nch);
        while ((int)ctx->lanes.size() < NS - 1) {
            gwt_ctx::Lane ln;
            ck(cudaStreamCreateWithFlags(&ln.st, cudaStreamNonBlocking), "cudaStreamCreate");
            ck(cudaEventCreateWithFlags(&ln.ev, cudaEventDisableTiming), "cudaEventCreate");
            ctx->lanes.push_back(ln);
        }
        ctx->copy_streams();
        cudaStream_t hs = ctx->cp_h2d, ds2 = ctx->cp_d2h;
        auto lane_st = [&](int l) { return l == 0 ? ctx->stream : ctx->lanes[l - 1].st; };
        ck(cudaEventRecord(ctx->ev[10], ctx->stream), "cudaEventRecord");
        ck(cudaStreamWaitEvent(hs, ctx->ev[10], 0), "cudaStreamWaitEvent");
        for (int l = 1; l < NS; ++l) ck(cudaStreamWaitEvent(lane_st(l), ctx->ev[10], 0), "cudaStreamWaitEvent");
        // whole-call device buffers (inputs ~13 MB, outputs ~10 MB at C2): chunks are offsets, no reuse
        void* cdv = ctx->ws(WS_C, cs * ngroups * c_g);
        void* gdv = ctx->ws(WS_G, cs * ngroups * g_g);
        double* tav = nullptr;
        double* frv = nullptr;
        char* cov = nullptr;
        if (coeffs) cov = (char*)ctx->ws(WS_COEF, cs * ngroups * F * links * t.P);
        else {
            tav = (double*)ctx->ws(WS_TAU, 8 * ngroups * links * t.P);
            frv = (double*)ctx->ws(WS_FREQ, 8 * F);
            ck(cudaMemcpyAsync(frv, freqs, 8 * F, cudaMemcpyHostToDevice, hs), "H2D freqs");
        }
        double* so = (double*)ctx->ws(WS_SINR, 8 * out_rows * t.L);
        double* sg = (double*)ctx->ws(WS_SIG, 8 * out_rows * t.L);
        int* stt = (int*)ctx->ws(WS_STATUS, 4 * out_rows);
        const int64_t cg = (ngroups + nch - 1) / nch;
        double dr = 0, dp = 0, ds = 0;
        int64_t nchunks = 0;
        for (int64_t c = 0, g0 = 0; g0 < ngroups; ++c, g0 += cg) {
            const int l = (int)(c % NS);
            cudaStream_t s2 = lane_st(l);
            const int64_t G = std::min(cg, ngroups - g0), rows = G * F * users, r0 = g0 * F * users;
            char* cdc = (char*)cdv + cs * g0 * c_g;
            char* gdc = (char*)gdv + cs * g0 * g_g;
            ck(cudaMemcpyAsync(cdc, (const char*)Cf + cs * g0 * c_g, cs * G * c_g, cudaMemcpyHostToDevice, hs), "H2D C");
            ck(cudaMemcpyAsync(gdc, (const char*)Gc + cs * g0 * g_g, cs * G * g_g, cudaMemcpyHostToDevice, hs), "H2D G");
            if (coeffs)
                ck(cudaMemcpyAsync(cov + cs * g0 * F * links * t.P, (const char*)coeffs + cs * g0 * F * links * t.P,
                                   cs * G * F * links * t.P, cudaMemcpyHostToDevice, hs), "H2D coeffs");
            else
                ck(cudaMemcpyAsync(tav + g0 * links * t.P, tau + g0 * links * t.P, 8 * G * links * t.P,
                                   cudaMemcpyHostToDevice, hs), "H2D tau");
            cudaEvent_t eh = ctx->chunk_event(2 * c), ek = ctx->chunk_event(2 * c + 1);
            ck(cudaEventRecord(eh, hs), "cudaEventRecord");
            ck(cudaStreamWaitEvent(s2, eh, 0), "cudaStreamWaitEvent");
            sinr_device<T>(ctx, l, s2, t, topo, G, cdc, gdc, coeffs ? nullptr : tav + g0 * links * t.P, frv,
                           coeffs ? cov + cs * g0 * F * links * t.P : nullptr, F, scope, so + r0 * t.L, sg + r0 * t.L,
                           stt + r0, false, dr, dp, ds);
            ck(cudaEventRecord(ek, s2), "cudaEventRecord");
            ck(cudaStreamWaitEvent(ds2, ek, 0), "cudaStreamWaitEvent");
            ck(cudaMemcpyAsync(sinr + r0 * t.L, so + r0 * t.L, 8 * rows * t.L, cudaMemcpyDeviceToHost, ds2), "D2H sinr");
            ck(cudaMemcpyAsync(signal + r0 * t.L, sg + r0 * t.L, 8 * rows * t.L, cudaMemcpyDeviceToHost, ds2), "D2H signal");
            ck(cudaMemcpyAsync(status + r0, stt + r0, 4 * rows, cudaMemcpyDeviceToHost, ds2), "D2H status");
            ++nchunks;
        }
        cudaEvent_t ed = ctx->chunk_event(2 * nchunks);
        ck(cudaEventRecord(ed, ds2), "cudaEventRecord");
        ck(cudaStreamWaitEvent(ctx->stream, ed, 0), "cudaStreamWaitEvent");
        for (int l = 1; l < NS; ++l) {
            ck(cudaEventRecord(ctx->lanes[l - 1].ev, lane_st(l)), "cudaEventRecord");
            ck(cudaStreamWaitEvent(ctx->stream, ctx->lanes[l - 1].ev, 0), "cudaStreamWaitEvent");
        }
        tm.mark(6);
        ck(cudaStreamSynchronize(ctx->stream), "sync");
        std::fill(ctx->stage_ms, ctx->stage_ms + 8, 0.0);
        ctx->stage_ms[0] = tm.between(0, 6);
        return;
    }
    if (mem == GWT_MEM_HOST && nch > 1) {
        // host buffers: 4 group chunks on 4 stream lanes (GWT_SINR_PIPELINE / GWT_SINR_LANES), each chunk H2D -> device
        // pipeline -> D2H on its lane, so copies in both directions overlap the other chunks' kernels
        const int NS = (int)std::min<int64_t>(ctx->opt.sinr_lanes > 0 ? ctx->opt.sinr_lanes : 4, nch);
        while ((int)ctx->lanes.size() < NS - 1) {
            gwt_ctx::Lane ln;
            ck(cudaStreamCreateWithFlags(&ln.st, cudaStreamNonBlocking), "cudaStreamCreate");
            ck(cudaEventCreateWithFlags(&ln.ev, cudaEventDisableTiming), "cudaEventCreate");
            ctx->lanes.push_back(ln);
        }
        auto lane_st = [&](int l) { return l == 0 ? ctx->stream : ctx->lanes[l - 1].st; };
        ck(cudaEventRecord(ctx->ev[10], ctx->stream), "cudaEventRecord");
        for (int l = 1; l < NS; ++l) ck(cudaStreamWaitEvent(lane_st(l), ctx->ev[10], 0), "cudaStreamWaitEvent");
        const int64_t cg = (ngroups + nch - 1) / nch;
        double dr = 0, dp = 0, ds = 0;
        for (int64_t c = 0, g0 = 0; g0 < ngroups; ++c, g0 += cg) {
            const int l = (int)(c % NS);
            cudaStream_t s2 = lane_st(l);
            const int64_t G = std::min(cg, ngroups - g0), rows = G * F * users;
            void* cdv = ctx->lws(l, WS_C, cs * cg * c_g);
            void* gdv = ctx->lws(l, WS_G, cs * cg * g_g);
            ck(cudaMemcpyAsync(cdv, (const char*)Cf + cs * g0 * c_g, cs * G * c_g, cudaMemcpyHostToDevice, s2), "H2D C");
            ck(cudaMemcpyAsync(gdv, (const char*)Gc + cs * g0 * g_g, cs * G * g_g, cudaMemcpyHostToDevice, s2), "H2D G");
            const void* codv = nullptr;
            const double *tav = nullptr, *frv = nullptr;
            if (coeffs) {
                void* co = ctx->lws(l, WS_COEF, cs * cg * F * links * t.P);
                ck(cudaMemcpyAsync(co, (const char*)coeffs + cs * g0 * F * links * t.P, cs * G * F * links * t.P,
                                   cudaMemcpyHostToDevice, s2), "H2D coeffs");
                codv = co;
            } else {
                double* ta = (double*)ctx->lws(l, WS_TAU, 8 * cg * links * t.P);
                double* fr = (double*)ctx->lws(l, WS_FREQ, 8 * F);
                ck(cudaMemcpyAsync(ta, tau + g0 * links * t.P, 8 * G * links * t.P, cudaMemcpyHostToDevice, s2), "H2D tau");
                ck(cudaMemcpyAsync(fr, freqs, 8 * F, cudaMemcpyHostToDevice, s2), "H2D freqs");
                tav = ta;
                frv = fr;
            }
            double* so = (double*)ctx->lws(l, WS_SINR, 8 * cg * F * users * t.L);
            double* sg = (double*)ctx->lws(l, WS_SIG, 8 * cg * F * users * t.L);
            int* stt = (int*)ctx->lws(l, WS_STATUS, 4 * cg * F * users);
            sinr_device<T>(ctx, l, s2, t, topo, G, cdv, gdv, tav, frv, codv, F, scope, so, sg, stt, false, dr, dp, ds);
            ck(cudaMemcpyAsync(sinr + g0 * F * users * t.L, so, 8 * rows * t.L, cudaMemcpyDeviceToHost, s2), "D2H sinr");
            ck(cudaMemcpyAsync(signal + g0 * F * users * t.L, sg, 8 * rows * t.L, cudaMemcpyDeviceToHost, s2), "D2H signal");
            ck(cudaMemcpyAsync(status + g0 * F * users, stt, 4 * rows, cudaMemcpyDeviceToHost, s2), "D2H status");
        }
        for (int l = 1; l < NS; ++l) {
            ck(cudaEventRecord(ctx->lanes[l - 1].ev, lane_st(l)), "cudaEventRecord");
            ck(cudaStreamWaitEvent(ctx->stream, ctx->lanes[l - 1].ev, 0), "cudaStreamWaitEvent");
        }
        tm.mark(6);
        ck(cudaStreamSynchronize(ctx->stream), "sync");
        std::fill(ctx->stage_ms, ctx->stage_ms + 8, 0.0);
        ctx->stage_ms[0] = tm.between(0, 6);
        return;
    }
    if (mem == GWT_MEM_HOST) {
        tm.mark(4);
        void* c = ctx->ws(WS_C, cs * ngroups * c_g);
        void* g = ctx->ws(WS_G, cs * ngroups * g_g);
        ck(cudaMemcpyAsync(c, Cf, cs * ngroups * c_g, cudaMemcpyHostToDevice, st), "H2D C");
        ck(cudaMemcpyAsync(g, Gc, cs * ngroups * g_g, cudaMemcpyHostToDevice, st), "H2D G");
        Cd = c;
        Gd = g;
        if (coeffs) {
            void* co = ctx->ws(WS_COEF, cs * ngroups * F * links * t.P);
            ck(cudaMemcpyAsync(co, coeffs, cs * ngroups * F * links * t.P, cudaMemcpyHostToDevice, st), "H2D coeffs");
            cod = co;
        } else {
            double* ta = (double*)ctx->ws(WS_TAU, 8 * ngroups * links * t.P);
            double* fr = (double*)ctx->ws(WS_FREQ, 8 * F);
            ck(cudaMemcpyAsync(ta, tau, 8 * ngroups * links * t.P, cudaMemcpyHostToDevice, st), "H2D tau");
            ck(cudaMemcpyAsync(fr, freqs, 8 * F, cudaMemcpyHostToDevice, st), "H2D freqs");
            taud = ta;
            fd = fr;
        }
        sd = (double*)ctx->ws(WS_SINR, 8 * out_rows * t.L);
        sgd = (double*)ctx->ws(WS_SIG, 8 * out_rows * t.L);
        std_ = (int*)ctx->ws(WS_STATUS, 4 * out_rows);
        tm.mark(5);
    }
    double ms_r = 0, ms_p = 0, ms_s = 0;
    sinr_device<T>(ctx, 0, st, t, topo, ngroups, Cd, Gd, taud, fd, cod, F, scope, sd, sgd, std_, true, ms_r, ms_p, ms_s);
    if (mem == GWT_MEM_HOST) {
        tm.mark(12);
        ck(cudaMemcpyAsync(sinr, sd, 8 * out_rows * t.L, cudaMemcpyDeviceToHost, st), "D2H sinr");
        ck(cudaMemcpyAsync(signal, sgd, 8 * out_rows * t.L, cudaMemcpyDeviceToHost, st), "D2H signal");
        ck(cudaMemcpyAsync(status, std_, 4 * out_rows, cudaMemcpyDeviceToHost, st), "D2H status");
        tm.mark(13);
    }
    tm.mark(6);
    ck(cudaStreamSynchronize(st), "sync");
    if (mem == GWT_MEM_HOST) copy_ms = tm.between(4, 5) + tm.between(12, 13);
    std::fill(ctx->stage_ms, ctx->stage_ms + 8, 0.0);
    ctx->stage_ms[0] = tm.between(0, 6);
    ctx->stage_ms[4] = ms_r;
    ctx->stage_ms[5] = ms_p;
    ctx->stage_ms[6] = ms_s;
    ctx->stage_ms[7] = copy_ms;
}

void ledger_for(const gwt_topology& tp, const gwt_ranks& r, int path, gwt_ledger* out) {  // sinr.cpp:353-382
    const int64_t J = tp.num_cells, K = tp.users_per_cell, M = tp.rx_antennas, N = tp.tx_antennas, P = tp.num_taps;
    const int64_t L = tp.num_streams, m = r.m, n = r.n, p = r.p;
    const int64_t links = J * J * K, users = J * K;
    if (path == 0) {
        out->reconstruct = links * (M * N * P);
        out->precoder = users * (M * N * L);
        out->covariance = users * users * (M * N * L + M * M * L);
        out->inverse = users * (M * M * M);
        out->filter = users * (M * M * L);
        out->sinr = users * L * (M * M + 2 * M);
    } else {
        out->reconstruct = links * (m * n * p + P * p);
        out->precoder = users * (m * n * L);
        out->covariance = users * users * (m * n * L + m * m * L);
        out->inverse = users * (2 * m * m * m);
        out->filter = users * (m * m * L + m * L);
        out->sinr = users * L * (m * m + 2 * m);
    }
}

}  // namespace

// ---------------------------------------------------------------------------
extern "C" {

int gwt_ctx_create(gwt_ctx** out, int device) {
    if (!out) return GWT_INVALID_ARGUMENT;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return GWT_NO_DEVICE;
    if (device < 0 || device >= n) return GWT_INVALID_ARGUMENT;
    gwt_ctx* c = new gwt_ctx();
    c->device = device;
    c->opt.read();
    if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete c;
        return GWT_CUDA_ERROR;
    }
    c->stream = c->own_stream;
    *out = c;
    return GWT_OK;
}

void gwt_ctx_destroy(gwt_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto& s : ctx->slots)
        if (s.p) cudaFree(s.p);
    for (auto& ln : ctx->lanes) {
        cudaStreamSynchronize(ln.st);
        for (auto& s : ln.slots)
            if (s.p) cudaFree(s.p);
        cudaStreamDestroy(ln.st);
        cudaEventDestroy(ln.ev);
    }
    for (auto& e : ctx->ev)
        if (e) cudaEventDestroy(e);
    for (auto* p : ctx->pinned)
        if (p) cudaFreeHost(p);
    for (cudaStream_t s : {ctx->cp_h2d, ctx->cp_d2h})
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    for (auto e : ctx->chev) cudaEventDestroy(e);
    for (int l = 0; l < 8; ++l)
        if (ctx->side[l]) {
            cudaStreamSynchronize(ctx->side[l]);
            cudaStreamDestroy(ctx->side[l]);
            for (auto& e : ctx->side_ev[l]) cudaEventDestroy(e);
        }
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
}

const char* gwt_last_error(const gwt_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "null gwt_ctx"; }

int gwt_ctx_set_stream(gwt_ctx* ctx, void* stream) {
    if (!ctx) return GWT_INVALID_ARGUMENT;
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
    return GWT_OK;
}

int64_t gwt_ctx_launch_count(const gwt_ctx* ctx) { return ctx ? ctx->launches : 0; }

int gwt_ctx_stage_times(const gwt_ctx* ctx, double* ms8) {
    if (!ctx || !ms8) return GWT_INVALID_ARGUMENT;
    std::memcpy(ms8, ctx->stage_ms, sizeof(ctx->stage_ms));
    return GWT_OK;
}

int gwt_groupwise_solve(gwt_ctx* ctx, const gwt_topology* topo, const gwt_ranks* ranks, int64_t ngroups,
                        gwt_dtype dtype, gwt_mem mem, const void* X, int32_t sweeps, uint32_t flags, void* A, void* B,
                        void* C, void* G, double* trace, int32_t* iters, double* energy) {
    return guarded(ctx, [&] {
        if (!topo || !ranks) invalid("groupwise_solve: null topology/ranks");
        if (dtype == GWT_C64)
            groupwise_solve_impl<float>(ctx, topo, ranks, ngroups, mem, X, sweeps, flags, A, B, C, G, trace, iters, energy);
        else
            groupwise_solve_impl<double>(ctx, topo, ranks, ngroups, mem, X, sweeps, flags, A, B, C, G, trace, iters, energy);
    });
}

int gwt_sinr_compressed(gwt_ctx* ctx, const gwt_topology* topo, const gwt_ranks* ranks, int64_t ngroups,
                        gwt_dtype dtype, gwt_mem mem, const void* C, const void* G, const double* tau,
                        const double* freqs, int64_t F, gwt_scope scope, double* sinr, double* signal,
                        int32_t* status, gwt_ledger* ledger) {
    return guarded(ctx, [&] {
        if (!topo || !ranks) invalid("sinr: null topology/ranks");
        validate_sinr(*topo, *ranks, scope);
        if (F < 0 || ngroups < 0) invalid("sinr: negative batch size");
        if (ledger) {
            ledger_for(*topo, *ranks, 1, ledger);
            const int64_t mul = F * ngroups;
            ledger->reconstruct *= mul; ledger->precoder *= mul; ledger->covariance *= mul;
            ledger->inverse *= mul; ledger->filter *= mul; ledger->sinr *= mul;
        }
        if (F == 0 || ngroups == 0) return;
        if (dtype == GWT_C64)
            sinr_impl<float>(ctx, topo, ranks, ngroups, mem, C, G, tau, freqs, nullptr, F, scope, sinr, signal, status);
        else
            sinr_impl<double>(ctx, topo, ranks, ngroups, mem, C, G, tau, freqs, nullptr, F, scope, sinr, signal, status);
    });
}

int gwt_sinr_compressed_coeffs(gwt_ctx* ctx, const gwt_topology* topo, const gwt_ranks* ranks, int64_t ngroups,
                               gwt_dtype dtype, gwt_mem mem, const void* C, const void* G, const void* coeffs,
                               int64_t F, gwt_scope scope, double* sinr, double* signal, int32_t* status,
                               gwt_ledger* ledger) {
    return guarded(ctx, [&] {
        if (!topo || !ranks) invalid("sinr: null topology/ranks");
        validate_sinr(*topo, *ranks, scope);
        if (!coeffs) invalid("assemble_all_compressed: coefficient grid does not match cores");
        if (ledger) {
            ledger_for(*topo, *ranks, 1, ledger);
            const int64_t mul = F * ngroups;
            ledger->reconstruct *= mul; ledger->precoder *= mul; ledger->covariance *= mul;
            ledger->inverse *= mul; ledger->filter *= mul; ledger->sinr *= mul;
        }
        if (F == 0 || ngroups == 0) return;
        if (dtype == GWT_C64)
            sinr_impl<float>(ctx, topo, ranks, ngroups, mem, C, G, nullptr, nullptr, coeffs, F, scope, sinr, signal, status);
        else
            sinr_impl<double>(ctx, topo, ranks, ngroups, mem, C, G, nullptr, nullptr, coeffs, F, scope, sinr, signal, status);
    });
}

// Full-size SINR (run_full_pipeline, sinr.cpp:287-294 / evaluate_assembled :259-285): H(f) = X x3 c(f)^*
// is the compressed rebuild with cores = X and delay factor = I_P, so the same kernels run with
// ranks (M, N, P); precoder/covariance/filter/SINR act on the M x N channels.
int gwt_sinr_full(gwt_ctx* ctx, const gwt_topology* topo, int64_t ngroups, gwt_dtype dtype, gwt_mem mem,
                  const void* X, const double* tau, const double* freqs, const void* coeffs, int64_t F,
                  gwt_scope scope, double* sinr, double* signal, int32_t* status, gwt_ledger* ledger) {
    return guarded(ctx, [&] {
        if (!topo) invalid("sinr_full: null topology");
        validate_topology(*topo);
        if (topo->rx_antennas > 8)
            invalid("sinr_full: receive antennas M > 8 are not supported by the B200 small-matrix kernel");
        gwt_ranks r{topo->rx_antennas, topo->tx_antennas, topo->num_taps};
        if (ledger) {
            ledger_for(*topo, r, 0, ledger);
            const int64_t mul = F * ngroups;
            ledger->reconstruct *= mul; ledger->precoder *= mul; ledger->covariance *= mul;
            ledger->inverse *= mul; ledger->filter *= mul; ledger->sinr *= mul;
        }
        if (F == 0 || ngroups == 0) return;
        const Topo t = mk_topo(*topo, r);
        const int links = t.links();
        const size_t cs = csize(dtype);
        const int64_t x_g = (int64_t)links * t.M * t.N * t.P;
        cudaStream_t st = ctx->stream;
        // identity delay factors, device resident
        std::vector<unsigned char> eye(cs * (size_t)ngroups * links * t.P * t.P, 0);
        for (int64_t gl = 0; gl < ngroups * links; ++gl)
            for (int q = 0; q < t.P; ++q) {
                unsigned char* e = eye.data() + cs * ((size_t)gl * t.P * t.P + (size_t)q * t.P + q);
                if (dtype == GWT_C64) { const float one = 1.0f; std::memcpy(e, &one, 4); }
                else { const double one = 1.0; std::memcpy(e, &one, 8); }
            }
        void* Cid = ctx->ws(WS_MISC, eye.size());
        ck(cudaMemcpyAsync(Cid, eye.data(), eye.size(), cudaMemcpyHostToDevice, st), "H2D identity");
        const void* Xd = X;
        if (mem == GWT_MEM_HOST) {
            void* xb = ctx->ws(WS_X, cs * ngroups * x_g);
            ck(cudaMemcpyAsync(xb, X, cs * ngroups * x_g, cudaMemcpyHostToDevice, st), "H2D X");
            Xd = xb;
        }
        ck(cudaStreamSynchronize(st), "sync");
        // inputs now on device; run the compressed machinery on (C = I, G = X) with device cores
        const gwt_mem inner_mem = GWT_MEM_DEVICE;
        if (mem == GWT_MEM_HOST) {
            // copy tau/freqs/coeffs and outputs through the host-mode path of sinr_impl: the cores/delay are
            // already device pointers, so stage the small host inputs here
            const int64_t out_rows = ngroups * F * t.users();
            double* sd = (double*)ctx->ws(WS_SINR, 8 * out_rows * t.L);
            double* sgd = (double*)ctx->ws(WS_SIG, 8 * out_rows * t.L);
            int* std_ = (int*)ctx->ws(WS_STATUS, 4 * out_rows);
            const double *taud = nullptr, *fd = nullptr;
            const void* cod = nullptr;
            if (coeffs) {
                void* co = ctx->ws(WS_COEF, cs * ngroups * F * links * t.P);
                ck(cudaMemcpyAsync(co, coeffs, cs * ngroups * F * links * t.P, cudaMemcpyHostToDevice, st), "H2D");
                cod = co;
            } else {
                double* ta = (double*)ctx->ws(WS_TAU, 8 * ngroups * links * t.P);
                double* fr = (double*)ctx->ws(WS_FREQ, 8 * F);
                ck(cudaMemcpyAsync(ta, tau, 8 * ngroups * links * t.P, cudaMemcpyHostToDevice, st), "H2D");
                ck(cudaMemcpyAsync(fr, freqs, 8 * F, cudaMemcpyHostToDevice, st), "H2D");
                taud = ta;
                fd = fr;
            }
            if (dtype == GWT_C64)
                sinr_impl<float>(ctx, topo, &r, ngroups, inner_mem, Cid, Xd, taud, fd, cod, F, scope, sd, sgd, std_);
            else
                sinr_impl<double>(ctx, topo, &r, ngroups, inner_mem, Cid, Xd, taud, fd, cod, F, scope, sd, sgd, std_);
            ck(cudaMemcpyAsync(sinr, sd, 8 * out_rows * t.L, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaMemcpyAsync(signal, sgd, 8 * out_rows * t.L, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaMemcpyAsync(status, std_, 4 * out_rows, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaStreamSynchronize(st), "sync");
        } else {
            if (dtype == GWT_C64)
                sinr_impl<float>(ctx, topo, &r, ngroups, inner_mem, Cid, Xd, tau, freqs, coeffs, F, scope, sinr, signal,
                                 status);
            else
                sinr_impl<double>(ctx, topo, &r, ngroups, inner_mem, Cid, Xd, tau, freqs, coeffs, F, scope, sinr,
                                  signal, status);
        }
    });
}

int gwt_assemble_compressed(gwt_ctx* ctx, const gwt_topology* topo, const gwt_ranks* ranks, int64_t ngroups,
                            gwt_dtype dtype, gwt_mem mem, const void* C, const void* G, const double* tau,
                            const double* freqs, const void* coeffs, int64_t F, void* H) {
    return guarded(ctx, [&] {
        if (!topo || !ranks) invalid("assemble_compressed: null topology/ranks");
        if (ranks->m < 1 || ranks->n < 1 || ranks->p < 1 || ranks->p > topo->num_taps)
            invalid("assemble_channel_compressed: delay factor has " + std::to_string(topo->num_taps) +
                    " rows but core mode-3 size is " + std::to_string(ranks->p));
        if (F == 0 || ngroups == 0) return;
        const Topo t = mk_topo(*topo, *ranks);
        const size_t cs = csize(dtype);
        const int links = t.links();
        const int64_t c_g = (int64_t)links * t.P * t.p, g_g = (int64_t)links * t.m * t.n * t.p;
        const int64_t h_bytes = cs * ngroups * F * links * t.m * t.n;
        const void *Cd = C, *Gd = G, *cod = coeffs;
        const double *taud = tau, *fd = freqs;
        void* Hd = H;
        cudaStream_t st = ctx->stream;
        if (mem == GWT_MEM_HOST) {
            void* c = ctx->ws(WS_C, cs * ngroups * c_g);
            void* g = ctx->ws(WS_G, cs * ngroups * g_g);
            ck(cudaMemcpyAsync(c, C, cs * ngroups * c_g, cudaMemcpyHostToDevice, st), "H2D");
            ck(cudaMemcpyAsync(g, G, cs * ngroups * g_g, cudaMemcpyHostToDevice, st), "H2D");
            Cd = c;
            Gd = g;
            if (coeffs) {
                void* co = ctx->ws(WS_COEF, cs * ngroups * F * links * t.P);
                ck(cudaMemcpyAsync(co, coeffs, cs * ngroups * F * links * t.P, cudaMemcpyHostToDevice, st), "H2D");
                cod = co;
            } else {
                double* ta = (double*)ctx->ws(WS_TAU, 8 * ngroups * links * t.P);
                double* fr = (double*)ctx->ws(WS_FREQ, 8 * F);
                ck(cudaMemcpyAsync(ta, tau, 8 * ngroups * links * t.P, cudaMemcpyHostToDevice, st), "H2D");
                ck(cudaMemcpyAsync(fr, freqs, 8 * F, cudaMemcpyHostToDevice, st), "H2D");
                taud = ta;
                fd = fr;
            }
            Hd = ctx->ws(WS_H, h_bytes);
        }
        if (dtype == GWT_C64)
            ctx->launched(launch_rebuild<float>(t, (int)ngroups, (int)F, 0, F, Cd, Gd, taud, fd, cod, Hd, st));
        else
            ctx->launched(launch_rebuild<double>(t, (int)ngroups, (int)F, 0, F, Cd, Gd, taud, fd, cod, Hd, st));
        if (mem == GWT_MEM_HOST) ck(cudaMemcpyAsync(H, Hd, h_bytes, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
    });
}

int gwt_leading_eigenvectors(gwt_ctx* ctx, int32_t n, int32_t count, int64_t batch, gwt_dtype dtype, gwt_mem mem,
                             const void* H, void* out, double* evals) {
    return guarded(ctx, [&] {
        if (n < 1) invalid("leading_eigenvectors: matrix is not square");
        if (count < 1 || count > n)  // linalg.cpp:28-32
            invalid("leading_eigenvectors: count " + std::to_string(count) + " out of range for size " + std::to_string(n));
        if (n > 256) invalid("leading_eigenvectors: sizes above 256 are not supported by the batched eigensolver");
        if (batch == 0) return;
        const size_t cs = csize(dtype);
        cudaStream_t st = ctx->stream;
        const void* Hd = H;
        void* Od = out;
        double* Ed = evals;
        if (mem == GWT_MEM_HOST) {
            void* h = ctx->ws(WS_GRAM, cs * batch * n * n);
            ck(cudaMemcpyAsync(h, H, cs * batch * n * n, cudaMemcpyHostToDevice, st), "H2D");
            Hd = h;
            Od = ctx->ws(WS_POOL, cs * batch * n * count);
            Ed = evals ? (double*)ctx->ws(WS_MISC, 8 * batch * count) : nullptr;
        }
        double2* eA = (double2*)ctx->ws(WS_EIGA, 16 * batch * heev_ws_a_elems(n));
        double* eZ = (double*)ctx->ws(WS_EIGZ, 8 * batch * heev_ws_z_elems(n, count));
        double2* eX = (double2*)ctx->ws(WS_EIGX, 16 * batch * n * count);
        int* fl = (int*)ctx->ws(WS_FAIL, 4);
        ck(cudaMemsetAsync(fl, 0, 4, st), "memset");
        if (dtype == GWT_C64)
            ctx->launched(launch_heev_topk<float>(n, count, batch, Hd, Od, Ed, eA, eZ, eX, fl, st));
        else
            ctx->launched(launch_heev_topk<double>(n, count, batch, Hd, Od, Ed, eA, eZ, eX, fl, st));
        int hf = 0;
        ck(cudaMemcpyAsync(&hf, fl, 4, cudaMemcpyDeviceToHost, st), "D2H");
        if (mem == GWT_MEM_HOST) {
            ck(cudaMemcpyAsync(out, Od, cs * batch * n * count, cudaMemcpyDeviceToHost, st), "D2H");
            if (evals) ck(cudaMemcpyAsync(evals, Ed, 8 * batch * count, cudaMemcpyDeviceToHost, st), "D2H");
        }
        ck(cudaStreamSynchronize(st), "sync");
        if (hf) fail(GWT_RUNTIME_ERROR, "leading_eigenvectors: eigendecomposition failed");
    });
}

int gwt_hpd_solve(gwt_ctx* ctx, int32_t m, int32_t nrhs, int64_t batch, gwt_mem mem, const void* Q, const void* B,
                  int32_t check_cond, void* X, int32_t* status) {
    return guarded(ctx, [&] {
        if (m < 1 || nrhs < 0 || batch < 0) invalid("hpd_solve: bad covariance or right-hand-side size");
        if (batch == 0 || nrhs == 0) return;
        cudaStream_t st = ctx->stream;
        const size_t qb = 16 * (size_t)batch * m * m, bb = 16 * (size_t)batch * m * nrhs;
        const void* Qd = Q;
        const void* Bd = B;
        void* Xd = X;
        int* Sd = (int*)status;
        if (mem == GWT_MEM_HOST) {
            void* q = ctx->ws(WS_GRAM, qb);
            void* r = ctx->ws(WS_EIGX, bb);
            ck(cudaMemcpyAsync(q, Q, qb, cudaMemcpyHostToDevice, st), "H2D");
            ck(cudaMemcpyAsync(r, B, bb, cudaMemcpyHostToDevice, st), "H2D");
            Qd = q;
            Bd = r;
            Xd = ctx->ws(WS_POOL, bb);
            Sd = (int*)ctx->ws(WS_STATUS, 4 * batch);
        }
        void* Lw = ctx->ws(WS_EIGA, qb);
        ctx->launched(launch_hpd_solve(m, nrhs, batch, Qd, Bd, check_cond, Lw, Xd, Sd, st));
        if (mem == GWT_MEM_HOST) {
            ck(cudaMemcpyAsync(X, Xd, bb, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaMemcpyAsync(status, Sd, 4 * batch, cudaMemcpyDeviceToHost, st), "D2H");
        }
        ck(cudaStreamSynchronize(st), "sync");
    });
}

int gwt_reconstruct(gwt_ctx* ctx, const gwt_topology* topo, const gwt_ranks* ranks, int64_t ngroups, gwt_dtype dtype,
                    gwt_mem mem, const void* A, const void* B, const void* C, const void* G, void* X) {
    return guarded(ctx, [&] {
        if (!topo || !ranks) invalid("reconstruct: null topology/ranks");
        validate_ranks(*ranks, topo->rx_antennas, topo->tx_antennas, topo->num_taps);
        if (ngroups == 0) return;
        const Topo t = mk_topo(*topo, *ranks);
        const size_t cs = csize(dtype);
        const int links = t.links(), users = t.users();
        const int64_t a_g = (int64_t)users * t.M * t.m, b_g = (int64_t)t.J * t.N * t.n, c_g = (int64_t)links * t.P * t.p,
                      g_g = (int64_t)links * t.m * t.n * t.p, x_g = (int64_t)links * t.M * t.N * t.P;
        cudaStream_t st = ctx->stream;
        const void *Ad = A, *Bd = B, *Cd = C, *Gd = G;
        void* Xd = X;
        if (mem == GWT_MEM_HOST) {
            void* a = ctx->ws(WS_A, cs * ngroups * a_g);
            void* b = ctx->ws(WS_B, cs * ngroups * b_g);
            void* c = ctx->ws(WS_C, cs * ngroups * c_g);
            void* g = ctx->ws(WS_G, cs * ngroups * g_g);
            ck(cudaMemcpyAsync(a, A, cs * ngroups * a_g, cudaMemcpyHostToDevice, st), "H2D");
            ck(cudaMemcpyAsync(b, B, cs * ngroups * b_g, cudaMemcpyHostToDevice, st), "H2D");
            ck(cudaMemcpyAsync(c, C, cs * ngroups * c_g, cudaMemcpyHostToDevice, st), "H2D");
            ck(cudaMemcpyAsync(g, G, cs * ngroups * g_g, cudaMemcpyHostToDevice, st), "H2D");
            Ad = a; Bd = b; Cd = c; Gd = g;
            Xd = ctx->ws(WS_X, cs * ngroups * x_g);
        }
        void* T1 = ctx->ws(WS_Z, cs * ngroups * links * t.M * t.n * t.p);
        void* T2 = ctx->ws(WS_Z2, cs * ngroups * links * t.M * t.N * t.p);
        // X1 = G x1 A: rows = (d, r) fibers of length m; U(k=c, col=a) = A(a, c) = A[a + M c]
        GemmDesc d1{};
        d1.R = t.n * t.p; d1.S = 1; d1.Kd = t.m; d1.Cols = t.M;
        d1.in_item = (int64_t)t.m * t.n * t.p; d1.rs_in = t.m; d1.s_in = 0; d1.ks_in = 1;
        d1.out_item = (int64_t)t.M * t.n * t.p; d1.rs_out = t.M; d1.s_out = 0; d1.cs_out = 1; d1.fkind = FI_USER;
        d1.ublk = (int64_t)t.M * t.m; d1.uk = t.M; d1.ucol = 1; d1.uconj = 0;
        // X2 = X1 x2 B: rows (a, r); U(k=d, col=b) = B(b, d) = B[b + N d]
        GemmDesc d2{};
        d2.R = t.M; d2.S = t.p; d2.Kd = t.n; d2.Cols = t.N;
        d2.in_item = (int64_t)t.M * t.n * t.p; d2.rs_in = 1; d2.s_in = (int64_t)t.M * t.n; d2.ks_in = t.M;
        d2.out_item = (int64_t)t.M * t.N * t.p; d2.rs_out = 1; d2.s_out = (int64_t)t.M * t.N; d2.cs_out = t.M;
        d2.fkind = FI_BASE; d2.ublk = (int64_t)t.N * t.n; d2.uk = t.N; d2.ucol = 1; d2.uconj = 0;
        // X = X2 x3 C: rows (a,b); U(k=r, col=q) = C(q, r) = C[q + P r]
        GemmDesc d3{};
        d3.R = t.M * t.N; d3.S = 1; d3.Kd = t.p; d3.Cols = t.P;
        d3.in_item = (int64_t)t.M * t.N * t.p; d3.rs_in = 1; d3.s_in = 0; d3.ks_in = (int64_t)t.M * t.N;
        d3.out_item = x_g / links; d3.rs_out = 1; d3.s_out = 0; d3.cs_out = (int64_t)t.M * t.N;
        d3.fkind = FI_LINK; d3.ublk = (int64_t)t.P * t.p; d3.uk = t.P; d3.ucol = 1; d3.uconj = 0;
        auto run = [&](auto tag) {
            using T = decltype(tag);
            ctx->launched(launch_cgemm<T>(t, d1, ngroups, Gd, Ad, T1, st));
            ctx->launched(launch_cgemm<T>(t, d2, ngroups, T1, Bd, T2, st));
            ctx->launched(launch_cgemm<T>(t, d3, ngroups, T2, Cd, Xd, st));
        };
        if (dtype == GWT_C64) run(float{});
        else run(double{});
        if (mem == GWT_MEM_HOST) ck(cudaMemcpyAsync(X, Xd, cs * ngroups * x_g, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
    });
}

int gwt_mode_product(gwt_ctx* ctx, gwt_dtype dtype, gwt_mem mem, int64_t batch, int32_t d1, int32_t d2, int32_t d3,
                     const void* X, int32_t rows, const void* U, int32_t mode, void* Y) {
    return guarded(ctx, [&] {
        if (mode < 1 || mode > 3)  // tensor.cpp:96-101
            invalid("mode_product: mode must be 1, 2 or 3, got " + std::to_string(mode));
        if (d1 < 1 || d2 < 1 || d3 < 1 || rows < 1) invalid("mode_product: dims must be positive");
        if (batch == 0) return;
        const int dm = mode == 1 ? d1 : mode == 2 ? d2 : d3;
        const size_t cs = csize(dtype);
        const int o1 = mode == 1 ? rows : d1, o2 = mode == 2 ? rows : d2, o3 = mode == 3 ? rows : d3;
        const int64_t xn = (int64_t)d1 * d2 * d3, yn = (int64_t)o1 * o2 * o3;
        cudaStream_t st = ctx->stream;
        const void *Xd = X, *Ud = U;
        void* Yd = Y;
        if (mem == GWT_MEM_HOST) {
            void* x = ctx->ws(WS_X, cs * batch * xn);
            void* u = ctx->ws(WS_A, cs * (size_t)rows * dm);
            ck(cudaMemcpyAsync(x, X, cs * batch * xn, cudaMemcpyHostToDevice, st), "H2D");
            ck(cudaMemcpyAsync(u, U, cs * (size_t)rows * dm, cudaMemcpyHostToDevice, st), "H2D");
            Xd = x;
            Ud = u;
            Yd = ctx->ws(WS_Y1, cs * batch * yn);
        }
        // Out(row, col) = sum_k In(row, k) U(col, k): U read transposed, not conjugated, shared (FI_GROUP, 1 link)
        Topo t{1, 1, d1, d2, d3, 1, 1, 1, 1};
        GemmDesc d{};
        d.Kd = dm; d.Cols = rows; d.fkind = FI_GROUP; d.ublk = 0; d.uk = rows; d.ucol = 1; d.uconj = 0;
        d.in_item = xn; d.out_item = yn;
        if (mode == 1) {  // rows = fibers (i2,i3), k = i1 contiguous
            d.R = d2 * d3; d.S = 1; d.rs_in = d1; d.s_in = 0; d.ks_in = 1;
            d.rs_out = o1; d.s_out = 0; d.cs_out = 1;
        } else if (mode == 2) {  // rows = (i1, i3)
            d.R = d1; d.S = d3; d.rs_in = 1; d.s_in = (int64_t)d1 * d2; d.ks_in = d1;
            d.rs_out = 1; d.s_out = (int64_t)o1 * o2; d.cs_out = o1;
        } else {  // rows = (i1, i2) flattened, k = i3
            d.R = d1 * d2; d.S = 1; d.rs_in = 1; d.s_in = 0; d.ks_in = (int64_t)d1 * d2;
            d.rs_out = 1; d.s_out = 0; d.cs_out = (int64_t)d1 * d2;
        }
        // treat the batch as groups of one link each
        if (dtype == GWT_C64) ctx->launched(launch_cgemm<float>(t, d, batch, Xd, Ud, Yd, st));
        else ctx->launched(launch_cgemm<double>(t, d, batch, Xd, Ud, Yd, st));
        if (mem == GWT_MEM_HOST) ck(cudaMemcpyAsync(Y, Yd, cs * batch * yn, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
    });
}

int gwt_flop_estimate(const gwt_topology* topo, const gwt_ranks* ranks, int32_t path, gwt_ledger* out) {
    if (!topo || !ranks || !out) return GWT_INVALID_ARGUMENT;
    try {
        validate_topology(*topo);
        validate_ranks(*ranks, topo->rx_antennas, topo->tx_antennas, topo->num_taps);
    } catch (const GwtError& e) {
        return e.code;
    }
    ledger_for(*topo, *ranks, path, out);
    return GWT_OK;
}

}  // extern "C"
