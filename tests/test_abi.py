"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/gwt_b200.h declares, carries sm_100a code, and its host-side
pieces (closed-form ledger, input generator, validation) behave."""
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

import paper_2401_09792_b200 as gw
from paper_2401_09792_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "gwt_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|int64_t|const char\*)\s+(gwt_\w+)\(", txt, re.M)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_lib.EXPORTS) == syms


def test_library_is_sm100a():
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(gw.CudaError, match="no CPU fallback"):
        gw.Context(0)


def test_flop_estimate_validation():
    with pytest.raises(gw.InvalidArgument):
        gw.flop_estimate(gw.SystemTopology(2, 2, 4, 8, 5, 9, 0.1), gw.CompressionRanks(2, 2, 2))
    led = gw.flop_estimate(gw.SystemTopology(2, 2, 6, 8, 5, 2, 0.1), gw.CompressionRanks(4, 5, 3))
    links, users = 8, 4
    assert led.reconstruct == links * (4 * 5 * 3 + 5 * 3)
    assert led.covariance == users * users * (4 * 5 * 2 + 4 * 4 * 2)
    assert led.inverse == users * 2 * 4 ** 3


def test_generator_deterministic_and_chunkable():
    cfg = gw.CONFIGS["C2"]
    t = cfg.topology()
    X1, tau1 = gw.generate_channels(t, 4, seed=3)
    X2, tau2 = gw.generate_channels(t, 4, seed=3, nthreads=1)
    np.testing.assert_array_equal(X1, X2)
    a, ta = gw.generate_channels(t, 2, seed=3, group0=0)
    b, tb = gw.generate_channels(t, 2, seed=3, group0=2)
    np.testing.assert_array_equal(np.concatenate([a, b]), X1)
    np.testing.assert_array_equal(np.concatenate([ta, tb]), tau1)
    X3, _ = gw.generate_channels(t, 4, seed=4)
    assert not np.array_equal(X1, X3)
    x64, _ = gw.generate_channels(t, 4, seed=3, dtype=np.complex64)
    np.testing.assert_array_equal(x64, X1.astype(np.complex64))
    assert tau1.min() >= 0 and tau1.max() <= 1e-6


def test_generator_matches_baseline_spec():
    """One ray per tap: each slice has rank one and |X(:,:,q)|_F^2 = |a_q|^2 M N; PDP exp(-0.3 q)."""
    t = gw.SystemTopology(2, 4, 4, 64, 32, 4, 0.3)
    X, _ = gw.generate_channels(t, 32, seed=0)
    s = np.linalg.svd(np.transpose(X[0, 0], (0, 2, 1)), compute_uv=False)
    assert (s[:, 1] <= 1e-12 * s[:, 0]).all()
    power = np.mean(np.abs(X) ** 2, axis=(0, 1, 3, 4))  # per tap, averaged
    pdp = np.exp(-0.3 * np.arange(32))
    pdp /= pdp.sum()
    assert np.abs(power / pdp - 1).max() < 0.25  # 512 links per tap
    assert abs(power.sum() - 1.0) < 0.1


def test_configs_follow_baseline():
    c = gw.CONFIGS
    assert (c["C1"].M, c["C1"].N, c["C1"].P, c["C1"].G, c["C1"].groups, c["C1"].F) == (4, 32, 24, 8, 4, 64)
    assert (c["C4"].m, c["C4"].n, c["C4"].p, c["C4"].L) == (8, 64, 24, 8)
    for k in ("C1", "C2", "C3", "C4", "C5"):
        assert c[k].J * c[k].J * c[k].K == c[k].G


def test_cpp_dropin_library_exports_gwt_api():
    lib = os.path.join(ROOT, "paper_2401_09792_b200", "_build", "libgwtucker_b200.so")
    assert os.path.exists(lib)
    out = subprocess.run(["nm", "-DC", lib], capture_output=True, text=True).stdout
    for sym in ("gwt::groupwise_solve(", "gwt::run_compressed_pipeline(", "gwt::mode_product(", "gwt::hosvd(",
                "gwt::leading_eigenvectors(", "gwt::assemble_channel_compressed(", "gwt::reconstruct(",
                "gwt::flop_estimate(", "gwt::shared_solve(", "gwt::truncated_svd(", "gwt::precoder_compressed(",
                "gwt::covariance_compressed(", "gwt::woodbury_inverse_apply(", "gwt::filter_compressed(",
                "gwt::sinr_compressed(", "gwt::run_full_pipeline(", "gwt::update_rx_factor(",
                "gwt::tx_update_gram(", "gwt::update_delay_factor(", "gwt::individual_solve(",
                "gwt::evaluate_assembled(", "gwt::run_reconstructed_pipeline(", "gwt::filter_full("):
        assert sym in out, sym


def test_paper_metrics_reference_values():
    """R_s of the paper's Table 2 rows (test_metrics.cpp:38-57 pins these from the count formula)."""
    from paper_2401_09792_b200 import metrics
    t = gw.SystemTopology(21, 5, 64, 512, 401, 4, 0.1)
    assert abs(metrics.storage_ratio(t, gw.CompressionRanks(60, 230, 150)) - 6.1648) < 5e-5
    assert abs(metrics.storage_ratio(t, gw.CompressionRanks(60, 230, 150), "shared") - 6.1684) < 5e-5
    assert abs(metrics.storage_ratio(t, gw.CompressionRanks(60, 230, 150), "individual") - 5.8354) < 5e-5
    t10 = gw.SystemTopology(21, 10, 64, 512, 401, 4, 0.1)
    assert abs(metrics.storage_ratio(t10, gw.CompressionRanks(60, 270, 190)) - 4.1648) < 5e-5
    assert metrics.sinr_error([2.0, 4.0], [1.0, 5.0]) == 0.375
    with pytest.raises(gw.InvalidArgument, match="zero at flat index 1"):
        metrics.sinr_error([1.0, 0.0], [1.0, 1.0])
    assert metrics.speedup(6.0, 2.0) == 3.0


def test_runner_callsites_compile():
    """The reference control plane's hot-path call sites (runner.cpp:82-140: the model switch over
    groupwise/shared/individual solves, both compressed pipelines, the full-size comparator with its
    seconds/ledger fields, model_name/model_from_name) compile against the drop-in headers."""
    cxx = shutil.which("g++")
    if not cxx:
        pytest.skip("g++ not available")
    inc = os.path.join(ROOT, "paper_2401_09792_b200", "host", "include")
    src = os.path.join(ROOT, "tests", "cpp", "runner_callsites.cpp")
    r = subprocess.run([cxx, "-std=c++17", "-fsyntax-only", "-I", inc, src], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_model_name_roundtrip_cpp(tmp_path):
    """gwt::model_name / model_from_name of the C++ drop-in (decompose.cpp:42-56), including the error text."""
    cxx = shutil.which("g++")
    if not cxx:
        pytest.skip("g++ not available")
    inc = os.path.join(ROOT, "paper_2401_09792_b200", "host", "include")
    libdir = os.path.join(ROOT, "paper_2401_09792_b200", "_build")
    src = tmp_path / "m.cpp"
    src.write_text(r'''
#include <cstdio>
#include <stdexcept>
#include "gwtucker/decompose.hpp"
int main() {
    for (auto k : {gwt::ModelKind::individual, gwt::ModelKind::shared, gwt::ModelKind::groupwise})
        if (gwt::model_from_name(gwt::model_name(k)) != k) return 1;
    try { gwt::model_from_name("tucker"); } catch (const std::invalid_argument& e) { std::puts(e.what()); return 0; }
    return 2;
}''')
    exe = tmp_path / "m"
    r = subprocess.run([cxx, "-std=c++17", "-I", inc, str(src), "-o", str(exe), "-L", libdir, "-lgwtucker_b200",
                        "-lgwt_b200", f"-Wl,-rpath,{libdir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0
    assert out.stdout.strip() == "unknown model 'tucker' (expected individual, shared or groupwise)"
