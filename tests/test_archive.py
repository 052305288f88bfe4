"""The .gwtk archive (reference archive.cpp:127-311): header, exact-length payload, round trips,
corruption errors (restating proj/tests/test_runner.cpp:113-219)."""
import os
import struct

import numpy as np
import pytest

import paper_2401_09792_b200 as gw
from paper_2401_09792_b200 import archive as ar


def _factors(rng, g=1, J=2, K=2, M=6, N=8, P=5, m=4, n=5, p=3):
    c = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)
    links, users = J * J * K, J * K
    return gw.GroupwiseFactorSet(c(g, users, m, M), c(g, J, n, N), c(g, links, p, P), c(g, links, p, n, m)), c(links, P)


def test_round_trip_bit_identical(tmp_path):
    rng = np.random.default_rng(0)
    fs, co = _factors(rng)
    p = tmp_path / "compressed.gwtk"
    ar.save_archive(p, "groupwise", fs, co, 2, 2)
    data = p.read_bytes()
    assert data[:4] == b"GWTK" and struct.unpack_from("<9I", data, 4) == (1, 2, 2, 6, 8, 5, 4, 5, 3) and data[40] == 2
    assert len(data) == 41 + 16 * ar.payload_complex_count("groupwise", 2, 2, 6, 8, 5, 4, 5, 3)
    out = ar.load_archive(p)
    for a, b in zip((out["factors"].rx, out["factors"].tx, out["factors"].delay, out["factors"].cores),
                    (fs.rx, fs.tx, fs.delay, fs.cores)):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(out["coeffs"], co)
    ar.save_archive(tmp_path / "again.gwtk", "groupwise", out["factors"], out["coeffs"], 2, 2)
    assert (tmp_path / "again.gwtk").read_bytes() == data


def test_shared_and_individual(tmp_path):
    rng = np.random.default_rng(1)
    fs, co = _factors(rng)
    ar.save_archive(tmp_path / "s.gwtk", "shared", fs, co, 2, 2)
    out = ar.load_archive(tmp_path / "s.gwtk")
    assert out["model"] == "shared"
    np.testing.assert_array_equal(out["factors"].rx[0, 3], fs.rx[0, 0])
    c = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)
    ar.save_archive_individual(tmp_path / "i.gwtk", c(8, 4, 6), c(8, 5, 8), c(8, 3, 5), c(8, 3, 5, 4), co, 2, 2)
    out = ar.load_archive(tmp_path / "i.gwtk")
    assert out["model"] == "individual" and out["links"]["cores"].shape == (8, 3, 5, 4)


def test_corruption_is_detected(tmp_path):
    rng = np.random.default_rng(2)
    fs, co = _factors(rng)
    p = tmp_path / "c.gwtk"
    ar.save_archive(p, "groupwise", fs, co, 2, 2)
    data = p.read_bytes()
    (tmp_path / "magic.gwtk").write_bytes(b"XXXX" + data[4:])
    with pytest.raises(ar.BadMagicError, match="bad magic"):
        ar.load_archive(tmp_path / "magic.gwtk")
    (tmp_path / "ver.gwtk").write_bytes(data[:4] + struct.pack("<I", 2) + data[8:])
    with pytest.raises(ar.VersionMismatchError, match="version 2 not supported"):
        ar.load_archive(tmp_path / "ver.gwtk")
    (tmp_path / "short.gwtk").write_bytes(data[:-16])
    with pytest.raises(ar.TruncatedArchiveError, match="expected exactly"):
        ar.load_archive(tmp_path / "short.gwtk")
    (tmp_path / "long.gwtk").write_bytes(data + b"\0" * 16)
    with pytest.raises(ar.TruncatedArchiveError):
        ar.load_archive(tmp_path / "long.gwtk")
    (tmp_path / "tag.gwtk").write_bytes(data[:40] + bytes([7]) + data[41:])
    with pytest.raises(ar.ArchiveError, match="unknown model tag 7"):
        ar.load_archive(tmp_path / "tag.gwtk")
    with pytest.raises(gw.InvalidArgument, match="coefficient grid has 3 entries, expected 8"):
        ar.save_archive(tmp_path / "x.gwtk", "groupwise", fs, co[:3], 2, 2)


CPP_ROUNDTRIP = r'''
#include <cstdio>
#include <string>
#include "gwtucker/archive.hpp"
int main(int argc, char** argv) {
    // argv: mode in out   (mode "rt": load + re-save;  mode "err": print the loader's error text)
    const std::string mode = argv[1];
    try {
        gwt::LoadedArchive a = gwt::load_archive(argv[2]);
        if (mode == "err") { std::puts("no error"); return 0; }
        if (a.model == gwt::ModelKind::individual)
            gwt::save_archive(argv[3], a.links, a.num_cells, a.users_per_cell, a.coeffs);
        else
            gwt::save_archive(argv[3], a.model, a.factors, a.coeffs);
        std::puts(gwt::model_name(a.model));
    } catch (const gwt::BadMagicError& e) { std::printf("BadMagicError: %s\n", e.what());
    } catch (const gwt::VersionMismatchError& e) { std::printf("VersionMismatchError: %s\n", e.what());
    } catch (const gwt::TruncatedArchiveError& e) { std::printf("TruncatedArchiveError: %s\n", e.what());
    } catch (const gwt::ArchiveError& e) { std::printf("ArchiveError: %s\n", e.what());
    } catch (const std::invalid_argument& e) { std::printf("invalid_argument: %s\n", e.what()); }
    return 0;
}
'''


@pytest.fixture(scope="module")
def cpp_archive_tool(tmp_path_factory):
    import shutil
    import subprocess
    cxx = shutil.which("g++")
    if not cxx:
        pytest.skip("g++ not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    d = tmp_path_factory.mktemp("cpparchive")
    (d / "rt.cpp").write_text(CPP_ROUNDTRIP)
    libdir = os.path.join(root, "paper_2401_09792_b200", "_build")
    r = subprocess.run([cxx, "-std=c++17", "-I", os.path.join(root, "paper_2401_09792_b200", "host", "include"),
                        str(d / "rt.cpp"), "-o", str(d / "rt"), "-L", libdir, "-lgwtucker_b200", "-lgwt_b200",
                        f"-Wl,-rpath,{libdir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return lambda *a: subprocess.run([str(d / "rt"), *map(str, a)], capture_output=True, text=True).stdout.strip()


@pytest.mark.parametrize("model", ["groupwise", "shared", "individual"])
def test_cpp_dropin_archive_bytes_equal_python(tmp_path, cpp_archive_tool, model):
    """gwt::save_archive / load_archive of the C++ drop-in (archive.cpp:178-311) read what archive.py writes
    and write back the identical bytes, for all three models."""
    rng = np.random.default_rng(7)
    fs, co = _factors(rng)
    src = tmp_path / f"{model}.gwtk"
    if model == "individual":
        links = 8
        c = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)
        ar.save_archive_individual(src, c(links, 4, 6), c(links, 5, 8), c(links, 3, 5), c(links, 3, 5, 4), co, 2, 2)
    else:
        ar.save_archive(src, model, fs, co, 2, 2)
    out = tmp_path / f"{model}_cpp.gwtk"
    assert cpp_archive_tool("rt", src, out) == model
    assert out.read_bytes() == src.read_bytes()


def test_cpp_dropin_archive_errors_match_python(tmp_path, cpp_archive_tool):
    rng = np.random.default_rng(8)
    fs, co = _factors(rng)
    good = tmp_path / "g.gwtk"
    ar.save_archive(good, "groupwise", fs, co, 2, 2)
    data = good.read_bytes()
    cases = {"magic": b"XXXX" + data[4:], "version": data[:4] + struct.pack("<I", 9) + data[8:],
             "short": data[:-16], "header": data[:20]}
    for name, blob in cases.items():
        p = tmp_path / f"{name}.gwtk"
        p.write_bytes(blob)
        got = cpp_archive_tool("err", p)
        with pytest.raises(ar.ArchiveError) as ei:
            ar.load_archive(p)
        assert got == f"{type(ei.value).__name__}: {ei.value}", (name, got)


def test_sweep_csv_text_and_axis_error():
    """sweep.csv text as runner.cpp:288-298 writes it; a missing / unknown axis raises the reference's text."""
    from paper_2401_09792_b200 import sweep
    rows = [sweep.SweepRow(16, 12.5, 3.25, 0.0123), sweep.SweepRow(32, 6.25, 2.0, 0.001)]
    assert sweep.sweep_csv_text(rows) == "axis,Rs,Rt,ec\n16,12.500000,3.250000,0.01230000\n32,6.250000,2.000000,0.00100000\n"
    with pytest.raises(gw.InvalidArgument, match="run_sweep: config has no sweep axis"):
        sweep.run_sweep(None, None, gw.CompressionRanks(4, 16, 8), "m", [1], None, None, None)
