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
