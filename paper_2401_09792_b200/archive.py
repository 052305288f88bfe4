"""`compressed.gwtk` archive, byte-compatible with the reference loader (proj/src/archive.cpp:127-311).

Layout (little endian): 'GWTK' | u32 version=1 | u32 J K M N P m n p | u8 model tag
(0 individual, 1 shared, 2 groupwise) | complex128 payload: groupwise rx[J*K] (M x m col-major),
tx[J] (N x n), delay[links] (P x p), cores[links] (m,n,p mode-1 fastest), coeffs[links] (P);
shared stores one rx and one tx; individual stores rx/tx/delay/core per link. The loader
validates the exact payload length. Our device layouts are exactly these per-group arrays,
so a group's factor set is written as one contiguous concatenation.
"""
from __future__ import annotations

import struct

import numpy as np

from .api import CompressionRanks, GroupwiseFactorSet, InvalidArgument

MAGIC = b"GWTK"
VERSION = 1
TAGS = {"individual": 0, "shared": 1, "groupwise": 2}


class ArchiveError(RuntimeError):
    pass


class BadMagicError(ArchiveError):
    pass


class VersionMismatchError(ArchiveError):
    pass


class TruncatedArchiveError(ArchiveError):
    pass


def payload_complex_count(model, J, K, M, N, P, m, n, p):  # archive.cpp:144-156
    links = J * J * K
    per_link = m * n * p + P * p
    stored = {"groupwise": links * per_link + J * K * M * m + J * N * n,
              "shared": links * per_link + M * m + N * n,
              "individual": links * (per_link + M * m + N * n)}[model]
    return stored + links * P


def _c128(a):
    a = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
    return np.ascontiguousarray(a, dtype=np.complex128).reshape(-1)


def save_archive(path, model: str, factors: GroupwiseFactorSet, coeffs, J: int, K: int, group: int = 0):
    """Write group `group` of a (batched) factor set. coeffs: [links, P] (or [g, links, P])."""
    if model == "individual":
        raise InvalidArgument("save_archive: individual model takes the per-link overload")
    if model not in TAGS:
        raise InvalidArgument(f"unknown model '{model}' (expected individual, shared or groupwise)")
    A, B, C, G = (np.asarray(x.cpu().numpy() if hasattr(x, "cpu") else x)[group]
                  for x in (factors.rx, factors.tx, factors.delay, factors.cores))
    users, M = A.shape[0], A.shape[2]
    m = A.shape[1]
    n, N = B.shape[1], B.shape[2]
    links, p, P = C.shape
    if users != J * K or B.shape[0] != J or links != J * J * K:
        raise InvalidArgument("save_archive: factor set is incomplete")
    co = np.asarray(coeffs)
    if co.ndim == 3:
        co = co[group]
    if co.shape[0] != links:
        raise InvalidArgument(f"archive: coefficient grid has {co.shape[0]} entries, expected {links}")
    if co.shape[1] != P:
        raise InvalidArgument("archive: coefficient vector length mismatch")
    head = MAGIC + struct.pack("<9I", VERSION, J, K, M, N, P, m, n, p) + bytes([TAGS[model]])
    parts = [_c128(A) if model == "groupwise" else _c128(A[0]), _c128(B) if model == "groupwise" else _c128(B[0]),
             _c128(C), _c128(G), _c128(co)]
    with open(path, "wb") as f:
        f.write(head)
        for x in parts:
            f.write(x.astype("<c16").tobytes())


def save_archive_individual(path, rx, tx, delay, cores, coeffs, J: int, K: int):
    """Per-link overload (archive.cpp:202-224): rx [links, m, M], tx [links, n, N], delay [links, p, P],
    cores [links, p, n, m]."""
    links = J * J * K
    rx, tx, delay, cores = (np.asarray(x) for x in (rx, tx, delay, cores))
    if rx.shape[0] != links:
        raise InvalidArgument("save_archive: link grid does not match J^2*K")
    m, M = rx.shape[1], rx.shape[2]
    n, N = tx.shape[1], tx.shape[2]
    p, P = delay.shape[1], delay.shape[2]
    co = np.asarray(coeffs)
    if co.shape != (links, P):
        raise InvalidArgument("archive: coefficient vector length mismatch")
    head = MAGIC + struct.pack("<9I", VERSION, J, K, M, N, P, m, n, p) + bytes([TAGS["individual"]])
    with open(path, "wb") as f:
        f.write(head)
        for x in (rx, tx, delay, cores, co):
            f.write(_c128(x).astype("<c16").tobytes())


def load_archive(path):
    """Returns dict(model, J, K, M, N, P, ranks, factors | links, coeffs) (archive.cpp:228-311)."""
    try:
        data = open(path, "rb").read()
    except OSError:
        raise ArchiveError(f"cannot open '{path}' for reading")
    if len(data) < 4 or data[:4] != MAGIC:
        raise BadMagicError("archive: bad magic (expected GWTK)")
    if len(data) < 8:
        raise TruncatedArchiveError(f"archive truncated: need 4 bytes at offset 4")
    version = struct.unpack_from("<I", data, 4)[0]
    if version != VERSION:
        raise VersionMismatchError(f"archive: version {version} not supported (expected {VERSION})")
    if len(data) < 41:
        raise TruncatedArchiveError(f"archive truncated: need 4 bytes at offset {min(len(data), 40) // 4 * 4}")
    J, K, M, N, P, m, n, p = struct.unpack_from("<8I", data, 8)
    tag = data[40]
    models = {v: k for k, v in TAGS.items()}
    if tag not in models:
        raise ArchiveError(f"archive: unknown model tag {tag}")
    model = models[tag]
    if min(J, K, M, N, P) < 1:
        raise ArchiveError("archive: non-positive dimension in header")
    for name, r, d, mode in (("m", m, M, 1), ("n", n, N, 2), ("p", p, P, 3)):
        if r < 1 or r > d:
            raise InvalidArgument(f"rank {name} = {r} out of range for mode-{mode} size {d}")
    expected = payload_complex_count(model, J, K, M, N, P, m, n, p)
    actual = len(data) - 41
    if actual != expected * 16:
        raise TruncatedArchiveError(f"archive: payload is {actual} bytes, expected exactly {expected * 16}")
    pay = np.frombuffer(data, dtype="<c16", offset=41).astype(np.complex128)
    links, users = J * J * K, J * K
    pos = 0

    def take(count, shape):
        nonlocal pos
        out = pay[pos:pos + count].reshape(shape)
        pos += count
        return out

    out = dict(model=model, J=J, K=K, M=M, N=N, P=P, ranks=CompressionRanks(m, n, p))
    if model == "individual":
        out["links"] = dict(rx=take(links * M * m, (links, m, M)), tx=take(links * N * n, (links, n, N)),
                            delay=take(links * P * p, (links, p, P)), cores=take(links * m * n * p, (links, p, n, m)))
    else:
        if model == "groupwise":
            A = take(users * M * m, (users, m, M))
            B = take(J * N * n, (J, n, N))
        else:
            A = np.repeat(take(M * m, (1, m, M)), users, axis=0)
            B = np.repeat(take(N * n, (1, n, N)), J, axis=0)
        C = take(links * P * p, (links, p, P))
        G = take(links * m * n * p, (links, p, n, m))
        out["factors"] = GroupwiseFactorSet(A[None], B[None], C[None], G[None])
    out["coeffs"] = take(links * P, (links, P))
    return out
