"""tcgen05 plumbing check: a 128x128 TF32 / 3xTF32 GEMM tile through TMEM against fp64 torch."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("K,split3", [(32, 0), (96, 0), (96, 1), (200, 1)])
def test_tc_gemm_tile(K, split3):
    torch = pytest.importorskip("torch")
    from paper_2401_09792_b200 import _lib
    lib = _lib.load()
    g = torch.Generator().manual_seed(K)
    A = torch.randn(128, K, generator=g, dtype=torch.float32)
    B = torch.randn(128, K, generator=g, dtype=torch.float32)
    Ad, Bd = A.cuda(), B.cuda()
    Cd = torch.zeros(128, 128, dtype=torch.float32, device="cuda")
    rc = lib.gwt_debug_tc_gemm(C.c_int(K), C.c_void_p(Ad.data_ptr()), C.c_void_p(Bd.data_ptr()),
                               C.c_void_p(Cd.data_ptr()), C.c_int(split3))
    assert rc == 0
    want = A.double() @ B.double().T
    err = (Cd.cpu().double() - want).abs().max().item() / want.abs().max().item()
    assert err < (1e-5 if split3 else 3e-3), err


@pytest.mark.parametrize("name,ngroups,sweeps", [("C3", 2, 3), ("C5", 2, 3), ("C4", 1, 2)])
def test_gram_tc_matches_cuda_core_gram(name, ngroups, sweeps, monkeypatch):
    """The tcgen05 3xTF32 transmit Gram (row-block unfoldings, N = 128 at C3 / C5: one 128 x 128 strip;
    N = 256 at C4: the 128 x 256 strip) gives the same Tucker solve as the FP32 CUDA-core Gram
    (GWT_GRAM_TC=0). The switch is read when a Context is created, so each setting gets its own."""
    import paper_2401_09792_b200 as gw
    from tests.helpers import baseline_inputs
    cfg = gw.CONFIGS[name]
    X, _, _ = baseline_inputs(cfg, ngroups)
    out = {}
    for tcv in ("0", "1"):
        monkeypatch.setenv("GWT_GRAM_TC", tcv)
        ctx = gw.Context(0)
        out[tcv] = ctx.groupwise_solve(cfg.topology(), X, cfg.ranks(), sweeps, early_stop=False)
        ctx.close()
    a, b = out["0"], out["1"]
    assert np.max(np.abs(a.trace / a.energy[:, None] - b.trace / b.energy[:, None])) <= 1e-6
    assert np.max(np.abs(a.energy - b.energy) / a.energy) <= 1e-6
