"""CPU checks of the C-ABI boundary (no GPU needed): the library built for
sm_100a loads, exports every symbol include/odescan_b200.h declares, and
validates its descriptors without launching anything."""

import re
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]


def _declared():
    text = (REPO / "include" / "odescan_b200.h").read_text()
    return sorted(set(re.findall(r"\b(odx_[a-z_0-9]+)\s*\(", text)))


def test_header_symbols_exported():
    from paper_2511_01465_b200 import _native as N
    L = N.lib()
    declared = _declared()
    assert declared, "no declarations parsed"
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    assert set(declared) == set(N.EXPORTS)


def test_abi_version_and_structs():
    import ctypes as C
    from paper_2511_01465_b200 import _native as N
    assert N.lib().odx_abi_version() == 1
    assert C.sizeof(N.OdxProblem) == 16 + 64 * 8
    assert C.sizeof(N.OdxStepper) == 8 + 16 * 8 + 4 * 8 + 2 * 8
    assert C.sizeof(N.OdxNewtonCfg) == 24


def test_supported_matrix():
    import paper_2511_01465_b200 as pkg
    from paper_2511_01465_b200 import _native as N
    L = N.lib()
    for name in ("logistic", "vdp", "cartpole", "dahlquist", "robertson", "lorenz63"):
        p = pkg.get_problem(name)
        for sname in ("euler", "rk4", "backward_euler", "trapezoidal"):
            assert L.odx_supported(p.native(), pkg.get_stepper(sname, p).native()) == 1
    ac = pkg.allen_cahn()
    assert L.odx_supported(ac.native(), pkg.get_stepper("backward_euler", ac).native()) == 1
    assert L.odx_supported(ac.native(), pkg.get_stepper("rk4", ac).native()) == 0
    bad = N.make_problem(99, 2, ())
    assert L.odx_supported(bad, N.make_implicit(0.0, 1.0)) == 0


def test_workspace_queries_without_gpu():
    import paper_2511_01465_b200 as pkg
    from paper_2511_01465_b200 import _native as N
    L = N.lib()
    p = pkg.van_der_pol()
    s = pkg.get_stepper("rk4", p)
    cfg = N.make_cfg(10, 0.0, 0.0, True)
    assert L.odx_solve_workspace_bytes(p.native(), s.native(), 1, 1024, cfg) == 0  # resident
    assert L.odx_solve_workspace_bytes(p.native(), s.native(), 1, 1 << 20, cfg) > (1 << 20) * 16
    assert L.odx_scan_affine_workspace_bytes(1000, 3) > 0
    assert L.odx_shard_workspace_bytes(p.native(), s.native(), 1000) > 0


def test_invalid_arguments_fail_without_launch():
    import paper_2511_01465_b200 as pkg
    from paper_2511_01465_b200 import _native as N
    L = N.lib()
    p = pkg.van_der_pol()
    s = pkg.get_stepper("rk4", p)
    cfg0 = N.make_cfg(0, 0.0, 0.0, True)
    rc = L.odx_solve(p.native(), s.native(), 0, 0, 1, 10, 0.1, cfg0, 0, 0, 0, 0, 0, 0, 0, 0)
    assert rc == N.ODX_EINVAL
    assert b"max_iters" in L.odx_last_error()
    cfg = N.make_cfg(3, 0.0, 0.0, True)
    rc = L.odx_solve(p.native(), s.native(), 0, 0, 1, 10, -1.0, cfg, 0, 0, 0, 0, 0, 0, 0, 0)
    assert rc == N.ODX_EINVAL
    with pytest.raises(ValueError):
        N.check(N.ODX_EINVAL)


def test_solve_host_validates_before_any_device_work():
    """odx_solve_host rejects null host buffers and empty shapes with
    ODX_EINVAL and a message, before touching CUDA (runs without a GPU)."""
    import numpy as np
    import paper_2511_01465_b200 as pkg
    from paper_2511_01465_b200 import _native as N
    L = N.lib()
    p = pkg.van_der_pol()
    s = pkg.get_stepper("rk4", p)
    cfg = N.make_cfg(3, 0.0, 0.0, True)
    x0 = np.zeros(2)
    X = np.zeros((8, 2))
    out = np.zeros((8, 2))
    it = np.zeros(1, np.int32)
    st = np.zeros(1, np.int32)
    ix = np.zeros(1, np.int64)
    rc = L.odx_solve_host(p.native(), s.native(), x0.ctypes.data, None, out.ctypes.data, 1, 8,
                          1e-3, cfg, None, None, it.ctypes.data, st.ctypes.data, ix.ctypes.data,
                          None)
    assert rc == N.ODX_EINVAL and b"null" in L.odx_last_error()
    rc = L.odx_solve_host(p.native(), s.native(), x0.ctypes.data, X.ctypes.data, out.ctypes.data,
                          1, 0, 1e-3, cfg, None, None, it.ctypes.data, st.ctypes.data,
                          ix.ctypes.data, None)
    assert rc == N.ODX_EINVAL
