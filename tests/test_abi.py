"""C-ABI library: builds, loads, exports every symbol include/cpa_svt.h declares,
validates arguments before any device work, and its host-side coefficient
function agrees with the oracle (no GPU needed)."""

import ctypes
import importlib.util
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cpa_svt.h")


def _build():
    spec = importlib.util.spec_from_file_location("cpa_build", os.path.join(ROOT, "paper_1705_07112_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.build()


@pytest.fixture(scope="module")
def P():
    _build()
    import paper_1705_07112_b200 as P
    return P


def test_exports_every_declared_symbol(P):
    declared = set(re.findall(r"\b(cpa_svt_\w+)\s*\(", open(HEADER).read()))
    assert {"cpa_svt_init", "cpa_svt_coeffs", "cpa_svt_apply", "cpa_svt_apply_batched", "cpa_svt_apply_csr",
            "cpa_svt_free"} <= declared
    out = subprocess.run(["nm", "-D", "--defined-only", P.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (cpa_svt_\w+)", out))
    assert declared <= exported, declared - exported
    for name in declared:
        assert hasattr(P.lib, name)


def test_sm100a_code_only(P):
    out = subprocess.run(["cuobjdump", "--list-elf", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass  # fp64 recurrence on the tensor pipe


def test_argument_validation_without_device(P):
    L = P.lib
    k = P.kernel_from_dict({"kind": "soft", "tau": 1.0})
    lam = P.Lambda(30, 0, 1.01, 0.0, 0.0)
    # NULL handle / pointers are rejected before any CUDA call
    assert L.cpa_svt_apply(None, 0, 0, 4, 4, 0, 0, None, 4, None, 4, ctypes.byref(k), 5, None,
                           ctypes.byref(lam), None) == 1
    assert L.cpa_svt_apply_batched(None, 1, 8, 8, None, None, ctypes.byref(k), 5, ctypes.byref(lam), None) == 1
    assert L.cpa_svt_apply_csr(None, 4, 4, 0, None, None, None, 0, 4, None, 4, ctypes.byref(k), 5, None,
                               ctypes.byref(lam), None) == 1
    nr, rk = ctypes.c_int(), ctypes.c_int()
    assert L.cpa_svt_comm_info(None, ctypes.byref(nr), ctypes.byref(rk)) == 1
    assert L.cpa_svt_set_option(None, 3, 1) == 1
    h = ctypes.c_void_p()
    assert L.cpa_svt_init(ctypes.byref(h), 0, None, None, 1, 1) == 1     # rank >= world
    assert L.cpa_svt_init(ctypes.byref(h), 0, None, None, 0, 2) == 1     # world > 1 needs an id
    assert L.cpa_svt_status_string(7) == b"unsupported by this build"


@pytest.mark.parametrize("kind", ["hard", "soft", "wsoft"])
@pytest.mark.parametrize("K", [2, 7, 30, 64])
def test_host_coeffs_match_oracle(P, kind, K):
    import oracle as O
    d = {"kind": kind, "tau": 3.0, "tau_relative": True, "w_c": 22.4, "w_shift": 0.0, "w_eps": 1e-6}
    lam, sig = 1.01 * 95.0, 95.0 ** 0.5
    c_lib = P.coeffs(d, K, lam, sig)
    c_or = O.kernel_coefficients(O.Kernel(**d), K, lam, sig)
    assert max(abs(a - b) for a, b in zip(c_lib, c_or)) <= 1e-14 * max(1.0, max(abs(v) for v in c_or))


def test_host_coeffs_domain(P):
    with pytest.raises(P.CpaSvtError):
        P.coeffs({"kind": "soft", "tau": -1.0}, 5, 10.0)
    with pytest.raises(P.CpaSvtError):
        P.coeffs({"kind": "soft", "tau": 1.0}, 5, -10.0)
