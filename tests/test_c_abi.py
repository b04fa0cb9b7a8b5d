"""The C ABI used from plain C99 (examples/c_abi_example.c): no Python, no CUDA headers.

CPU: the example compiles with -Werror against include/cpa_svt.h and links against
libcpasvt.so (every entry point it uses resolves).  GPU: it runs one dense fp64 shrinkage
through cpa_svt_apply_host and checks every element against the closed form of Alg. 1 for a
signed-permuted rectangular diagonal X (Y_ij = X_ij H_hat(X_ij^2)),
<= 1e-10 relative Frobenius -- a check that needs neither the oracle nor the binding.
"""

import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1705_07112_b200")


def _build(tmp_path):
    gcc = shutil.which("gcc") or shutil.which("cc")
    if gcc is None:
        pytest.skip("no C compiler")
    if not os.path.exists(os.path.join(LIBDIR, "libcpasvt.so")):
        pytest.fail("libcpasvt.so missing: run __graft_entry__.build()")
    exe = str(tmp_path / "c_abi_example")
    cmd = [gcc, "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", "c_abi_example.c"), "-L", LIBDIR, "-lcpasvt", f"-Wl,-rpath,{LIBDIR}",
           "-lm", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_example_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    assert os.access(exe, os.X_OK)


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,K,T,side", [
    (64, 48, 20, 30, "right"),        # c1 shape: the single-block kernel (form 4)
    (300, 500, 30, 300, "left"),      # s x s form, ragged tiles
    (700, 260, 12, 50, "right"),      # right side, ragged
    (1024, 1024, 30, 300, "left"),    # c2 shape: two chains, host pipeline
])
def test_c_example_closed_form(tmp_path, m, n, K, T, side):
    exe = _build(tmp_path)
    r = subprocess.run([exe, str(m), str(n), str(K), str(T)], capture_output=True, text=True, timeout=120)
    out = r.stdout.strip()
    assert r.returncode == 0, (out, r.stderr)
    mo = re.search(r"side=(\w+) form=(\d+) lambda_max=(\S+) rel_fro=(\S+)", out)
    assert mo, out
    assert mo.group(1) == side
    assert float(mo.group(4)) <= 1e-10, out
    print(out)
