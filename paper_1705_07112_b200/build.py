"""Build libcpasvt.so in-tree with nvcc for sm_100a (no torch JIT, no cache)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcpasvt.so")
SOURCES = ["api.cu", "dense_f64.cu", "power.cu", "batched_f32.cu", "batched_tc.cu", "sparse_f64.cu", "tc_tf32.cu", "admm.cu",
           "transform.cu", "small_f64.cu", "check.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"]


def build(verbose=False, force=False, defines=(), lib=LIB, tag=""):
    objs, cmds = [], []
    bdir = os.path.join(HERE, "build" + tag)
    os.makedirs(bdir, exist_ok=True)
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(bdir, s.replace(".cu", ".o"))
        deps = [src, os.path.join(CSRC, "common.cuh"), os.path.join(CSRC, "tma.cuh"), os.path.join(CSRC, "series.cuh"),
                os.path.join(ROOT, "include", "cpa_svt.h")]
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(d) for d in deps):
            cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd))
            cmds.append(cmd)
        objs.append(obj)
    # translation units compile in parallel (nvcc is single-threaded per file)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1) or 1) as ex:
        for r in list(ex.map(lambda c: subprocess.run(c), cmds)):
            if r.returncode:
                raise subprocess.CalledProcessError(r.returncode, r.args)
    if force or not os.path.exists(lib) or os.path.getmtime(lib) < max(os.path.getmtime(o) for o in objs):
        subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *objs,
                        "-ldl"], check=True)
    return lib


if __name__ == "__main__":
    # python build.py [-v] [-f] [--variant TAG DEF1=V DEF2=V ...]  (experiments: lib_TAG.so)
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        tag, defs = sys.argv[i + 1], sys.argv[i + 2:]
        print(build(verbose="-v" in sys.argv[:i], force=True, defines=defs,
                    lib=os.path.join(HERE, f"libcpasvt_{tag}.so"), tag="_" + tag))
    else:
        build(verbose="-v" in sys.argv, force="-f" in sys.argv)
        print(LIB)
