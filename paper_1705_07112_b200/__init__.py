"""B200-native CPA singular-value shrinkage (arXiv 1705.07112) -- Python binding.

A thin ctypes layer over ``libcpasvt.so`` (C ABI declared in
``include/cpa_svt.h``).  It only marshals arguments: every step of the method
runs in the library's sm_100a kernels.  PyTorch is used for device memory and
streams.  There is no CPU fallback: if the library is missing, importing this
package raises.
"""

from __future__ import annotations

import ctypes
import os

__all__ = ["Kernel", "Lambda", "Info", "Handle", "coeffs", "CpaSvtError", "kernel_from_dict",
           "LIB_PATH", "STATUS", "HARD", "SOFT", "WSOFT", "lib"]

LIB_PATH = os.environ.get("CPA_SVT_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libcpasvt.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_1705_07112_b200/build.py` "
                      "(there is no CPU fallback)")
lib = ctypes.CDLL(LIB_PATH)

HARD, SOFT, WSOFT = 0, 1, 2
F64, F32 = 0, 1
MATH = {"native": 0, "tf32": 1, "3xtf32": 2}
SHARD = {"none": 0, "cols": 1, "rows": 2}
STATUS = {0: "ok", 1: "E_ARG", 2: "E_DOMAIN", 3: "E_DIVERGED", 4: "E_CUDA", 5: "E_NCCL", 6: "E_NOMEM",
          7: "E_UNSUPPORTED"}


def _require(cond, msg: str):
    """Argument check of the binding (raises ValueError; not an assert, so it survives python -O):
    the library writes through the pointers it is given, so shapes, dtypes and devices of every
    output buffer are checked before the call."""
    if not cond:
        raise ValueError(msg)


class Kernel(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("tau_relative", ctypes.c_int32), ("tau", ctypes.c_double),
                ("w_c", ctypes.c_double), ("w_shift", ctypes.c_double), ("w_eps", ctypes.c_double)]


class Admm(ctypes.Structure):
    _fields_ = [("rho", ctypes.c_double), ("eta", ctypes.c_double), ("tol", ctypes.c_double),
                ("max_iter", ctypes.c_int32), ("iters", ctypes.c_int32), ("last_rel", ctypes.c_double),
                ("ms_shrink", ctypes.c_double), ("ms_total", ctypes.c_double),
                ("adaptive_eps", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class Lambda(ctypes.Structure):
    _fields_ = [("power_iters", ctypes.c_int32), ("want_lambda", ctypes.c_int32), ("safety", ctypes.c_double),
                ("lambda_max", ctypes.c_double), ("lambda_hat", ctypes.c_double)]


class Info(ctypes.Structure):
    _fields_ = [("lambda_hat", ctypes.c_double), ("lambda_max", ctypes.c_double),
                ("sigma_max_hat", ctypes.c_double), ("tau_used", ctypes.c_double),
                ("side", ctypes.c_int32), ("degenerate", ctypes.c_int32),
                ("ms_gram", ctypes.c_float), ("ms_allreduce", ctypes.c_float), ("ms_power", ctypes.c_float),
                ("ms_recurrence", ctypes.c_float), ("ms_total", ctypes.c_float),
                ("kernel_launches", ctypes.c_int32), ("form", ctypes.c_int32), ("rec_products", ctypes.c_int32),
                ("line12_in_recurrence", ctypes.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_p = ctypes.c_void_p
_i64 = ctypes.c_int64
lib.cpa_svt_init.argtypes = [ctypes.POINTER(_p), ctypes.c_int, _p, _p, ctypes.c_int, ctypes.c_int]
lib.cpa_svt_free.argtypes = [_p]
lib.cpa_svt_nccl_unique_id.argtypes = [_p]
lib.cpa_svt_coeffs.argtypes = [ctypes.POINTER(Kernel), ctypes.c_int, ctypes.c_double, ctypes.c_double,
                               ctypes.POINTER(ctypes.c_double)]
lib.cpa_svt_apply.argtypes = [_p, ctypes.c_int, ctypes.c_int, _i64, _i64, ctypes.c_int, _i64, _p, _i64, _p, _i64,
                              ctypes.POINTER(Kernel), ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                              ctypes.POINTER(Lambda), ctypes.POINTER(Info)]
lib.cpa_svt_apply_host.argtypes = [_p, ctypes.c_int, ctypes.c_int, _i64, _i64, _p, _p, ctypes.POINTER(Kernel),
                                   ctypes.c_int, ctypes.POINTER(Lambda), ctypes.POINTER(Info)]
lib.cpa_svt_apply_csr.argtypes = [_p, _i64, _i64, _i64, _p, _p, _p, _i64, _i64, _p, _i64, ctypes.POINTER(Kernel),
                                  ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(Lambda),
                                  ctypes.POINTER(Info)]
lib.cpa_svt_apply_batched.argtypes = [_p, _i64, ctypes.c_int, ctypes.c_int, _p, _p, ctypes.POINTER(Kernel),
                                      ctypes.c_int, ctypes.POINTER(Lambda), _p]
lib.cpa_svt_status_string.restype = ctypes.c_char_p
lib.cpa_svt_status_string.argtypes = [ctypes.c_int]
lib.cpa_svt_last_error.restype = ctypes.c_char_p
lib.cpa_svt_last_error.argtypes = [_p]
lib.cpa_svt_launch_count.restype = ctypes.c_int64
lib.cpa_svt_launch_count.argtypes = [_p]
lib.cpa_svt_debug_gemm_tf32.argtypes = [_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _p, _i64, _p, _i64,
                                        ctypes.c_int, _p, _i64, ctypes.c_int]
lib.cpa_svt_debug_gemm_tf32.restype = ctypes.c_int
lib.cpa_svt_profile.argtypes = [_p, ctypes.c_int]
lib.cpa_svt_profile_read.argtypes = [_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]
PHASES = ["gram", "allreduce", "power", "init", "step", "sparse_z", "sparse_w", "batched", "final", "exchange"]
lib.cpa_svt_set_option.argtypes = [_p, ctypes.c_int, _i64]
lib.cpa_svt_comm_info.argtypes = [_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
lib.cpa_svt_comm_info.restype = ctypes.c_int
lib.cpa_svt_admm_recover.argtypes = [_p, _i64, _i64, _p, _p, ctypes.c_int, ctypes.POINTER(Lambda), ctypes.POINTER(Admm), _p]
lib.cpa_svt_admm_recover.restype = ctypes.c_int
lib.cpa_svt_set_epsilon.argtypes = [_p, ctypes.c_int, ctypes.c_double]
lib.cpa_svt_set_epsilon.restype = ctypes.c_int
lib.cpa_svt_set_option.restype = ctypes.c_int
FORM = {"auto": 0, "apply": 1, "poly": 2, "poly_full": 3}
for _f in ("cpa_svt_init", "cpa_svt_free", "cpa_svt_nccl_unique_id", "cpa_svt_coeffs", "cpa_svt_apply",
           "cpa_svt_apply_host", "cpa_svt_apply_csr", "cpa_svt_apply_batched", "cpa_svt_profile",
           "cpa_svt_profile_read"):
    getattr(lib, _f).restype = ctypes.c_int


class CpaSvtError(RuntimeError):
    def __init__(self, status, detail=""):
        self.status = status
        super().__init__(f"cpa_svt status {status} ({STATUS.get(status, '?')}): {detail}")


def kernel_from_dict(d) -> Kernel:
    """{'kind': 'hard'|'soft'|'wsoft', 'tau', 'tau_relative', 'w_c', 'w_shift', 'w_eps'} -> Kernel."""
    if isinstance(d, Kernel):
        return d
    kind = {"hard": HARD, "soft": SOFT, "wsoft": WSOFT}[d["kind"]]
    return Kernel(kind, int(bool(d.get("tau_relative", False))), float(d.get("tau", 0.0)),
                  float(d.get("w_c", 0.0)), float(d.get("w_shift", 0.0)), float(d.get("w_eps", 0.0)))


def coeffs(kernel, K: int, lambda_max: float, sigma_max_hat: float = 0.0):
    """cpa_svt_coeffs: the K Chebyshev-Gauss coefficients (host, fp64)."""
    out = (ctypes.c_double * K)()
    st = lib.cpa_svt_coeffs(ctypes.byref(kernel_from_dict(kernel)), K, lambda_max, sigma_max_hat, out)
    if st:
        raise CpaSvtError(st)
    return list(out)


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = lib.cpa_svt_nccl_unique_id(buf)
    if st:
        raise CpaSvtError(st, "ncclGetUniqueId")
    return buf.raw


class Handle:
    """cpa_svt_init / cpa_svt_free around a device and a CUDA stream."""

    def __init__(self, device: int | None = None, stream=None, nccl_id: bytes | None = None,
                 rank: int = 0, world: int = 1):
        import torch
        self._torch = torch
        self.device = torch.cuda.current_device() if device is None else device
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        h = _p()
        idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id else None
        st = lib.cpa_svt_init(ctypes.byref(h), self.device, _p(stream.cuda_stream), idbuf, rank, world)
        if st:
            raise CpaSvtError(st, "cpa_svt_init")
        self._h = h
        self.rank, self.world = rank, world
        self.has_comm = nccl_id is not None   # the library created an NCCL communicator (any world size)

    def _on_device(self, t):
        _require(t.device.index == self.device,
                 f"tensor on {t.device}, handle on cuda:{self.device} (the library's kernels run on the handle's device)")

    def _check(self, st, what):
        if st:
            raise CpaSvtError(st, f"{what}: {lib.cpa_svt_last_error(self._h).decode()}")

    def comm_info(self):
        """cpa_svt_comm_info -> (nranks, rank) of the library's NCCL communicator ((0, -1): none)."""
        nr, rk = ctypes.c_int(0), ctypes.c_int(0)
        self._check(lib.cpa_svt_comm_info(self._h, ctypes.byref(nr), ctypes.byref(rk)), "cpa_svt_comm_info")
        return nr.value, rk.value

    @property
    def launches(self) -> int:
        return lib.cpa_svt_launch_count(self._h)

    def set_form(self, form: str):
        """cpa_svt_set_option(FORM): 'auto' | 'apply' (W_k = Psi_k X) | 'poly' (Alg. 1 s x s form,
        symmetric lower-triangle tiles) | 'poly_full' (s x s form on full tiles, cross-check)."""
        self._check(lib.cpa_svt_set_option(self._h, 0, FORM[form]), "cpa_svt_set_option")

    def set_divergence(self, mode: str):
        """cpa_svt_set_option(DIVERGENCE): 'off' | 'on' (E_DIVERGED reported by syncing calls) |
        'sync' (every call synchronises and reports it).  SPEC.md:215."""
        self._check(lib.cpa_svt_set_option(self._h, 3, {"off": 0, "on": 1, "sync": 2}[mode]), "cpa_svt_set_option")

    def set_batched_engine(self, engine: str):
        """cpa_svt_set_option(BATCHED): 'auto' | 'ffma' (fp32 FFMA) | 'tc' (tcgen05 3xTF32)."""
        self._check(lib.cpa_svt_set_option(self._h, 2, {"auto": 0, "ffma": 1, "tc": 2}[engine]), "cpa_svt_set_option")

    def set_transform(self, transform: str):
        """cpa_svt_set_option(TRANSFORM): 'none' (T = I) | 'haar1' (one-level Haar DWT of the Gram
        index, high-frequency components of Phi set to 0; NEXT-2) | 'dct'
        (orthonormal DCT-II) | 'dct8' (8 x 8 block DCT)."""
        self._check(lib.cpa_svt_set_option(self._h, 1, {"none": 0, "haar1": 1, "dct": 2, "dct8": 3}[transform]),
                    "cpa_svt_set_option")

    def set_epsilon(self, mode: str = "none", value: float = 0.0):
        """cpa_svt_set_epsilon: 'none' | 'abs' (keep |Phi_ij| >= value) | 'topk' (keep the value largest)."""
        st = lib.cpa_svt_set_epsilon(self._h, {"none": 0, "abs": 1, "topk": 2}[mode], float(value))
        self._check(st, "cpa_svt_set_epsilon")

    def profile(self, enable: bool = True):
        """cpa_svt_profile: reset and start (or stop) per-phase CUDA-event timing."""
        self._check(lib.cpa_svt_profile(self._h, int(enable)), "cpa_svt_profile")

    def profile_read(self):
        """cpa_svt_profile_read -> {phase: (total_ms, launches)} (synchronises)."""
        ms = (ctypes.c_double * len(PHASES))()
        n = (ctypes.c_int64 * len(PHASES))()
        self._check(lib.cpa_svt_profile_read(self._h, ms, n), "cpa_svt_profile_read")
        return {p: (ms[i], n[i]) for i, p in enumerate(PHASES)}

    def debug_gemm_tf32(self, A, B, b_mn: bool, terms: int = 3):
        """Kernel unit-test hook: C = A @ B (b_mn) or A @ B.T on the tcgen05 TF32 engine."""
        torch = self._torch
        M, Kd = A.shape
        N = B.shape[1] if b_mn else B.shape[0]
        C = torch.zeros((M, (N + 3) // 4 * 4), dtype=torch.float32, device=A.device)
        self._check(lib.cpa_svt_debug_gemm_tf32(self._h, M, N, Kd, A.data_ptr(), A.stride(0), B.data_ptr(),
                                                B.stride(0), int(b_mn), C.data_ptr(), C.stride(0), terms),
                    "cpa_svt_debug_gemm_tf32")
        return C[:, :N]

    def close(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.cpa_svt_free(self._h)
        self._h = None

    __del__ = close

    @staticmethod
    def _lambda(T, safety, lambda_max, want):
        return Lambda(int(T), int(bool(want)), float(safety), float(lambda_max or 0.0), 0.0)

    def apply(self, X, kernel, K: int, T: int = 30, safety: float = 1.01, lambda_max: float = 0.0,
              coeffs=None, Y=None, math: str | None = None, shard: str = "none", long_global: int = 0,
              info: bool = False, want_lambda: bool = False):
        """cpa_svt_apply on a 2-D CUDA tensor (float64: DMMA path; float32: tcgen05 3xTF32 by
        default, math='tf32' for the single-pass reduced-accuracy mode)."""
        torch = self._torch
        _require(X.is_cuda and X.dim() == 2 and X.stride(1) == 1 and X.dtype in (torch.float64, torch.float32),
                 "X must be a 2-D float64 / float32 CUDA tensor with unit column stride")
        self._on_device(X)
        if math is None:
            math = "native" if X.dtype == torch.float64 else "3xtf32"
        if Y is None:
            Y = torch.empty(X.shape, dtype=X.dtype, device=X.device)
        _require(Y.shape == X.shape and Y.dtype == X.dtype and Y.stride(1) == 1 and Y.device == X.device,
                 "Y must be a CUDA tensor shaped like X, of X's dtype, with unit column stride")
        dt = F64 if X.dtype == torch.float64 else F32
        lam = self._lambda(T, safety, lambda_max, want_lambda)
        inf = Info() if info else None
        cbuf = (ctypes.c_double * len(coeffs))(*coeffs) if coeffs is not None else None
        K = len(coeffs) if coeffs is not None else K
        st = lib.cpa_svt_apply(self._h, dt, MATH[math], X.shape[0], X.shape[1], SHARD[shard], long_global,
                               X.data_ptr(), X.stride(0), Y.data_ptr(), Y.stride(0),
                               ctypes.byref(kernel_from_dict(kernel if kernel is not None else {"kind": "soft"})),
                               K, cbuf, ctypes.byref(lam), ctypes.byref(inf) if inf is not None else None)
        self._check(st, "cpa_svt_apply")
        if info or want_lambda:
            return Y, (inf.as_dict() if inf is not None else {"lambda_hat": lam.lambda_hat,
                                                                 "lambda_max": lam.lambda_max})
        return Y

    def apply_host(self, X, Y, kernel, K: int, T: int = 30, safety: float = 1.01, lambda_max: float = 0.0,
                   math: str = "native", info: bool = False):
        """cpa_svt_apply_host: X, Y are contiguous CPU tensors (pinned for full bandwidth)."""
        torch = self._torch
        # the library copies m*n elements of X's dtype into Y: Y must be that large and of that dtype
        _require(not X.is_cuda and not Y.is_cuda and X.dim() == 2 and X.is_contiguous() and Y.is_contiguous()
                 and X.shape == Y.shape and X.dtype == Y.dtype and X.dtype in (torch.float64, torch.float32),
                 "X and Y must be contiguous 2-D host tensors of one shape and dtype (float64 / float32)")
        dt = F64 if X.dtype == torch.float64 else F32
        lam = self._lambda(T, safety, lambda_max, False)
        inf = Info() if info else None
        st = lib.cpa_svt_apply_host(self._h, dt, MATH[math], X.shape[0], X.shape[1], X.data_ptr(), Y.data_ptr(),
                                    ctypes.byref(kernel_from_dict(kernel)), K, ctypes.byref(lam),
                                    ctypes.byref(inf) if inf is not None else None)
        self._check(st, "cpa_svt_apply_host")
        return inf.as_dict() if inf is not None else None

    def apply_batched(self, X, kernel, K: int, T: int = 30, safety: float = 1.01, lambda_max: float = 0.0,
                      Y=None, lambda_out=None):
        """cpa_svt_apply_batched on a [batch, m, n] float32 CUDA tensor."""
        torch = self._torch
        _require(X.is_cuda and X.dim() == 3 and X.dtype == torch.float32 and X.is_contiguous(),
                 "X must be a contiguous [batch, m, n] float32 CUDA tensor")
        self._on_device(X)
        if Y is None:
            Y = torch.empty_like(X)
        # the kernel writes batch*m*n floats at Y and one float per matrix at lambda_out
        _require(Y.is_cuda and Y.device == X.device and Y.dtype == torch.float32 and Y.is_contiguous()
                 and Y.shape == X.shape, "Y must be a contiguous float32 CUDA tensor shaped like X")
        if lambda_out is not None:
            _require(lambda_out.is_cuda and lambda_out.device == X.device and lambda_out.dtype == torch.float32
                     and lambda_out.is_contiguous() and lambda_out.numel() >= X.shape[0],
                     "lambda_out must be a contiguous float32 CUDA tensor with >= batch elements")
        lam = self._lambda(T, safety, lambda_max, False)
        st = lib.cpa_svt_apply_batched(self._h, X.shape[0], X.shape[1], X.shape[2], X.data_ptr(), Y.data_ptr(),
                                       ctypes.byref(kernel_from_dict(kernel)), K, ctypes.byref(lam),
                                       lambda_out.data_ptr() if lambda_out is not None else None)
        self._check(st, "cpa_svt_apply_batched")
        return Y

    def admm_recover(self, D, mask, K: int, rho: float, eta: float, T: int = 30, tol: float = 1e-4,
                     max_iter: int = 300, safety: float = 1.01, L=None, adaptive_eps: bool = False):
        """cpa_svt_admm_recover (NEXT-3): ADMM recovery of the observed entries of D (float64 CUDA
        m x n) under a uint8 CUDA mask (nonzero = observed); returns (L, info).  adaptive_eps: the
        recommended epsilon(E_t) schedule of PAPER.md:968-975 (needs set_transform('dct'|'dct8'))."""
        torch = self._torch
        _require(D.is_cuda and D.dtype == torch.float64 and D.is_contiguous() and D.dim() == 2,
                 "D must be a contiguous 2-D float64 CUDA tensor")
        self._on_device(D)
        _require(mask.is_cuda and mask.dtype == torch.uint8 and mask.shape == D.shape and mask.is_contiguous()
                 and mask.device == D.device, "mask must be a contiguous uint8 CUDA tensor shaped like D")
        if L is None:
            L = torch.empty_like(D)
        _require(L.is_cuda and L.dtype == torch.float64 and L.is_contiguous() and L.shape == D.shape
                 and L.device == D.device, "L must be a contiguous float64 CUDA tensor shaped like D")
        lam = self._lambda(T, safety, 0.0, False)
        opt = Admm(float(rho), float(eta), float(tol), int(max_iter), 0, 0.0, 0.0, 0.0, int(bool(adaptive_eps)), 0)
        st = lib.cpa_svt_admm_recover(self._h, D.shape[0], D.shape[1], D.data_ptr(), mask.data_ptr(), K,
                                      ctypes.byref(lam), ctypes.byref(opt), L.data_ptr())
        self._check(st, "cpa_svt_admm_recover")
        return L, {"iters": opt.iters, "last_rel": opt.last_rel, "ms_shrink": opt.ms_shrink, "ms_total": opt.ms_total}

    def apply_csr(self, row_ptr, col, val, m: int, n: int, kernel, K: int, T: int = 300, safety: float = 1.01,
                  lambda_max: float = 0.0, row_begin: int = 0, row_end: int | None = None, Y=None,
                  info: bool = False, want_lambda: bool = False, coeffs=None):
        """cpa_svt_apply_csr: CSR X (int64 row_ptr, int32 col, float64 val, all CUDA); returns dense rows."""
        torch = self._torch
        row_end = m if row_end is None else row_end
        _require(row_ptr.is_cuda and row_ptr.dtype == torch.int64 and row_ptr.is_contiguous()
                 and row_ptr.numel() == m + 1, "row_ptr must be a contiguous int64 CUDA tensor of m + 1 entries")
        self._on_device(row_ptr)
        _require(col.is_cuda and col.dtype == torch.int32 and col.is_contiguous() and col.device == row_ptr.device,
                 "col must be a contiguous int32 CUDA tensor")
        _require(val.is_cuda and val.dtype == torch.float64 and val.is_contiguous() and col.numel() == val.numel()
                 and val.device == row_ptr.device, "val must be a contiguous float64 CUDA tensor, one per col entry")
        _require(0 <= row_begin <= row_end <= m, "need 0 <= row_begin <= row_end <= m")
        if Y is None:
            Y = torch.empty((row_end - row_begin, n), dtype=torch.float64, device=val.device)
        _require(Y.is_cuda and Y.device == val.device and Y.dtype == torch.float64 and Y.dim() == 2
                 and Y.stride(1) == 1 and Y.shape[0] >= row_end - row_begin and Y.shape[1] == n,
                 "Y must be a float64 CUDA tensor with >= row_end - row_begin rows of n columns")
        lam = self._lambda(T, safety, lambda_max, want_lambda)
        inf = Info() if info else None
        cbuf = (ctypes.c_double * len(coeffs))(*coeffs) if coeffs is not None else None
        K = len(coeffs) if coeffs is not None else K
        st = lib.cpa_svt_apply_csr(self._h, m, n, val.numel(), row_ptr.data_ptr(), col.data_ptr(), val.data_ptr(),
                                   row_begin, row_end, Y.data_ptr(), Y.stride(0),
                                   ctypes.byref(kernel_from_dict(kernel if kernel is not None else {"kind": "hard"})),
                                   K, cbuf, ctypes.byref(lam), ctypes.byref(inf) if inf is not None else None)
        self._check(st, "cpa_svt_apply_csr")
        if info or want_lambda:
            return Y, (inf.as_dict() if inf is not None else {"lambda_hat": lam.lambda_hat,
                                                                 "lambda_max": lam.lambda_max})
        return Y
