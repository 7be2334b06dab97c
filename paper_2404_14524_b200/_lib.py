"""ctypes binding of libnysipm.so (include/nysipm.h) — argument marshalling only.

Every step of the hot path runs in the CUDA library; this module only converts torch
tensors / numpy arrays into pointers and sizes.  There is no CPU fallback: if the shared
library or a CUDA device is missing, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libnysipm.so")

NYS_OK, NYS_NOTCONV = 0, 1
ERRORS = {-1: "EINVAL", -2: "ENONPOS", -3: "ECHOL", -4: "EBREAKDOWN", -5: "EMAXITER", -6: "ECUDA",
          -7: "ENCCL", -8: "ENOMEM", 1: "NOTCONV"}


class NysError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class SketchInfo(C.Structure):
    _fields_ = [("nu", C.c_double), ("chol_retries", C.c_int), ("orth_err", C.c_double), ("t_ms", C.c_double),
                ("jacobi_sweeps", C.c_int)]


class PcgInfo(C.Structure):
    _fields_ = [("iters", C.c_int), ("converged", C.c_int), ("res_norm", C.c_double),
                ("true_res_norm", C.c_double), ("t_ms", C.c_double)]


class UnitBlock(C.Structure):
    _fields_ = [("row0", C.c_int64), ("count", C.c_int64), ("scale", C.c_double)]


class QP(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("A", C.c_void_p), ("lda", C.c_int64), ("q", C.c_void_p),
                ("b", C.c_void_p), ("c", C.c_void_p), ("host_ptrs", C.c_int), ("structure", C.c_int),
                ("nd", C.c_int64), ("vtype", C.c_void_p), ("ub", C.c_void_p), ("n_unit_blocks", C.c_int),
                ("unit_blocks", C.POINTER(UnitBlock))]


class Options(C.Structure):
    _fields_ = [("tol", C.c_double), ("ell", C.c_int), ("seed", C.c_uint64), ("max_outer", C.c_int),
                ("pcg_max_iter", C.c_int), ("rho0", C.c_double), ("delta0", C.c_double),
                ("reg_floor", C.c_double), ("pcg_c", C.c_double), ("pcg_floor", C.c_double),
                ("init_delta", C.c_double), ("init_tol_rel", C.c_double), ("verbose", C.c_int),
                ("prec_refresh", C.c_int), ("prec_growth", C.c_double), ("precond", C.c_int),
                ("ell_max", C.c_int), ("ell_tau", C.c_double)]


class IterRecord(C.Structure):
    _fields_ = [("k", C.c_int), ("mu", C.c_double), ("rel_p", C.c_double), ("rel_d", C.c_double),
                ("alpha_p", C.c_double), ("alpha_d", C.c_double), ("pcg_pred", C.c_int), ("pcg_corr", C.c_int),
                ("rho", C.c_double), ("delta", C.c_double), ("t_sketch_ms", C.c_double),
                ("t_pcg_ms", C.c_double), ("t_other_ms", C.c_double), ("prec_built", C.c_int), ("ell", C.c_int),
                ("lam_ell", C.c_double)]


class Solution(C.Structure):
    _fields_ = [("x", C.c_void_p), ("y", C.c_void_p), ("z", C.c_void_p), ("obj", C.c_double),
                ("dual_obj", C.c_double), ("w", C.c_void_p), ("s", C.c_void_p)]


class Report(C.Structure):
    _fields_ = [("status", C.c_int), ("outer_iters", C.c_int), ("inner_iters", C.c_int), ("rel_p", C.c_double),
                ("rel_d", C.c_double), ("mu", C.c_double), ("t_total_ms", C.c_double),
                ("t_sketch_ms", C.c_double), ("t_pcg_ms", C.c_double), ("t_other_ms", C.c_double),
                ("n_records", C.c_int), ("max_records", C.c_int), ("records", C.POINTER(IterRecord)),
                ("matvecs", C.c_int64), ("kernel_launches", C.c_int64)]


EXPORTED = ["nys_create", "nys_destroy", "nys_nccl_unique_id", "nys_strerror", "nys_last_error", "nys_normal_matvec",
            "nys_check_scaling", "nys_sketch", "nys_sketch_apply", "nys_gaussian", "nys_pcg_solve", "nys_default_options",
            "nys_ipppmm_solve", "nys_kernel_launches", "nys_loopback_comm_create", "nys_loopback_comm_destroy",
            "nys_partial_cholesky", "nys_chol_precond_apply"]

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libnysipm.so and declare the C signatures (no CUDA call is made)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise OSError(f"{path} not built: run __graft_entry__.build() or python -m paper_2404_14524_b200.build")
    lib = C.CDLL(path)
    vp, i64, dbl, i32 = C.c_void_p, C.c_int64, C.c_double, C.c_int
    lib.nys_create.argtypes = [C.POINTER(vp), i32, vp, vp, i32, i32]
    lib.nys_destroy.argtypes = [vp]
    lib.nys_nccl_unique_id.argtypes = [vp]
    lib.nys_loopback_comm_create.argtypes = [C.c_int, vp]
    lib.nys_partial_cholesky.argtypes = [vp, i64, i64, vp, i64, vp, vp, C.c_double, C.c_int, vp, vp, vp]
    lib.nys_chol_precond_apply.argtypes = [vp, i64, vp, vp]
    lib.nys_loopback_comm_destroy.argtypes = [vp]
    lib.nys_strerror.argtypes = [i32]
    lib.nys_strerror.restype = C.c_char_p
    lib.nys_last_error.argtypes = [vp]
    lib.nys_last_error.restype = C.c_char_p
    lib.nys_normal_matvec.argtypes = [vp, i64, i64, vp, i64, vp, vp, dbl, vp, vp]
    lib.nys_check_scaling.argtypes = [vp, i64, vp, C.POINTER(i64)]
    lib.nys_sketch.argtypes = [vp, i64, i64, vp, i64, vp, vp, dbl, i32, vp, vp, vp, C.POINTER(SketchInfo)]
    lib.nys_sketch_apply.argtypes = [vp, i64, i64, vp, i64, vp, vp, i32, vp, vp]
    lib.nys_gaussian.argtypes = [vp, i64, i32, C.c_uint64, C.c_uint64, vp]
    lib.nys_pcg_solve.argtypes = [vp, i64, i64, vp, i64, vp, vp, dbl, i32, vp, vp, dbl, vp, vp, dbl, i32,
                                  C.POINTER(PcgInfo)]
    lib.nys_default_options.argtypes = [C.POINTER(Options)]
    lib.nys_default_options.restype = None
    lib.nys_ipppmm_solve.argtypes = [vp, C.POINTER(QP), C.POINTER(Options), C.POINTER(Solution), C.POINTER(Report)]
    lib.nys_kernel_launches.argtypes = [vp]
    lib.nys_kernel_launches.restype = i64
    for name in EXPORTED:
        getattr(lib, name).restype = getattr(lib, name).restype or C.c_int
    _lib = lib
    return lib


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _check_cuda(*ts):
    for t in ts:
        if t is None:
            continue
        if isinstance(t, np.ndarray) or not t.is_cuda:
            raise TypeError("device tensors (torch, cuda) are required for this call")
        if t.dtype.__repr__() != "torch.float64":
            raise TypeError(f"fp64 tensor required, got {t.dtype}")


def colmajor_device(A: np.ndarray, device="cuda", lda_multiple: int = 32):
    """Copy an m x n numpy matrix to the device in the library's layout: a torch tensor of shape
    (n, lda) (row-major) == A column-major with leading dimension lda (even, padded)."""
    import torch
    m, n = A.shape
    lda = ((m + lda_multiple - 1) // lda_multiple) * lda_multiple
    host = np.zeros((n, lda), dtype=np.float64)
    host[:, :m] = A.T
    return torch.from_numpy(host).to(device), lda


def nccl_unique_id() -> bytes:
    lib = load_library()
    buf = C.create_string_buffer(128)
    rc = lib.nys_nccl_unique_id(C.cast(buf, C.c_void_p))
    if rc != 0:
        raise NysError(rc, "ncclGetUniqueId failed")
    return buf.raw


class LoopbackComm:
    """In-process loopback communicator: `world` ranks on ONE device, each driven by its own host
    thread (validation of the multi-rank path; production multi-GPU runs use NCCL).  `id` is passed
    to Context(nccl_id=...) in place of an NCCL unique id."""

    def __init__(self, world: int):
        lib = load_library()
        self._buf = C.create_string_buffer(128)
        rc = lib.nys_loopback_comm_create(int(world), C.cast(self._buf, C.c_void_p))
        if rc != 0:
            raise NysError(rc, "nys_loopback_comm_create failed")
        self.id = self._buf.raw
        self.world = world

    def close(self):
        if self._buf is not None:
            load_library().nys_loopback_comm_destroy(C.cast(self._buf, C.c_void_p))
            self._buf = None


def _ordered(fn):
    """Stream semantics of the binding: the library works on the context's stream; a call made while
    another torch stream is current first waits for that stream (inputs written there are visible) and
    makes it wait for the library's work (outputs are visible to the caller's next torch op)."""
    import functools

    @functools.wraps(fn)
    def wrapper(self, *a, **k):
        cur = self.torch.cuda.current_stream(self.device)
        other = cur.cuda_stream != self.stream.cuda_stream
        if other:
            self.stream.wait_stream(cur)
        try:
            return fn(self, *a, **k)
        finally:
            if other:
                cur.wait_stream(self.stream)
    return wrapper


class Context:
    """One library context (device + stream [+ NCCL communicator])."""

    def __init__(self, device: int = 0, stream=None, nccl_id: Optional[bytes] = None, rank: int = 0,
                 world: int = 1):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("libnysipm requires a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self.torch = torch
        self.device = device
        torch.cuda.set_device(device)
        if stream is None or stream.cuda_stream == 0:
            # the library needs a capturable (non-legacy) stream for its CUDA graphs: give it its own
            # torch stream; every call below is ordered after / before the caller's current stream
            stream = torch.cuda.Stream(device)
        self.stream = stream
        h = C.c_void_p()
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        rc = self.lib.nys_create(C.byref(h), device, C.c_void_p(stream.cuda_stream),
                                 C.cast(idbuf, C.c_void_p) if idbuf is not None else None, rank, world)
        self.h = h
        if rc != 0:
            msg = self.lib.nys_last_error(h).decode() if h.value else ""
            raise NysError(rc, msg)

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.nys_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _rc(self, rc, allow=(0,)):
        if rc not in allow:
            raise NysError(rc, self.lib.nys_last_error(self.h).decode())
        return rc

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.nys_kernel_launches(self.h))

    # ---- the four hot-path calls (same names as the C ABI) -----------------------------
    @_ordered
    def nys_normal_matvec(self, A, lda: int, m: int, d, e, delta: float, v, w):
        _check_cuda(A, d, e, v, w)
        n = A.shape[0]
        return self._rc(self.lib.nys_normal_matvec(self.h, m, n, _ptr(A), lda, _ptr(d), _ptr(e), float(delta),
                                                   _ptr(v), _ptr(w)))

    @_ordered
    def nys_gaussian(self, m: int, ell: int, seed: int, stream: int, Omega):
        _check_cuda(Omega)
        return self._rc(self.lib.nys_gaussian(self.h, m, ell, seed, stream, _ptr(Omega)))

    @_ordered
    def nys_sketch(self, A, lda: int, m: int, d, e, delta: float, ell: int, Omega, U, lam) -> SketchInfo:
        _check_cuda(A, d, e, Omega, U, lam)
        info = SketchInfo()
        self._rc(self.lib.nys_sketch(self.h, m, A.shape[0], _ptr(A), lda, _ptr(d), _ptr(e), float(delta), ell,
                                     _ptr(Omega), _ptr(U), _ptr(lam), C.byref(info)))
        return info

    @_ordered
    def nys_sketch_apply(self, A, lda: int, m: int, d, e, ell: int, Omega, Y):
        _check_cuda(A, d, e, Omega, Y)
        return self._rc(self.lib.nys_sketch_apply(self.h, m, A.shape[0], _ptr(A), lda, _ptr(d), _ptr(e), ell,
                                                  _ptr(Omega), _ptr(Y)))

    @_ordered
    def nys_partial_cholesky(self, A, lda: int, m: int, d, e, delta: float, ell: int, piv=None, L=None, dS=None):
        _check_cuda(A, d, e, L, dS)
        if piv is not None and (not piv.is_cuda or piv.dtype.__repr__() != "torch.int64"):
            raise TypeError("piv must be a cuda int64 tensor")
        return self._rc(self.lib.nys_partial_cholesky(self.h, m, A.shape[0], _ptr(A), lda, _ptr(d), _ptr(e),
                                                      float(delta), int(ell), _ptr(piv), _ptr(L), _ptr(dS)))

    @_ordered
    def nys_chol_precond_apply(self, m: int, v, out):
        _check_cuda(v, out)
        return self._rc(self.lib.nys_chol_precond_apply(self.h, m, _ptr(v), _ptr(out)))

    @_ordered
    def nys_pcg_solve(self, A, lda: int, m: int, d, e, delta: float, ell: int, U, lam, mu_prec: float, rhs, x,
                      tol_abs: float, max_iter: int) -> PcgInfo:
        _check_cuda(A, d, e, U, lam, rhs, x)
        info = PcgInfo()
        self._rc(self.lib.nys_pcg_solve(self.h, m, A.shape[0], _ptr(A), lda, _ptr(d), _ptr(e), float(delta), ell,
                                        _ptr(U), _ptr(lam), float(mu_prec), _ptr(rhs), _ptr(x), float(tol_abs),
                                        int(max_iter), C.byref(info)), allow=(0, 1))
        return info

    @_ordered
    def nys_ipppmm_solve(self, A, lda: int, m: int, q, b, c, ell: int = 0, tol: float = 1e-8, seed: int = 0,
                         max_outer: int = 100, host: bool = False, max_records: int = 256, verbose: bool = False,
                         structure: int = 0, vtype=None, ub=None, unit_blocks=None, **opt_overrides):
        """A: device tensor (ncols, lda) [or host numpy when host=True]; q, c: n; b: m.
        structure=1: A holds the dense block Xt (nd columns) of A = [Xt, -Xt, I, -I]; n = 2 nd + 2 m.
        vtype (int8, n; 0 = I, 1 = F free, 2 = J box) and ub (n, read on J): problem (P~)/(D~), f1.
        structure=2: A holds the dense block B (nd columns) of A = [B, S_0, ...], unit_blocks =
        [(row0, count, scale), ...] the scaled identity blocks S_k (nys_unit_block)."""
        import torch
        nd = A.shape[0]
        n = q.shape[0]
        opts = Options()
        self.lib.nys_default_options(C.byref(opts))
        opts.ell, opts.tol, opts.seed, opts.max_outer, opts.verbose = ell, tol, seed, max_outer, int(verbose)
        for k, v in opt_overrides.items():
            setattr(opts, k, v)
        if host:
            arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (A, q, b, c)]
            A, q, b, c = arrs
            if vtype is not None:
                vtype = np.ascontiguousarray(vtype, dtype=np.int8)
            if ub is not None:
                ub = np.ascontiguousarray(ub, dtype=np.float64)
            x, y, z, w, s = np.zeros(n), np.zeros(m), np.zeros(n), np.zeros(n), np.zeros(n)
        else:
            _check_cuda(A, q, b, c)
            if vtype is not None and (not isinstance(vtype, torch.Tensor) or vtype.dtype != torch.int8
                                      or not vtype.is_cuda or not vtype.is_contiguous()):
                raise TypeError("vtype must be a contiguous int8 CUDA tensor")
            if ub is not None:
                _check_cuda(ub)
            mk = lambda k: torch.zeros(k, dtype=torch.float64, device=A.device)  # noqa: E731
            x, y, z, w, s = mk(n), mk(m), mk(n), mk(n), mk(n)
            self.stream.wait_stream(torch.cuda.current_stream(self.device))   # outputs allocated there
        blocks = list(unit_blocks or [])
        ub_arr = (UnitBlock * max(1, len(blocks)))(*[UnitBlock(int(r), int(k), float(sc)) for r, k, sc in blocks])
        qp = QP(m, n, _ptr(A), lda, _ptr(q), _ptr(b), _ptr(c), 1 if host else 0, structure, nd if structure else 0,
                _ptr(vtype) if vtype is not None else None, _ptr(ub) if ub is not None else None, len(blocks),
                C.cast(ub_arr, C.POINTER(UnitBlock)))
        recs = (IterRecord * max_records)()
        rep = Report()
        rep.max_records = max_records
        rep.records = C.cast(recs, C.POINTER(IterRecord))
        sol = Solution(_ptr(x), _ptr(y), _ptr(z), 0.0, 0.0, _ptr(w), _ptr(s))
        rc = self.lib.nys_ipppmm_solve(self.h, C.byref(qp), C.byref(opts), C.byref(sol), C.byref(rep))
        if rc not in (0, -5):
            raise NysError(rc, self.lib.nys_last_error(self.h).decode())
        log = [{f: getattr(recs[i], f) for f, _ in IterRecord._fields_} for i in range(rep.n_records)]
        return {"x": x, "y": y, "z": z, "w": w, "s": s, "obj": sol.obj, "dual_obj": sol.dual_obj, "status": rep.status,
                "outer": rep.outer_iters, "inner": rep.inner_iters, "rel_p": rep.rel_p, "rel_d": rep.rel_d,
                "mu": rep.mu, "t_total_ms": rep.t_total_ms, "t_sketch_ms": rep.t_sketch_ms,
                "t_pcg_ms": rep.t_pcg_ms, "t_other_ms": rep.t_other_ms, "matvecs": rep.matvecs,
                "kernel_launches": rep.kernel_launches, "log": log}
