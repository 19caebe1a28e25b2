"""Thin ctypes binding of libswr.so (include/swr.h).

Argument marshalling only: every step of the method runs in the library's
CUDA kernels.  PyTorch is used for device memory and streams.  There is no
CPU fallback: if libswr.so is missing or no GPU is usable, this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libswr.so")

SWR_OK, SWR_NOT_CONVERGED = 0, 2
STATUS = {0: "ok", 1: "invalid argument", 2: "not converged", 3: "zero pivot", 4: "breakdown",
          5: "inner not converged", 6: "unsupported", 7: "cuda error", 8: "nccl error", 9: "oom"}


class SWRError(RuntimeError):
    def __init__(self, status, where, detail=""):
        super().__init__(f"{where}: status {status} ({STATUS.get(status, '?')}) {detail}")
        self.status = status


class Config(C.Structure):
    _fields_ = [
        ("a0", C.c_double), ("b0", C.c_double), ("T", C.c_double), ("dx", C.c_double), ("dt", C.c_double),
        ("N", C.c_int32), ("potential", C.c_int32), ("V_x", C.c_void_p),
        ("n_terms", C.c_int32), ("tau", C.c_void_p), ("xi", C.c_void_p), ("lam", C.c_double),
        ("transmission", C.c_int32), ("robin_p", C.c_double), ("u0", C.c_void_p),
        ("inputs_on_device", C.c_int32), ("algorithm", C.c_int32), ("tol", C.c_double),
        ("restart", C.c_int32), ("maxit", C.c_int32), ("tol_inner", C.c_double), ("maxit_inner", C.c_int32),
        ("tol_fp", C.c_double), ("maxit_fp", C.c_int32), ("g0", C.c_void_p),
        ("rank", C.c_int32), ("world", C.c_int32), ("nccl_unique_id", C.c_void_p),
        ("cuda_stream", C.c_void_p), ("device", C.c_int32), ("gs_passes", C.c_int32), ("krylov", C.c_int32),
        ("pade_m", C.c_int32), ("pinv_exact", C.c_int32), ("march_form", C.c_int32), ("toeplitz_form", C.c_int32),
        ("nl_rows_per_thread", C.c_int32),
    ]


class Report(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32), ("inner_iterations", C.c_int32), ("fp_max", C.c_int32),
        ("converged", C.c_int32), ("residual_history", C.c_void_p), ("n_history", C.c_int32),
        ("t_build_ms", C.c_double), ("t_solve_ms", C.c_double), ("t_march_ms", C.c_double),
        ("t_interface_ms", C.c_double), ("cell_steps", C.c_double), ("n_marches", C.c_int32),
        ("n_kernel_launches", C.c_int32), ("t_setup_ms", C.c_double), ("t_comm_ms", C.c_double),
    ]


_lib = None


def lib():
    """Load libswr.so (built by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        _lib = load(LIB_PATH)
    return _lib


def load(path):
    """Bind a libswr build at `path` (the product library, or a variant built
    by _build.build_variant for kernel experiments and race-stress tests)."""
    if True:
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(path)
        vp, i32, H = C.c_void_p, C.c_int32, C.c_void_p
        L.swr_setup.argtypes = [C.POINTER(Config), C.POINTER(H)]
        L.swr_update_inputs.argtypes = [H, vp, vp, i32]
        L.swr_build_interface_operator.argtypes = [H]
        L.swr_solve.argtypes = [H, vp, i32, C.POINTER(Report)]
        L.swr_free.argtypes = [H]
        L.swr_free.restype = None
        L.swr_error_string.argtypes = [i32]
        L.swr_error_string.restype = C.c_char_p
        L.swr_last_error_detail.argtypes = []
        L.swr_last_error_detail.restype = C.c_char_p
        L.swr_apply_R.argtypes = [H, vp, i32, i32, vp, vp]
        L.swr_apply_I_minus_L.argtypes = [H, i32, vp, vp]
        L.swr_get_interface.argtypes = [H, i32, vp, vp]
        L.swr_set_interface.argtypes = [H, vp, vp]
        L.swr_get_g.argtypes = [H, vp]
        L.swr_sizes.argtypes = [H, vp, vp, vp, vp]
        L.swr_partition.argtypes = [i32, i32, i32, vp, vp]
        L.swr_owned_slots.argtypes = [i32, i32, i32, vp, vp]
        L.swr_nccl_unique_id.argtypes = [vp]
        L.swr_loopback_id.argtypes = [vp, i32]
        for f in ("swr_setup", "swr_update_inputs", "swr_build_interface_operator", "swr_solve", "swr_apply_R",
                  "swr_apply_I_minus_L", "swr_get_interface", "swr_set_interface", "swr_get_g", "swr_sizes",
                  "swr_partition", "swr_owned_slots", "swr_nccl_unique_id", "swr_loopback_id"):
            getattr(L, f).restype = i32
        return L


EXPORTED = ["swr_setup", "swr_update_inputs", "swr_build_interface_operator", "swr_solve", "swr_free",
            "swr_error_string", "swr_last_error_detail", "swr_apply_R", "swr_apply_I_minus_L",
            "swr_get_interface", "swr_set_interface", "swr_get_g", "swr_sizes", "swr_partition",
            "swr_owned_slots", "swr_nccl_unique_id", "swr_loopback_id"]


def partition(N: int, world: int, rank: int):
    """Subdomains [j_lo, j_hi] (1-based, inclusive) of a rank (swr_partition)."""
    lo, hi = C.c_int32(), C.c_int32()
    _check(lib().swr_partition(N, world, rank, C.byref(lo), C.byref(hi)), "swr_partition")
    return lo.value, hi.value


def owned_slots(N: int, world: int, rank: int):
    """Interface slots [s_lo, s_hi] of a rank (swr_owned_slots)."""
    lo, hi = C.c_int32(), C.c_int32()
    _check(lib().swr_owned_slots(N, world, rank, C.byref(lo), C.byref(hi)), "swr_owned_slots")
    return lo.value, hi.value


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (create on rank 0, broadcast)."""
    buf = C.create_string_buffer(128)
    _check(lib().swr_nccl_unique_id(buf), "swr_nccl_unique_id")
    return buf.raw


def loopback_id(world: int) -> bytes:
    """Test infrastructure: a communicator id for `world` logical ranks run as
    threads of this process on one GPU (swr_loopback_id)."""
    buf = C.create_string_buffer(128)
    _check(lib().swr_loopback_id(buf, world), "swr_loopback_id")
    return buf.raw


def _check(st, where, ok=(SWR_OK,), lib_=None):
    if st not in ok:
        raise SWRError(st, where, (lib_ or lib()).swr_last_error_detail().decode())
    return st


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


class SWR:
    """One SWR problem on one GPU: the whole problem (world = 1) or rank
    `rank` of a multi-GPU run (its subdomains and interface slots)."""

    def __init__(self, p, arrays: dict, device: int = 0, stream=None, on_device: bool = False,
                 rank: int = 0, world: int = 1, nccl_id: bytes | None = None, library=None):
        import torch
        self.torch = torch
        self.L = library if library is not None else lib()
        self.p = p
        self.dev = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.dev)
        keep = {}
        for k, v in arrays.items():
            if v is None:
                keep[k] = None
            elif on_device:
                dt = torch.complex128 if k in ("u0", "g0") else torch.float64
                with torch.cuda.stream(self.stream):   # ordered before the library's reads
                    keep[k] = torch.as_tensor(v, dtype=dt, device=self.dev).contiguous()
            else:
                dt = np.complex128 if k in ("u0", "g0") else np.float64
                keep[k] = np.ascontiguousarray(v, dtype=dt)
        self._keep = keep
        c = Config()
        c.a0, c.b0, c.T, c.dx, c.dt = p.a0, p.b0, p.T, p.dx, p.dt
        c.N, c.potential = p.N, p.potential
        c.V_x = _ptr(keep.get("V_x"))
        tau = keep.get("tau")
        c.n_terms = 0 if tau is None else int(tau.shape[0])
        c.tau, c.xi = _ptr(tau), _ptr(keep.get("xi"))
        c.lam, c.transmission, c.robin_p = p.lam, p.transmission, p.robin_p
        c.u0 = _ptr(keep["u0"])
        c.inputs_on_device = int(on_device)
        c.algorithm = p.algorithm
        c.tol, c.restart, c.maxit = p.tol, p.restart, p.maxit
        c.tol_inner, c.maxit_inner = p.tol_inner, p.maxit_inner
        c.tol_fp, c.maxit_fp = p.tol_fp, p.maxit_fp
        c.g0 = _ptr(keep.get("g0"))
        self._nccl_id = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        c.rank, c.world = rank, world
        c.nccl_unique_id = C.cast(self._nccl_id, C.c_void_p) if self._nccl_id else None
        c.cuda_stream = self.stream.cuda_stream
        c.device = device
        c.gs_passes = getattr(p, "gs_passes", 1)
        c.krylov = getattr(p, "krylov", 0)
        c.pade_m = getattr(p, "pade_m", 0)
        c.pinv_exact = getattr(p, "pinv_exact", 0)
        c.march_form = getattr(p, "march_form", 0)
        c.toeplitz_form = getattr(p, "toeplitz_form", 0)
        c.nl_rows_per_thread = getattr(p, "nl_rows_per_thread", 0)
        self.cfg = c
        h = C.c_void_p()
        with torch.cuda.device(self.dev):
            _check(self.L.swr_setup(C.byref(c), C.byref(h)), "swr_setup", lib_=self.L)
        self.h = h
        self.Nx, self.NT, self.Nj = p.Nx, p.NT, p.Nj
        self.ng = (2 * p.N - 2) * p.NT
        self.rank, self.world = rank, world
        if p.N >= 2:
            self.s_lo, self.s_hi = owned_slots(p.N, world, rank)
        else:
            self.s_lo, self.s_hi = 0, -1
        self.nloc = (self.s_hi - self.s_lo + 1) * p.NT

    def close(self):
        if getattr(self, "h", None):
            self.L.swr_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- main ABI -----------------------------------------------------------
    def update_inputs(self, u0=None, V_x=None, on_device=False):
        _check(self.L.swr_update_inputs(self.h, _ptr(u0), _ptr(V_x), int(on_device)), "swr_update_inputs")

    def build(self):
        _check(self.L.swr_build_interface_operator(self.h), "swr_build_interface_operator")

    def solve(self, out=None, on_device=None, allow_unconverged=True):
        """Returns (status, u(T), report dict).  out: numpy (host) or torch
        cuda tensor of N_x+1 complex; default a new host array."""
        if out is None:
            out = np.zeros(self.Nx + 1, np.complex128)
        if on_device is None:
            on_device = not isinstance(out, np.ndarray)
        rep = Report()
        ok = (SWR_OK, SWR_NOT_CONVERGED) if allow_unconverged else (SWR_OK,)
        st = _check(self.L.swr_solve(self.h, _ptr(out), int(on_device), C.byref(rep)), "swr_solve", ok)
        hist = np.ctypeslib.as_array((C.c_double * rep.n_history).from_address(rep.residual_history)).copy() \
            if rep.n_history else np.zeros(0)
        r = {f: getattr(rep, f) for f, _ in Report._fields_ if f != "residual_history"}
        r["history"] = hist
        r["status"] = st
        return st, out, r

    # ---- lower-level entry points (device tensors) ---------------------------
    def _cz(self, n):
        # zero-filled on the handle's stream: the library's copies into it are
        # ordered after the fill (a fill on another stream could land after them)
        with self.torch.cuda.stream(self.stream):
            return self.torch.zeros(n, dtype=self.torch.complex128, device=self.dev)

    def apply_R(self, g=None, use_u0=True, force_zero=False, want_uT=False):
        Rg = self._cz(max(self.ng, 1))
        uT = self._cz(self.Nx + 1) if want_uT else None
        _check(self.L.swr_apply_R(self.h, _ptr(g), int(use_u0), int(force_zero), _ptr(Rg), _ptr(uT)), "swr_apply_R")
        return Rg[: self.ng], uT

    def apply_I_minus_L(self, x, which=0):
        y = self._cz(self.ng)
        _check(self.L.swr_apply_I_minus_L(self.h, which, _ptr(x), _ptr(y)), "swr_apply_I_minus_L")
        return y

    def get_interface(self, which=0):
        d = self._cz(max(self.ng, 1))
        X = self._cz(self.p.N * 4 * self.NT)
        _check(self.L.swr_get_interface(self.h, which, _ptr(d), _ptr(X)), "swr_get_interface")
        return d[: self.ng], X.view(self.p.N, 4, self.NT)

    def set_interface(self, d, X):
        """Test infrastructure: use the given d and first columns X (layout of
        get_interface) as the interface operator of the next solve."""
        t = self.torch
        with t.cuda.stream(self.stream):
            dd = t.as_tensor(np.ascontiguousarray(d), dtype=t.complex128, device=self.dev)
            XX = t.as_tensor(np.ascontiguousarray(X), dtype=t.complex128, device=self.dev)
        _check(self.L.swr_set_interface(self.h, _ptr(dd), _ptr(XX)), "swr_set_interface")

    def get_g(self):
        """This rank's slots of g (the whole g on one GPU)."""
        g = self._cz(self.nloc)
        _check(self.L.swr_get_g(self.h, _ptr(g)), "swr_get_g")
        return g
