"""ctypes wrapper of the C oracle (oracle/swr_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py
(cpu_baseline, --impl reference) may import this module.  It shares no code
with the CUDA product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "swr_oracle.c")

CFLAGS = ["-O2", "-ffp-contract=off", "-fcx-limited-range", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile the oracle (plain gcc, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "swr_oracle.h"))):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _SO + ".tmp", _SRC, "-lm", "-lpthread"])
        os.replace(_SO + ".tmp", _SO)
    return _SO


class _Problem(C.Structure):
    _fields_ = [
        ("a0", C.c_double), ("b0", C.c_double), ("T", C.c_double), ("dx", C.c_double), ("dt", C.c_double),
        ("N", C.c_int32), ("potential", C.c_int32), ("V_x", C.c_void_p),
        ("n_terms", C.c_int32), ("tau", C.c_void_p), ("xi", C.c_void_p),
        ("lam", C.c_double), ("transmission", C.c_int32), ("robin_p", C.c_double),
        ("u0", C.c_void_p), ("algorithm", C.c_int32),
        ("tol", C.c_double), ("restart", C.c_int32), ("maxit", C.c_int32),
        ("tol_inner", C.c_double), ("maxit_inner", C.c_int32),
        ("tol_fp", C.c_double), ("maxit_fp", C.c_int32),
        ("g0", C.c_void_p), ("gs_passes", C.c_int32), ("krylov", C.c_int32),
        ("pade_m", C.c_int32), ("pinv_exact", C.c_int32),
    ]


class _Cplx(C.Structure):
    _fields_ = [("re", C.c_double), ("im", C.c_double)]


class _Report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("inner_iterations", C.c_int32), ("fp_max", C.c_int32),
                ("converged", C.c_int32), ("n_history", C.c_int32), ("history", C.c_void_p)]


_lib = None


_variants = {}


def _variant(tag, flags):
    if tag not in _variants:
        so = os.path.join(_HERE, f"liboracle_{tag}.so")
        if not os.path.exists(so) or os.path.getmtime(so) < max(
                os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "swr_oracle.h"))):
            subprocess.check_call(["gcc", *flags, "-o", so + ".tmp", _SRC, "-lm", "-lpthread"])
            os.replace(so + ".tmp", so)
        _variants[tag] = _bind(C.CDLL(so))
    return _variants[tag]


def lib_fma():
    """The same oracle source built with FMA contraction (-ffp-contract=fast):
    only its rounding differs, so the spread between the two builds measures
    how much a problem amplifies rounding (the parity floor of the full-size
    sampled tests)."""
    return _variant("fma", [f for f in CFLAGS if f != "-ffp-contract=off"] + ["-ffp-contract=fast", "-mfma"])


def lib_mutant(k: int):
    """The oracle with deliberate error k planted (-DOR_MUTANT=k, see the
    mutation hooks in swr_oracle.c): tests/test_oracle_mutants.py shows that
    the pins catch each one.  Never used for parity."""
    return _variant(f"mut{k}", CFLAGS + [f"-DOR_MUTANT={int(k)}"])


def lib():
    global _lib
    if _lib is None:
        _lib = _bind(C.CDLL(build()))
    return _lib


def _bind(_lib):
    if True:
        P = C.POINTER(_Problem)
        vp, i32 = C.c_void_p, C.c_int32
        _lib.or_coeffs.argtypes = [i32, vp, vp, vp]
        _lib.or_sizes.argtypes = [P, vp, vp, vp]
        _lib.or_fem.argtypes = [i32, C.c_double, vp, vp, vp, vp, vp, vp, vp]
        _lib.or_thomas.argtypes = [i32, vp, vp, vp, vp, vp]
        _lib.or_subdomain_matrix.argtypes = [P, i32, i32, i32, vp, vp, vp]
        _lib.or_march.argtypes = [P, i32, vp, vp, i32, i32, vp, vp, vp, vp]
        _lib.or_apply_R.argtypes = [P, vp, i32, i32, vp, vp]
        _lib.or_build_L.argtypes = [P, i32, vp]
        _lib.or_apply_L.argtypes = [P, vp, vp, vp]
        _lib.or_apply_L.restype = None
        _lib.or_dot.argtypes = [P, vp, vp]
        _lib.or_dot.restype = _Cplx
        _lib.or_gmres_dense.argtypes = [i32, i32, vp, vp, vp, C.c_double, i32, i32, vp, vp]
        _lib.or_bicgstab_dense.argtypes = [i32, vp, vp, vp, C.c_double, i32, vp, vp]
        _lib.or_solve.argtypes = [P, vp, C.POINTER(_Report), vp]
        _lib.or_monodomain.argtypes = [P, vp, vp]
        _lib.or_pade_coeffs.argtypes = [i32, vp, vp]
        _lib.or_pade_coeffs.restype = None
        _lib.or_tc_apply.argtypes = [P, C.c_double, C.c_double, i32, vp, vp]
        _lib.or_pinv_causal.argtypes = [P, vp, vp, vp]
        _lib.or_set_threads.argtypes = [i32]
        _lib.or_set_threads.restype = None
        _lib.or_get_threads.argtypes = []
        for f in ("or_sizes", "or_thomas", "or_subdomain_matrix", "or_march", "or_apply_R",
                  "or_build_L", "or_gmres_dense", "or_bicgstab_dense", "or_solve", "or_monodomain",
                  "or_tc_apply", "or_pinv_causal", "or_get_threads"):
            getattr(_lib, f).restype = i32
        _lib.or_coeffs.restype = None
        _lib.or_fem.restype = None
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def _c128(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.complex128)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


class Oracle:
    """The oracle bound to one problem (swr_inputs.Problem + input arrays)."""

    def __init__(self, p, arrays: dict, library=None):
        self.p = p
        self.keep = {k: (_c128(v) if k in ("u0", "g0") else _f64(v)) for k, v in arrays.items()}
        s = _Problem()
        s.a0, s.b0, s.T, s.dx, s.dt = p.a0, p.b0, p.T, p.dx, p.dt
        s.N, s.potential = p.N, p.potential
        s.V_x = _ptr(self.keep.get("V_x"))
        tau = self.keep.get("tau")
        s.n_terms = 0 if tau is None else tau.shape[0]
        s.tau, s.xi = _ptr(tau), _ptr(self.keep.get("xi"))
        s.lam, s.transmission, s.robin_p = p.lam, p.transmission, p.robin_p
        s.u0 = _ptr(self.keep["u0"])
        s.algorithm = p.algorithm
        s.tol, s.restart, s.maxit = p.tol, p.restart, p.maxit
        s.tol_inner, s.maxit_inner = p.tol_inner, p.maxit_inner
        s.tol_fp, s.maxit_fp = p.tol_fp, p.maxit_fp
        s.g0 = _ptr(self.keep.get("g0"))
        s.gs_passes = p.gs_passes
        s.krylov = p.krylov
        s.pade_m = getattr(p, "pade_m", 0)
        s.pinv_exact = getattr(p, "pinv_exact", 0)
        self.s = s
        self.L = library if library is not None else lib()
        self.Nx, self.NT, self.Nj = p.Nx, p.NT, p.Nj
        self.ng = (2 * p.N - 2) * p.NT

    # --- building blocks --------------------------------------------------
    def subdomain_matrix(self, j, n=1, force_zero=False):
        lo, di, up = (np.zeros(self.Nj, np.complex128) for _ in range(3))
        st = self.L.or_subdomain_matrix(C.byref(self.s), j, n, int(force_zero), _ptr(lo), _ptr(di), _ptr(up))
        assert st == 0, st
        return lo, di, up

    def pinv_causal(self, X, y):
        """x = (I - L0)^{-1} y by causal forward substitution (X: first columns)."""
        X, y = _c128(X), _c128(y)
        x = np.zeros(self.ng, np.complex128)
        st = self.L.or_pinv_causal(C.byref(self.s), _ptr(X), _ptr(y), _ptr(x))
        assert st == 0, st
        return x

    def tc_apply(self, v, W=0.0, dnW=0.0):
        """S v_n, n = 1..len(v)-1, of the configured operator at one boundary point."""
        v = _c128(v)
        out = np.zeros(len(v) - 1, np.complex128)
        st = self.L.or_tc_apply(C.byref(self.s), float(W), float(dnW), len(v) - 1, _ptr(v), _ptr(out))
        assert st == 0, st
        return out

    def march(self, j, lin=None, rin=None, use_u0=True, force_zero=False):
        lin, rin = _c128(lin), _c128(rin)
        ol = np.zeros(self.NT, np.complex128)
        orr = np.zeros(self.NT, np.complex128)
        uT = np.zeros(self.Nj, np.complex128)
        fp = np.zeros(1, np.int32)
        st = self.L.or_march(C.byref(self.s), j, _ptr(lin), _ptr(rin), int(use_u0), int(force_zero),
                             _ptr(ol), _ptr(orr), _ptr(uT), _ptr(fp))
        return st, ol, orr, uT, int(fp[0])

    def apply_R(self, g=None, use_u0=True, force_zero=False):
        g = _c128(g)
        Rg = np.zeros(self.ng, np.complex128)
        fp = np.zeros(1, np.int32)
        st = self.L.or_apply_R(C.byref(self.s), _ptr(g), int(use_u0), int(force_zero), _ptr(Rg), _ptr(fp))
        assert st in (0, 5), st
        return Rg

    def build_L(self, force_zero=False):
        X = np.zeros((self.p.N, 4, self.NT), np.complex128)
        st = self.L.or_build_L(C.byref(self.s), int(force_zero), _ptr(X))
        assert st == 0, st
        return X

    def apply_L(self, X, g):
        X, g = _c128(X), _c128(g)
        out = np.zeros(self.ng, np.complex128)
        self.L.or_apply_L(C.byref(self.s), _ptr(X), _ptr(g), _ptr(out))
        return out

    def dot(self, x, y):
        x, y = _c128(x), _c128(y)
        r = self.L.or_dot(C.byref(self.s), _ptr(x), _ptr(y))
        return complex(r.re, r.im)

    def solve(self):
        uT = np.zeros(self.Nx + 1, np.complex128)
        g = np.zeros(max(self.ng, 1), np.complex128)
        hist = np.zeros(self.p.maxit + 1, np.float64)
        rep = _Report()
        rep.history = _ptr(hist)
        st = self.L.or_solve(C.byref(self.s), _ptr(uT), C.byref(rep), _ptr(g))
        return dict(status=st, uT=uT, g=g[: self.ng], iterations=rep.iterations,
                    inner_iterations=rep.inner_iterations, fp_max=rep.fp_max,
                    converged=bool(rep.converged), history=hist[: rep.n_history].copy())

    def monodomain(self):
        uT = np.zeros(self.Nx + 1, np.complex128)
        fp = np.zeros(1, np.int32)
        st = self.L.or_monodomain(C.byref(self.s), _ptr(uT), _ptr(fp))
        return st, uT, int(fp[0])


def set_threads(n: int, library=None):
    """Threads of the oracle's subdomain-parallel loops (bitwise equal results
    for any count; default 1)."""
    (library or lib()).or_set_threads(int(n))


def coeffs(n):
    a, b, g = (np.zeros(n) for _ in range(3))
    lib().or_coeffs(n, _ptr(a), _ptr(b), _ptr(g))
    return a, b, g


def fem(nn, h, W=None):
    W = _f64(W)
    arrs = [np.zeros(nn) if i % 2 == 0 else np.zeros(max(nn - 1, 1)) for i in range(6)]
    lib().or_fem(nn, h, _ptr(W), *[_ptr(a) for a in arrs])
    return arrs  # Mdiag, Moff, Sdiag, Soff, MWdiag, MWoff


def pade_coeffs(m):
    a, d = np.zeros(m + 1, np.complex128), np.zeros(m + 1, np.complex128)
    lib().or_pade_coeffs(m, _ptr(a), _ptr(d))
    return a, d


def thomas(lo, di, up, rhs):
    lo, di, up, rhs = (_c128(a) for a in (lo, di, up, rhs))
    x = np.zeros_like(rhs)
    st = lib().or_thomas(len(di), _ptr(lo), _ptr(di), _ptr(up), _ptr(rhs), _ptr(x))
    return st, x


def gmres_dense(A, b, tol=1e-10, restart=30, maxit=2000, x0=None, gs_passes=1):
    A, b = _c128(A), _c128(b)
    n = len(b)
    x = np.zeros(n, np.complex128) if x0 is None else _c128(x0).copy()
    it = np.zeros(1, np.int32)
    hist = np.zeros(maxit + 1)
    st = lib().or_gmres_dense(n, gs_passes, _ptr(A), _ptr(b), _ptr(x), tol, restart, maxit, _ptr(it), _ptr(hist))
    return st, x, int(it[0]), hist[: int(it[0])]


def bicgstab_dense(A, b, tol=1e-10, maxit=2000, x0=None):
    A, b = _c128(A), _c128(b)
    n = len(b)
    x = np.zeros(n, np.complex128) if x0 is None else _c128(x0).copy()
    it = np.zeros(1, np.int32)
    hist = np.zeros(maxit + 1)
    st = lib().or_bicgstab_dense(n, _ptr(A), _ptr(b), _ptr(x), tol, maxit, _ptr(it), _ptr(hist))
    return st, x, int(it[0]), hist[: int(it[0])]
