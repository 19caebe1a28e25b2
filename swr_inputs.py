"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NONE of the method's arithmetic: it only produces the
problem parameters and the input arrays (initial datum u0, potential samples,
random initial interface vector g0) that the paper's experiments use
(PAPER.md P:1063-1068 for the workloads, P:1079 for zero/random g0).  Both the
CPU oracle (oracle/) and the CUDA path (paper_1503_02564_b200/) receive these
arrays as inputs; neither side imports the other.

Configs C1..C5 follow SURVEY.md section 8(d) / BASELINE.json "configs".
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

# enum values mirrored by both sides' own headers (include/swr.h and
# oracle/swr_oracle.h); they are the ABI's argument codes, not arithmetic.
POT_ZERO, POT_VX, POT_VTX, POT_CUBIC = 0, 1, 2, 3
TC_ROBIN, TC_S02, TC_S03, TC_S04, TC_S12, TC_S14, TC_S22, TC_S24 = 0, 1, 2, 3, 4, 5, 6, 7
ALG_NEW, ALG_PRECOND, ALG_CLASSICAL = 0, 1, 2
KRY_GMRES, KRY_BICGSTAB, KRY_FIXED_POINT = 0, 1, 2


@dataclasses.dataclass
class Problem:
    """Problem statement of the paper."""
    a0: float = -21.0
    b0: float = 21.0
    T: float = 0.5
    dx: float = 1e-5
    dt: float = 1e-3
    N: int = 2
    potential: int = POT_ZERO
    transmission: int = TC_S02
    robin_p: float = 5.0
    algorithm: int = ALG_NEW
    lam: float = 1.0
    u0_kind: str = "gaussian"          # "gaussian" | "soliton" | "zero"
    vtx_kind: str = "5tx"              # separable V(t,x) used for POT_VTX
    vx_kind: str = "-x2"               # V(x) used for POT_VX
    tol: float = 1e-10
    restart: int = 30
    maxit: int = 2000
    tol_inner: float = 1e-12
    maxit_inner: int = 2000
    tol_fp: float = 1e-12
    maxit_fp: int = 50
    g0_random: bool = False
    gs_passes: int = 1          # Gram-Schmidt passes in GMRES: 1 = CGS (PETSc default, reading A6), 2 = CGS2
    krylov: int = KRY_GMRES     # interface solver: GMRES, BiCGStab or the algorithm's fixed point (A20/A21)
    pade_m: int = 20            # Pade poles m for TC_S22 / TC_S24 (the paper tabulates m = 20, 50, 100)
    pinv_exact: int = 0         # PRECOND: 0 = inner Krylov P^{-1} (paper), 1 = exact causal solve (8(f)-4)
    # GPU kernel forms (swr_config; same arithmetic, the oracle ignores them): 0 = automatic
    march_form: int = 0         # 1 = streaming march
    toeplitz_form: int = 0      # 1 = direct causal convolution, 2 = shared-memory FFT
    nl_rows_per_thread: int = 0  # 8 or 11: force the NL march shape
    seed: int = 7
    name: str = ""

    # ---- sizes (reading A1: global uniform mesh, N | N_x) ----
    @property
    def Nx(self) -> int:
        return int(round((self.b0 - self.a0) / self.dx))

    @property
    def NT(self) -> int:
        return int(round(self.T / self.dt))

    @property
    def Nj(self) -> int:
        return self.Nx // self.N + 1

    @property
    def ng(self) -> int:
        return (2 * self.N - 2) * self.NT

    def nodes(self) -> np.ndarray:
        """x_i = a0 + i dx, i = 0..N_x (computed as a product)."""
        return self.a0 + np.arange(self.Nx + 1, dtype=np.float64) * self.dx

    def cell_steps_per_march(self) -> int:
        """sum_j N_j * N_T (interface nodes counted in both subdomains)."""
        return self.N * self.Nj * self.NT


def make_u0(p: Problem) -> np.ndarray:
    """Initial data of P:1065-1067 sampled at the nodes (complex128)."""
    x = p.nodes()
    if p.u0_kind == "gaussian":
        y = x + 10.0
        return np.exp(-(y * y) + 20j * y)
    if p.u0_kind == "soliton":
        y = x + 10.0
        return 2.0 / np.cosh(math.sqrt(2.0) * y) * np.exp(20j * y)
    if p.u0_kind == "zero":
        return np.zeros(p.Nx + 1, dtype=np.complex128)
    raise ValueError(p.u0_kind)


def make_vx(p: Problem) -> np.ndarray:
    """Time-independent potential samples V(x_i) (V = -x^2)."""
    x = p.nodes()
    if p.vx_kind == "-x2":
        return -(x * x)
    if p.vx_kind == "zero":
        return np.zeros_like(x)
    if p.vx_kind == "const":           # V = 5 (gauge-strategy pins)
        return np.full_like(x, 5.0)
    raise ValueError(p.vx_kind)


def make_vtx(p: Problem):
    """Separable V(t,x) = sum_k tau_k(t) xi_k(x) (V = 5 t x).

    Returns (tau [n_terms, N_T+1], xi [n_terms, N_x+1]).
    """
    if p.vtx_kind == "5tx":
        t = np.arange(p.NT + 1, dtype=np.float64) * p.dt
        return (5.0 * t)[None, :].copy(), p.nodes()[None, :].copy()
    raise ValueError(p.vtx_kind)


def splitmix64(seed: int, n: int) -> np.ndarray:
    """n outputs of the splitmix64 counter generator (uint64)."""
    mask = (1 << 64) - 1
    out = np.empty(n, dtype=np.uint64)
    state = seed & mask
    for i in range(n):
        state = (state + 0x9E3779B97F4A7C15) & mask
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
        out[i] = z ^ (z >> 31)
    return out


def make_g0(p: Problem) -> np.ndarray | None:
    """Initial interface vector (reading A15): zero, or Re and Im
    uniform in [0,1) from splitmix64(seed) (53-bit mantissa), slot order."""
    if not p.g0_random or p.N < 2:
        return None
    r = splitmix64(p.seed, 2 * p.ng)
    u = (r >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return u[0::2] + 1j * u[1::2]


def inputs(p: Problem) -> dict:
    """All arrays a run needs, keyed by ABI argument name."""
    d = {"u0": make_u0(p), "V_x": None, "tau": None, "xi": None, "g0": make_g0(p)}
    if p.potential == POT_VX:
        d["V_x"] = make_vx(p)
    elif p.potential == POT_VTX:
        d["tau"], d["xi"] = make_vtx(p)
    return d


# ---------------------------------------------------------------------------
# Configs (BASELINE.json configs[0..4]).
# ---------------------------------------------------------------------------
def config(name: str, **over) -> Problem:
    base = {
        # C1: zero potential, Gaussian u0, N=2, ~200 cells, 100 steps, Robin.
        "C1": dict(dx=0.21, dt=5e-3, N=2, potential=POT_ZERO, transmission=TC_ROBIN,
                   robin_p=5.0, algorithm=ALG_NEW),
        # C2: V(x) = -x^2, N=10, NEW + GMRES, fine grid (parity variant 1e-4).
        "C2": dict(dx=1e-5, N=10, potential=POT_VX, algorithm=ALG_NEW),
        # C3: V(t,x) = 5tx, N=100, preconditioned GMRES.
        "C3": dict(dx=1e-5, N=100, potential=POT_VTX, algorithm=ALG_PRECOND),
        # C4: |u|^2, N=100, preconditioned fixed point, S0^2, soliton.
        "C4": dict(dx=1e-4, N=100, potential=POT_CUBIC, algorithm=ALG_PRECOND,
                   u0_kind="soliton"),
        # C5: scaling target, N=500 on the fine grid, V = -x^2, NEW.
        "C5": dict(dx=1e-5, N=500, potential=POT_VX, algorithm=ALG_NEW),
    }[name]
    base.update(over)
    p = Problem(**base)
    p.name = name
    return p
