"""Pins of the CPU oracle against what the paper and the mathematics fix.

Each test checks an oracle function against something other than itself:
closed forms, the paper's printed values (tests/golden/), dense brute force
on tiny grids, exact invariants, or a textbook routine (numpy LAPACK).
These run with -m "not gpu".
"""
import math
import os
from fractions import Fraction

import dataclasses

import numpy as np
import pytest

import oracle_checks as oc
import swr_inputs as si

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _tiny(**over):
    """A tiny problem (brute-force sized): (-3,3), 12 cells, 6 steps."""
    base = dict(a0=-3.0, b0=3.0, T=0.06, dx=0.5, dt=0.01, N=3, potential=si.POT_VX,
                transmission=si.TC_S02, algorithm=si.ALG_NEW, vx_kind="-x2", u0_kind="gaussian")
    base.update(over)
    return si.Problem(**base)


def _tiny_inputs(p):
    d = si.inputs(p)
    # a Gaussian centred in this small domain (x0 = 0 instead of -10)
    x = p.nodes()
    d["u0"] = np.exp(-(x * x) + 2j * x)
    return d


# ---------------------------------------------------------------- coefficients
def test_coeffs_match_paper_prefix(oracle_mod):
    """alpha, beta, gamma against the values printed at P:225-227."""
    rows = [l.split() for l in open(os.path.join(GOLDEN, "coeffs_P225.txt")) if l[0] != "#"]
    a, b, g = oracle_mod.coeffs(8)
    for r in rows:
        s = int(r[0])
        num, den = map(int, r[1].split("/"))
        assert a[s] == num / den
        assert b[s] == (-1) ** s * num / den
        if len(r) > 2:
            assert g[s] == int(r[2])


def test_coeffs_closed_form(oracle_mod):
    """alpha_{2k} = alpha_{2k+1} = C(2k,k)/4^k, the Taylor coefficients of
    (1-z^2)^{-1/2}; beta(z) = sqrt((1-z)/(1+z)) = (1-z)(1-z^2)^{-1/2}."""
    n = 600
    a, b, _ = oracle_mod.coeffs(n)
    for s in range(n):
        k = s // 2
        exact = Fraction(math.comb(2 * k, k), 4 ** k)
        assert abs(a[s] - float(exact)) <= 2e-16 * float(exact) * (1 + s / 8)
    # generating function of beta, evaluated by the truncated series at z=0.3
    z = 0.3
    series = sum(b[s] * z ** s for s in range(n))
    assert abs(series - math.sqrt((1 - z) / (1 + z))) < 1e-14


# ---------------------------------------------------------------- FEM
def test_fem_examples_and_invariants(oracle_mod):
    Md, Mo, Sd, So, Wd, Wo = oracle_mod.fem(2, 1.0)
    assert np.allclose(Md, [1 / 3, 1 / 3], rtol=0, atol=1e-16) and np.allclose(Mo, [1 / 6])
    Md, Mo, Sd, So, Wd, Wo = oracle_mod.fem(3, 1.0)
    assert np.allclose(Md, [1 / 3, 2 / 3, 1 / 3], atol=1e-16) and np.allclose(Sd, [1, 2, 1]) and np.allclose(So, [-1, -1])
    rng = np.random.default_rng(0)
    nn, h = 17, 0.37
    Md, Mo, Sd, So, _, _ = oracle_mod.fem(nn, h)
    M = np.diag(Md) + np.diag(Mo, 1) + np.diag(Mo, -1)
    S = np.diag(Sd) + np.diag(So, 1) + np.diag(So, -1)
    assert abs(M.sum() - (nn - 1) * h) < 1e-13            # partition of unity
    assert np.abs(S @ np.ones(nn)).max() < 1e-12          # constants in the kernel
    _, _, _, _, Wd1, Wo1 = oracle_mod.fem(nn, h, np.ones(nn))
    assert np.allclose(Wd1, Md, rtol=1e-15) and np.allclose(Wo1, Mo, rtol=1e-15)
    # weighted mass = exact integral of (linear interpolant of W) phi_k phi_l,
    # checked by 5-point Gauss-Legendre quadrature on every element
    W = rng.standard_normal(nn)
    _, _, _, _, Wd, Wo = oracle_mod.fem(nn, h, W)
    gx, gw = np.polynomial.legendre.leggauss(5)
    t, wq = (gx + 1) / 2, gw / 2 * h
    Q = np.zeros((nn, nn))
    for e in range(nn - 1):
        phi = np.stack([1 - t, t])
        w_lin = W[e] * (1 - t) + W[e + 1] * t
        for p_ in range(2):
            for q in range(2):
                Q[e + p_, e + q] += np.sum(wq * w_lin * phi[p_] * phi[q])
    assert np.allclose(np.diag(Q), Wd, rtol=0, atol=1e-14)
    assert np.allclose(np.diag(Q, 1), Wo, rtol=0, atol=1e-14)


# ---------------------------------------------------------------- Thomas
def test_thomas_vs_lapack(oracle_mod):
    st, x = oracle_mod.thomas(np.zeros(2), np.ones(2), np.zeros(2), np.array([1 + 2j, 3]))
    assert st == 0 and np.array_equal(x, [1 + 2j, 3])
    st, x = oracle_mod.thomas(np.zeros(3), 2 * np.ones(3), np.zeros(3), np.array([2, 4, 6.0]))
    assert np.array_equal(x, [1, 2, 3])
    rng = np.random.default_rng(1)
    for n in (8, 33, 64):
        lo, up = (rng.standard_normal(n) + 1j * rng.standard_normal(n) for _ in range(2))
        di = 4 + rng.standard_normal(n) + 1j * rng.standard_normal(n)
        lo[0] = up[-1] = 0
        A = np.diag(di) + np.diag(up[:-1], 1) + np.diag(lo[1:], -1)
        b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        st, x = oracle_mod.thomas(lo, di, up, b)
        assert st == 0
        assert np.linalg.norm(x - np.linalg.solve(A, b)) <= 1e-13 * np.linalg.norm(x)
    st, _ = oracle_mod.thomas(np.zeros(2), np.array([0.0, 1.0]), np.zeros(2), np.ones(2))
    assert st == 3  # zero pivot


# ---------------------------------------------------------------- GMRES driver
@pytest.mark.parametrize("gs", [1, 2])
def test_gmres_dense(oracle_mod, gs):
    b = np.array([1, 2, 3], np.complex128)
    st, x, it, _ = oracle_mod.gmres_dense(np.eye(3), b, gs_passes=gs)
    assert st == 0 and it == 1 and np.allclose(x, b, rtol=1e-15)
    st, x, it, _ = oracle_mod.gmres_dense(np.diag([1.0, 2, 3]), b, gs_passes=gs)
    assert st == 0 and np.allclose(x, 1, rtol=1e-10)
    rng = np.random.default_rng(2)
    A = np.eye(40) * 3 + (rng.standard_normal((40, 40)) + 1j * rng.standard_normal((40, 40))) / 8
    b = rng.standard_normal(40) + 1j * rng.standard_normal(40)
    st, x, it, hist = oracle_mod.gmres_dense(A, b, tol=1e-12, restart=7, gs_passes=gs)
    xs = np.linalg.solve(A, b)
    assert st == 0 and np.linalg.norm(x - xs) < 1e-10 * np.linalg.norm(xs)
    assert np.linalg.norm(b - A @ x) <= 1.01e-12 * np.linalg.norm(b) * 10
    assert len(hist) == it and hist[-1] <= 1e-12 * np.linalg.norm(b)


def test_bicgstab_dense(oracle_mod):
    """BiCGStab converges to numpy's solution.  Finite termination: its
    residual is Q_k(A) P_k(A) r0 with P_k the BiCG polynomial, which
    annihilates r0 once k reaches the number of distinct eigenvalues of a
    normal A: one iteration (at the half step) for A = 2I, two for two
    distinct eigenvalues."""
    rng = np.random.default_rng(4)
    A = np.eye(30) * 3 + (rng.standard_normal((30, 30)) + 1j * rng.standard_normal((30, 30))) / 6
    b = rng.standard_normal(30) + 1j * rng.standard_normal(30)
    st, x, it, hist = oracle_mod.bicgstab_dense(A, b, tol=1e-12)
    xs = np.linalg.solve(A, b)
    assert st == 0 and np.linalg.norm(x - xs) < 1e-10 * np.linalg.norm(xs)
    assert np.linalg.norm(b - A @ x) <= 1e-11 * np.linalg.norm(b)
    assert len(hist) == it and hist[-1] <= 1e-12 * np.linalg.norm(b)
    d = np.array([1.0] * 5 + [2.0] * 5)
    b2 = rng.standard_normal(10) + 1j * rng.standard_normal(10)
    st, x, it, _ = oracle_mod.bicgstab_dense(np.diag(d), b2, tol=1e-13)
    assert st == 0 and it == 2 and np.allclose(x, b2 / d, rtol=1e-12)
    st, x, it, _ = oracle_mod.bicgstab_dense(2 * np.eye(10), b2, tol=1e-13)
    assert st == 0 and it == 1 and np.allclose(x, b2 / 2, rtol=1e-14)


@pytest.mark.parametrize("gs", [1, 2])
def test_gmres_minimal_residual(oracle_mod, gs):
    """Unrestarted GMRES minimises ||b - A x|| over the Krylov space: the
    residual estimate after k steps equals min_y ||b - A K_k y|| with K_k an
    orthonormal basis of span{b, Ab, ..., A^{k-1} b} from numpy's QR of the
    explicit power basis (independent of the Arnoldi/Givens code)."""
    rng = np.random.default_rng(11)
    n = 12
    A = np.eye(n) * 2 + (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / 6
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    st, x, it, hist = oracle_mod.gmres_dense(A, b, tol=1e-13, restart=n, maxit=n, gs_passes=gs)
    for k in range(1, min(it, 8) + 1):
        P = np.stack([np.linalg.matrix_power(A, i) @ b for i in range(k)], axis=1)
        Q, _ = np.linalg.qr(P)
        y, *_ = np.linalg.lstsq(A @ Q, b, rcond=None)
        rmin = np.linalg.norm(b - A @ Q @ y)
        assert abs(hist[k - 1] - rmin) <= 1e-9 * np.linalg.norm(b), (k, hist[k - 1], rmin)


# ---------------------------------------------------------------- monodomain
@pytest.mark.parametrize("pot", [si.POT_ZERO, si.POT_VX, si.POT_VTX])
def test_monodomain_mass_conservation(oracle_mod, pot):
    """CN with a real potential conserves u^* M u exactly (A Hermitian part
    vanishes): drift <= 1e-12 relative over the whole window."""
    p = si.Problem(a0=-15, b0=5, T=0.05, dx=0.01, dt=1e-3, N=1, potential=pot)
    o = oracle_mod.Oracle(p, si.inputs(p))
    st, uT, _ = o.monodomain()
    assert st == 0
    Md, Mo, *_ = oracle_mod.fem(p.Nx + 1, p.dx)
    mass = lambda u: np.real(np.vdot(u, Md * u + np.r_[Mo * u[1:], 0] + np.r_[0, Mo * u[:-1]]))
    u0 = si.make_u0(p)
    assert abs(mass(uT) - mass(u0)) <= 1e-12 * mass(u0)


def test_monodomain_nl_mass_conservation(oracle_mod):
    """Duran-Sanz-Serna with the symmetric load M_{|z|^2} z (reading A3)
    conserves the discrete mass up to the fixed-point tolerance."""
    p = si.Problem(a0=-15, b0=5, T=0.05, dx=0.01, dt=1e-3, N=1, potential=si.POT_CUBIC,
                   u0_kind="soliton")
    o = oracle_mod.Oracle(p, si.inputs(p))
    st, uT, fp = o.monodomain()
    assert st == 0 and 1 <= fp <= 50
    Md, Mo, *_ = oracle_mod.fem(p.Nx + 1, p.dx)
    mass = lambda u: np.real(np.vdot(u, Md * u + np.r_[Mo * u[1:], 0] + np.r_[0, Mo * u[:-1]]))
    u0 = si.make_u0(p)
    assert abs(mass(uT) - mass(u0)) <= 1e-11 * mass(u0)


def _gauss_exact(x, t, x0=-10.0, k=20.0):
    """Free Schrodinger (i u_t + u_xx = 0) from exp(-y^2 + i k y), y = x-x0."""
    y = x - x0
    z = 1 + 4j * t
    return z ** -0.5 * np.exp((-(y * y) + 1j * k * y - 1j * k * k * t) / z)


def test_gaussian_closed_form_order(oracle_mod):
    """V = 0: error vs the closed-form Gaussian decreases at order >= 1.9
    along the refinement ladder (CN in time, P1 in space) before the packet
    reaches the Neumann ends."""
    errs = []
    for f in (1, 2, 4):
        p = si.Problem(a0=-16, b0=4, T=0.02, dx=4e-3 / f, dt=4e-4 / f, N=1, potential=si.POT_ZERO)
        o = oracle_mod.Oracle(p, si.inputs(p))
        st, uT, _ = o.monodomain()
        ex = _gauss_exact(p.nodes(), p.T)
        errs.append(np.linalg.norm(uT - ex) / np.linalg.norm(ex))
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert all(o_ >= 1.9 for o_ in orders), (errs, orders)
    assert errs[-1] < 2e-2


def test_n1_is_monodomain_bitwise(oracle_mod):
    p = _tiny(N=1)
    o = oracle_mod.Oracle(p, _tiny_inputs(p))
    r = o.solve()
    st, um, _ = o.monodomain()
    assert r["status"] == 0 and r["iterations"] == 0
    assert np.array_equal(r["uT"], um)


# ---------------------------------------------------------------- interface
@pytest.mark.parametrize("tc", [si.TC_ROBIN, si.TC_S02])
def test_R_is_affine_with_toeplitz_L(oracle_mod, tc):
    """Props 1-4: R(g) = L g + d for V(x), with L built from first columns."""
    p = _tiny(transmission=tc, N=4, dx=0.25)
    o = oracle_mod.Oracle(p, _tiny_inputs(p))
    rng = np.random.default_rng(3)
    g = rng.standard_normal(o.ng) + 1j * rng.standard_normal(o.ng)
    d = o.apply_R(None)
    X = o.build_L()
    lhs = o.apply_R(g)
    rhs = o.apply_L(X, g) + d
    assert np.linalg.norm(lhs - rhs) <= 1e-13 * np.linalg.norm(lhs)


def test_dense_interface_matrix_brute_force(oracle_mod):
    """Probe every column of R_0 = R(.; u0=0): the dense L equals the
    block-Toeplitz matrix rebuilt from the first columns, it is block lower
    triangular in time, and a dense solve of (I-L)g = d matches GMRES."""
    p = _tiny(N=3)
    o = oracle_mod.Oracle(p, _tiny_inputs(p))
    n = o.ng
    Ld = np.zeros((n, n), np.complex128)
    for c in range(n):
        e = np.zeros(n, np.complex128)
        e[c] = 1
        Ld[:, c] = o.apply_R(e, use_u0=False)
    X = o.build_L()
    Lt = np.zeros_like(Ld)
    for c in range(n):
        e = np.zeros(n, np.complex128)
        e[c] = 1
        Lt[:, c] = o.apply_L(X, e)
    assert np.abs(Ld - Lt).max() <= 1e-13 * np.abs(Ld).max()
    NT = p.NT
    for si_ in range(2 * p.N - 2):
        for so in range(2 * p.N - 2):
            blk = Ld[so * NT:(so + 1) * NT, si_ * NT:(si_ + 1) * NT]
            assert np.abs(np.triu(blk, 1)).max() == 0.0          # causal
    d = o.apply_R(None)
    g_dense = np.linalg.solve(np.eye(n) - Ld, d)
    r = o.solve()
    assert r["converged"]
    cond = np.linalg.cond(np.eye(n) - Ld)
    assert np.linalg.norm(r["g"] - g_dense) <= 10 * p.tol * cond * np.linalg.norm(g_dense)


def test_toeplitz_shift_bitwise(oracle_mod):
    """Prop. 3-4 with u0 = 0: an impulse at n=2 gives the n=1 response
    shifted by one step, bitwise (reading A14); every interior block of
    L0 is identical (translation invariance of the V = 0 problem) and
    mirror-symmetric (X^{j,1} = X^{j,4}, X^{j,2} = X^{j,3})."""
    p = _tiny(N=5, dx=0.3, T=0.08)
    o = oracle_mod.Oracle(p, _tiny_inputs(p))
    for j in (1, 2, 5):
        e1 = np.zeros(p.NT, np.complex128); e1[0] = 1
        e2 = np.zeros(p.NT, np.complex128); e2[1] = 1
        if j < p.N:
            _, a1, b1, _, _ = o.march(j, None, e1, use_u0=False)
            _, a2, b2, _, _ = o.march(j, None, e2, use_u0=False)
        else:
            _, a1, b1, _, _ = o.march(j, e1, None, use_u0=False)
            _, a2, b2, _, _ = o.march(j, e2, None, use_u0=False)
        assert np.array_equal(a2[1:], a1[:-1]) and a2[0] == 0
        assert np.array_equal(b2[1:], b1[:-1]) and b2[0] == 0
    X0 = o.build_L(force_zero=True)
    for j in range(3, p.N):
        assert np.array_equal(X0[j - 1], X0[1])
    sc = np.abs(X0[1]).max()
    assert np.abs(X0[1, 0] - X0[1, 3]).max() <= 1e-13 * sc
    assert np.abs(X0[1, 1] - X0[1, 2]).max() <= 1e-13 * sc
    # reading A13: the "-1" of x^{j,1}_{n,s} sits only at lag 0
    d = p.NT
    assert X0.shape == (p.N, 4, d)


def test_dot_is_order_fixed_inner_product(oracle_mod):
    p = _tiny(N=4, dx=0.25)
    o = oracle_mod.Oracle(p, _tiny_inputs(p))
    rng = np.random.default_rng(4)
    x, y = (rng.standard_normal(o.ng) + 1j * rng.standard_normal(o.ng) for _ in range(2))
    assert abs(o.dot(x, y) - np.vdot(x, y)) <= 1e-14 * np.linalg.norm(x) * np.linalg.norm(y)


# ---------------------------------------------------------------- algorithms
@pytest.mark.parametrize("tc,pot", [(si.TC_ROBIN, si.POT_ZERO), (si.TC_S02, si.POT_ZERO),
                                    (si.TC_S02, si.POT_VX), (si.TC_ROBIN, si.POT_VX)])
def test_new_algorithm_equals_monodomain(oracle_mod, tc, pot):
    """Converged SWR = the single-domain CN/FEM solution (c0 != 0 makes the
    FEM fluxes cancel): within tol * a modest factor."""
    p = si.config("C1", transmission=tc, potential=pot, N=4)
    o = oracle_mod.Oracle(p, si.inputs(p))
    r = o.solve()
    st, um, _ = o.monodomain()
    assert r["status"] == 0 and r["converged"]
    assert np.linalg.norm(r["uT"] - um) <= 1e-8 * np.linalg.norm(um)


@pytest.mark.parametrize("alg,kry", [(si.ALG_NEW, si.KRY_BICGSTAB), (si.ALG_NEW, si.KRY_FIXED_POINT),
                                     (si.ALG_CLASSICAL, si.KRY_FIXED_POINT), (si.ALG_CLASSICAL, si.KRY_GMRES),
                                     (si.ALG_CLASSICAL, si.KRY_BICGSTAB), (si.ALG_PRECOND, si.KRY_BICGSTAB)])
def test_solver_variants_equal_monodomain(oracle_mod, alg, kry):
    """Every interface solver of the paper (Algorithms 1-3 with fixed point,
    GMRES or BiCGStab) converges to the single-domain
    solution (V(x) for NEW/CLASSICAL, V(t,x) for PRECOND)."""
    pot = si.POT_VTX if alg == si.ALG_PRECOND else si.POT_VX
    p = si.config("C1", transmission=si.TC_S02, potential=pot, N=4, algorithm=alg, krylov=kry)
    o = oracle_mod.Oracle(p, si.inputs(p))
    r = o.solve()
    st, um, _ = o.monodomain()
    assert r["status"] == 0 and r["converged"], r["status"]
    assert np.linalg.norm(r["uT"] - um) <= 1e-8 * np.linalg.norm(um)


def test_fixed_point_iterations_agree(oracle_mod):
    """The fixed points of Algorithm 1 (g <- R(g)) and of the new algorithm
    (g <- d + L g) are the same iteration in exact arithmetic (R(g) = L g + d,
    Props 1-4): equal iteration counts and histories to rounding."""
    ps = [si.config("C1", transmission=si.TC_S02, potential=si.POT_VX, N=4, algorithm=a,
                    krylov=si.KRY_FIXED_POINT) for a in (si.ALG_NEW, si.ALG_CLASSICAL)]
    rs = [oracle_mod.Oracle(q, si.inputs(q)).solve() for q in ps]
    assert rs[0]["iterations"] == rs[1]["iterations"]
    h0, h1 = rs[0]["history"], rs[1]["history"]
    # the two evaluations of R differ by rounding only: |diff| at the scale of the first step
    assert np.abs(h0 - h1).max() <= 1e-12 * h0[0]


def test_precond_exact_for_zero_potential(oracle_mod):
    """With V = 0, P = I - L0 = I - L, so P^{-1}(I - L) = I: one outer
    iteration."""
    p = si.config("C1", transmission=si.TC_S02, potential=si.POT_ZERO, algorithm=si.ALG_PRECOND, N=4)
    o = oracle_mod.Oracle(p, si.inputs(p))
    r = o.solve()
    assert r["status"] == 0 and r["iterations"] == 1


@pytest.mark.parametrize("pot,u0", [(si.POT_VTX, "gaussian"), (si.POT_CUBIC, "soliton")])
def test_precond_equals_monodomain(oracle_mod, pot, u0):
    p = si.config("C1", transmission=si.TC_S02, potential=pot, algorithm=si.ALG_PRECOND, N=4, u0_kind=u0)
    o = oracle_mod.Oracle(p, si.inputs(p))
    r = o.solve()
    st, um, _ = o.monodomain()
    assert r["status"] == 0 and r["converged"]
    assert np.linalg.norm(r["uT"] - um) <= 1e-8 * np.linalg.norm(um)


def test_new_rejects_time_dependent(oracle_mod):
    p = si.config("C1", potential=si.POT_VTX, algorithm=si.ALG_NEW)
    o = oracle_mod.Oracle(p, si.inputs(p))
    assert o.solve()["status"] == 6


HIGHER_TC = [si.TC_S03, si.TC_S04, si.TC_S12, si.TC_S14]


@pytest.mark.parametrize("tc", HIGHER_TC)
def test_higher_order_tc_reduce_to_s02_for_zero_potential(oracle_mod, tc):
    """With V = 0 the potential and gauge operators of every order reduce to
    S0^2 (the extra terms carry V, d_n V or the phase int V):
    the interface operator d, L of the new algorithm agree to rounding."""
    p = si.config("C1", transmission=si.TC_S02, potential=si.POT_ZERO, N=4)
    q = si.config("C1", transmission=tc, potential=si.POT_ZERO, N=4)
    o, oq = oracle_mod.Oracle(p, si.inputs(p)), oracle_mod.Oracle(q, si.inputs(q))
    d0, dq = o.apply_R(np.zeros(o.ng), use_u0=True), oq.apply_R(np.zeros(oq.ng), use_u0=True)
    assert np.linalg.norm(dq - d0) <= 1e-13 * np.linalg.norm(d0)
    X0, Xq = o.build_L(), oq.build_L()
    assert np.abs(Xq - X0).max() <= 1e-13 * np.abs(X0).max()


@pytest.mark.parametrize("tc", HIGHER_TC)
def test_higher_order_tc_converge_to_monodomain(oracle_mod, tc):
    """Whatever the transmission operator, the converged SWR solution is the
    single-domain one (the operator only changes the convergence): pins that
    the leading coefficient on the matrix row, the history and the emitted
    traces of eq. (8) are the same operator."""
    p = si.config("C1", transmission=tc, potential=si.POT_VX, N=4)
    o = oracle_mod.Oracle(p, si.inputs(p))
    r = o.solve()
    st, um, _ = o.monodomain()
    assert r["status"] == 0 and r["converged"]
    assert np.linalg.norm(r["uT"] - um) <= 1e-8 * np.linalg.norm(um)


@pytest.mark.parametrize("tc", [si.TC_ROBIN, si.TC_S02])
def test_pinv_causal_inverts_I_minus_L0(oracle_mod, tc):
    """the causal forward substitution is the exact inverse of
    P = I - L0: applying I - L0 by the independent convolution
    of or_apply_L to its output returns the input to rounding."""
    p = si.config("C1", N=5, potential=si.POT_VTX, algorithm=si.ALG_PRECOND, transmission=tc)
    o = oracle_mod.Oracle(p, si.inputs(p))
    X = o.build_L(force_zero=True)
    rng = np.random.default_rng(3)
    y = rng.standard_normal(o.ng) + 1j * rng.standard_normal(o.ng)
    x = o.pinv_causal(X, y)
    assert np.linalg.norm(x - o.apply_L(X, x) - y) <= 1e-13 * np.linalg.norm(y)


@pytest.mark.parametrize("pot,kry", [(si.POT_VTX, si.KRY_GMRES), (si.POT_VTX, si.KRY_BICGSTAB),
                                     (si.POT_CUBIC, si.KRY_FIXED_POINT)])
def test_pinv_exact_equals_inner_krylov(oracle_mod, pot, kry):
    """The exact P^{-1} changes rounding only: the preconditioned algorithms
    take the same outer iterations as with the inner Krylov P^{-1} (tolerance
    1e-12), no inner iterations, and reach the monodomain solution."""
    p = si.config("C1", N=5, potential=pot, algorithm=si.ALG_PRECOND, transmission=si.TC_S02, krylov=kry)
    q = dataclasses.replace(p, pinv_exact=1)
    ra = oracle_mod.Oracle(p, si.inputs(p)).solve()
    oq = oracle_mod.Oracle(q, si.inputs(q))
    rb = oq.solve()
    assert ra["status"] == 0 and rb["status"] == 0 and rb["converged"]
    assert rb["iterations"] == ra["iterations"] and rb["inner_iterations"] == 0 < ra["inner_iterations"]
    assert np.linalg.norm(rb["uT"] - ra["uT"]) <= 1e-10 * np.linalg.norm(ra["uT"])
    st, um, _ = oq.monodomain()
    assert np.linalg.norm(rb["uT"] - um) <= 1e-8 * np.linalg.norm(um)


PADE_TC = [si.TC_S22, si.TC_S24]


@pytest.mark.parametrize("m", [1, 5, 20, 100])
def test_pade_coefficients_approximate_sqrt(oracle_mod, m):
    """Reading A26: sqrt(z) ~ R_m(z) = sum_s a_s - sum_s a_s d_s/(z + d_s)
    (the form of P:243-247) with the branch cut rotated by pi/4.  R_m is
    exact at the rotation point, R_m(e^{i pi/4}) = e^{i pi/8}, for every m,
    its poles -d_s lie on the rotated cut, and R_m converges to numpy's sqrt
    away from that cut (including z = 2i/dt, where the discrete operator
    evaluates it) as m grows."""
    a, d = oracle_mod.pade_coeffs(m)
    assert d[0] == 0.0
    assert np.allclose(np.angle(d[1:]), np.pi / 4) and np.all(np.diff(np.abs(d[1:])) > 0)

    def R(z):
        return a.sum() - np.sum(a[1:] * d[1:] / (z + d[1:]))

    assert abs(R(np.exp(1j * np.pi / 4)) - np.exp(1j * np.pi / 8)) <= 1e-13
    z = np.array([0.3, 2.0, 1 + 3j, 5j, 0.5 - 2j])
    err = max(abs(R(zz) - np.sqrt(zz)) / abs(np.sqrt(zz)) for zz in z)
    assert err <= {1: 1.0, 5: 1e-2, 20: 1e-8, 100: 1e-12}[m], err
    # far out on the imaginary axis (z = 2i/dt at dt = 1e-3) the error still
    # falls with m: 0.94 / 0.78 / 0.32 / 4.9e-4 for m = 1 / 5 / 20 / 100
    e2 = abs(R(2000j) - np.sqrt(2000j)) / abs(np.sqrt(2000j))
    assert e2 <= {1: 1.0, 5: 0.9, 20: 0.4, 100: 1e-3}[m], e2


@pytest.mark.parametrize("tc", PADE_TC)
@pytest.mark.parametrize("m", [3, 20])
def test_pade_operator_symbol(oracle_mod, tc, m):
    """The auxiliary recursions of P:248-265 are Crank-Nicolson for
    (i d_t + W + d_s) phi = v on the v-form (midpoint) sequence, so in the
    z-transform (tau = one-step delay, z_d = (2i/dt)(1 - tau)/(1 + tau)):
    S2^2 = -i R_m(z_d + W) and S2^4 = S2^2 + (d_n W/4)/(z_d + W).
    The impulse response of the oracle's operator, summed as a power series,
    matches the rational symbol evaluated directly (pins D_s, the 2i/dt
    factors, the phi/psi updates and the sign conventions)."""
    p = si.config("C1", transmission=tc, potential=si.POT_VX, pade_m=m)
    o = oracle_mod.Oracle(p, si.inputs(p))
    a, d = oracle_mod.pade_coeffs(m)
    nst = 300
    v = np.zeros(nst + 1, np.complex128)
    v[1] = 1.0
    for W, dnW in ((0.0, 0.0), (-3.0, 1.7), (2.0, -0.8)):
        k = o.tc_apply(v, W, dnW)
        for tau in (0.3, -0.5, 0.4j):
            zd = (2j / p.dt) * (1 - tau) / (1 + tau) + W
            ref = -1j * (a.sum() - np.sum(a[1:] * d[1:] / (zd + d[1:])))
            if tc == si.TC_S24:
                ref += (dnW / 4.0) / zd
            got = np.sum(k * tau ** np.arange(nst))
            assert abs(got - ref) <= 1e-13 * abs(ref), (W, dnW, tau)


def test_pade_tends_to_s02_without_potential(oracle_mod):
    """With W = 0, S2^{2,m} -> S0^2 = -i sqrt(z_d) (the beta
    convolution) as m grows, wherever the Pade approximant of sqrt converges
    on the symbol's range (dt = 1 keeps z_d = O(1)); m = 100 agrees to
    rounding on a random trace sequence, m = 20 only approximately."""
    base = si.config("C1", T=40.0, dt=1.0)
    rng = np.random.default_rng(1)
    v = rng.standard_normal(41) + 1j * rng.standard_normal(41)
    v[0] = 0.0   # v_0 enters S0^2 but not the Pade recursions (phi_0 = 0)
    ref = oracle_mod.Oracle(dataclasses.replace(base, transmission=si.TC_S02), si.inputs(base)).tc_apply(v)
    err = {}
    for m in (20, 100):
        q = dataclasses.replace(base, transmission=si.TC_S22, pade_m=m)
        err[m] = np.abs(oracle_mod.Oracle(q, si.inputs(q)).tc_apply(v) - ref).max() / np.abs(ref).max()
    assert err[100] <= 1e-12 < err[20], err


@pytest.mark.parametrize("tc", PADE_TC)
def test_pade_tc_converges_to_monodomain(oracle_mod, tc):
    """The Pade operators change the convergence, not the limit: the SWR
    solution equals the single-domain one; and the iteration count falls as
    m grows (the paper's observation)."""
    its = []
    for m in (5, 20, 50):
        p = si.config("C1", transmission=tc, potential=si.POT_VX, N=4, pade_m=m)
        o = oracle_mod.Oracle(p, si.inputs(p))
        r = o.solve()
        st, um, _ = o.monodomain()
        assert r["status"] == 0 and r["converged"]
        assert np.linalg.norm(r["uT"] - um) <= 1e-8 * np.linalg.norm(um)
        its.append(r["iterations"])
    assert its[0] > its[1] > its[2], its


def test_paper_table6_fixed_point_counts(oracle_mod):
    """Pin to the paper's printed numbers (tests/golden/table6_fixed_point.txt,
    all 12 fixed-point rows of Table 6): the fixed-point iteration
    counts of the new algorithm on the paper's problem (N = 2, V = -x^2,
    random g0) for every transmission operator (S0^2, S0^3, S0^4, S1^2, S1^4,
    the six Pade rows of reading A26, Robin p = 44), each within the stated
    per-row tolerance (0 for 9 rows).  Pins the operators, the interface
    operator and the fixed point together."""
    here = os.path.join(os.path.dirname(__file__), "golden", "table6_fixed_point.txt")
    rows = [l.split() for l in open(here) if l.strip() and not l.startswith("#")]
    assert len(rows) == 12
    tcs = {"S02": si.TC_S02, "S03": si.TC_S03, "S04": si.TC_S04, "S12": si.TC_S12, "S14": si.TC_S14,
           "S22": si.TC_S22, "S24": si.TC_S24, "ROBIN": si.TC_ROBIN}
    got = []
    try:
        oracle_mod.set_threads(2)   # N = 2: the two subdomains march in parallel (bitwise equal)
        for name, m, pr, n_iter, dx, tol in rows:
            p = si.config("C2", N=2, dx=float(dx), g0_random=True, krylov=si.KRY_FIXED_POINT, transmission=tcs[name],
                          pade_m=int(m) if int(m) > 0 else 20, robin_p=float(pr) if float(pr) > 0 else 5.0)
            r = oracle_mod.Oracle(p, si.inputs(p)).solve()
            got.append((name, m, r["iterations"], int(n_iter)))
            assert r["status"] == 0 and abs(r["iterations"] - int(n_iter)) <= int(tol), got
    finally:
        oracle_mod.set_threads(1)


def test_gauge_tc_is_transparent_for_constant_potential(oracle_mod):
    """For a constant potential V0 the solution is e^{i V0 t} times a free one
    and the gauge operator S1^2 = e^{-i pi/4} e^{i calV} d_t^{1/2} e^{-i calV}
     absorbs a packet as well as S0^2 does without a potential,
    while S0^2, blind to V0, reflects more (same set-up as the S0^2 pin)."""
    out = {}
    for tc in (si.TC_S12, si.TC_S02):
        p = si.Problem(a0=-16, b0=4, T=0.2, dx=2e-3, dt=2e-4, N=2, potential=si.POT_VX, vx_kind="const",
                       transmission=tc)
        o = oracle_mod.Oracle(p, si.inputs(p))
        st, _, _, uT, _ = o.march(1, None, None, use_u0=True)
        q = si.Problem(a0=-16, b0=24, T=0.2, dx=2e-3, dt=2e-4, N=1, potential=si.POT_VX, vx_kind="const")
        st2, ub, _ = oracle_mod.Oracle(q, si.inputs(q)).monodomain()
        out[tc] = np.abs(uT - ub[: p.Nj]).max()
    assert out[si.TC_S12] <= 1e-4, out
    assert out[si.TC_S02] >= 10 * out[si.TC_S12], out


def test_s02_transmission_is_transparent(oracle_mod):
    """S0^2 is the discrete transparent condition of the free equation
    (P:146-159): a Gaussian packet leaving subdomain 1 through b_1
    with zero incoming flux is absorbed (reflection <= 1e-4 of the packet
    amplitude vs the solution on a larger domain), whereas the memoryless
    Robin condition reflects O(1).  Pins the beta history sum and its index
    range (a shifted or mis-signed history term reflects strongly)."""
    out = {}
    for tc in (si.TC_S02, si.TC_ROBIN):
        p = si.Problem(a0=-16, b0=4, T=0.2, dx=2e-3, dt=2e-4, N=2, potential=si.POT_ZERO,
                       transmission=tc, robin_p=40.0)
        o = oracle_mod.Oracle(p, si.inputs(p))
        st, _, _, uT, _ = o.march(1, None, None, use_u0=True)
        q = si.Problem(a0=-16, b0=24, T=0.2, dx=2e-3, dt=2e-4, N=1, potential=si.POT_ZERO)
        st2, ub, _ = oracle_mod.Oracle(q, si.inputs(q)).monodomain()
        out[tc] = np.abs(uT - ub[: p.Nj]).max()
    assert out[si.TC_S02] <= 1e-4
    assert out[si.TC_ROBIN] >= 0.1


# ---------------------------------------------------------------- closed forms (round 2)
def test_nl_soliton_closed_form_order(oracle_mod):
    """f(u) = |u|^2 against the exact soliton u = 2 sech(sqrt2 (x +
    10 - 40 t)) e^{i (20 (x+10) - 398 t)} (the paper's u0): observed
    order >= 1.9 along a dt, dx ladder.  Pins the sign and the weighting of
    the load M_{|z|^2} z (a mis-signed load defocuses the soliton: O(1)
    error, tests/test_oracle_mutants.py) and the inner fixed point."""
    errs = oc.nl_soliton_errors(oracle_mod)
    assert min(oc.orders(errs)) >= 1.9, errs
    assert errs[-1] < 1e-3, errs


def test_linear_potential_closed_form_order(oracle_mod):
    """V(t, x) = E0 t x (the paper's V = 5tx family) against its exact
    solution (the gauge u = e^{i(a x + b)} w(x - c, t) of a free Gaussian,
    tests/oracle_checks.py): observed order >= 1.9.  Pins W_n = (V_n +
    V_{n-1})/2: the potential sampled at t_n instead is a first-
    order error (order ~1, tests/test_oracle_mutants.py)."""
    errs = oc.linear_potential_errors(oracle_mod)
    assert min(oc.orders(errs)) >= 1.9, errs
    assert errs[-1] < 1e-5, errs


@pytest.mark.parametrize("tc", [si.TC_S02, si.TC_S03, si.TC_S04, si.TC_S12, si.TC_S14])
def test_transmission_operator_symbols(oracle_mod, tc):
    """The discrete operators S0^2, S0^3, S0^4, S1^2, S1^4 are the
    continuous ones under the Crank-Nicolson symbol map d_t ->
    s_d(tau) = (2/dt)(1 - tau)/(1 + tau) (gauge: tau -> tau e^{i W dt}):
    the power series of the oracle's impulse response equals the closed-form
    symbol to rounding, for several W, d_n W and tau.  Pins every coefficient
    and sign of the alpha, beta, gamma convolutions and the gauge phase."""
    assert oc.tc_symbol_error(oracle_mod, tc) <= 1e-13


def test_threaded_oracle_is_bitwise_single_threaded(oracle_mod):
    """or_set_threads(P) parallelises independent subdomains and element
    ranges only: NEW and the preconditioned NL algorithm give bitwise the
    single-thread results (u(T), residual history, counts)."""
    cases = [si.Problem(dx=2e-3, dt=5e-3, N=12, potential=si.POT_VX),
             si.Problem(dx=4e-3, dt=5e-3, N=10, potential=si.POT_CUBIC, algorithm=si.ALG_PRECOND,
                        u0_kind="soliton")]
    try:
        for p in cases:
            res = []
            for t in (1, 5):
                oracle_mod.set_threads(t)
                res.append(oracle_mod.Oracle(p, si.inputs(p)).solve())
            a, b = res
            assert a["status"] == b["status"] == 0
            assert a["iterations"] == b["iterations"] and a["inner_iterations"] == b["inner_iterations"]
            assert np.array_equal(a["uT"], b["uT"]) and np.array_equal(a["history"], b["history"])
    finally:
        oracle_mod.set_threads(1)


def test_pade_tc_is_transparent(oracle_mod):
    """Independent of the Table 6 counts that selected reading A26: the Pade
    operator S2^{2,m} approximates the transparent condition -i sqrt(i d_t)
    (P:173-177), so a packet leaving subdomain 1 with zero incoming flux is
    absorbed better as m grows, reaching the S0^2 (exact discrete transparent
    condition) level by m = 100 (same set-up as the S0^2 pin)."""
    refl = {m: oc.transparency(oracle_mod, si.TC_S22, pade_m=m) for m in (5, 20, 50, 100)}
    s02 = oc.transparency(oracle_mod, si.TC_S02)
    assert refl[5] > refl[20] > refl[50] > refl[100], refl
    assert refl[50] <= 5e-4 and refl[100] <= 1.1 * s02, (refl, s02)
