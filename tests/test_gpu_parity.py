"""Parity of the CUDA path (libswr.so through the C ABI) with the CPU oracle.

Same seeded inputs (swr_inputs) on both sides; element-by-element relative
L2 comparisons.  Tolerances ("Parity bar"): a single march or
interface-operator build <= 1e-12 relative (rounding order differs: FMA,
scan-reassociated carries); converged solutions <= 1e-10 relative with equal
GMRES iteration counts (BASELINE.json north_star).
"""
import numpy as np
import pytest

import swr_inputs as si

pytestmark = pytest.mark.gpu


def rel(a, b, scale=0.0):
    """||a - b|| / max(||b||, scale sqrt(len)): relative L2, with a floor for
    outputs much smaller than the data they are computed from (e.g. d, whose
    entries are the Gaussian's tail at the interfaces, ~1e-5 of max|u0|)."""
    a = np.asarray(a)
    b = np.asarray(b)
    nb = max(np.linalg.norm(b), scale * np.sqrt(b.size))
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def gpu():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1503_02564_b200 as pkg
    pkg.lib()  # loads libswr.so or raises
    return pkg


def _pair(oracle_mod, gpu, p, arrays=None):
    arrays = arrays if arrays is not None else si.inputs(p)
    return oracle_mod.Oracle(p, arrays), gpu.SWR(p, arrays)


CASES = [
    ("C1-robin", si.config("C1")),
    ("C1-s02", si.config("C1", transmission=si.TC_S02)),
    ("C1-vx-s02-N4", si.config("C1", transmission=si.TC_S02, potential=si.POT_VX, N=4)),
    ("C1-vx-robin-N5", si.config("C1", transmission=si.TC_ROBIN, potential=si.POT_VX, N=5, robin_p=19.0)),
    # several CTAs and a ragged last CTA: N_j = 421, 1001
    ("mid-N100", si.Problem(dx=1e-3, dt=5e-3, N=100, potential=si.POT_VX, transmission=si.TC_S02)),
    ("mid-N42", si.Problem(dx=1e-3, dt=5e-3, N=42, potential=si.POT_VX, transmission=si.TC_S02)),
]


@pytest.mark.parametrize("name,p", CASES, ids=[c[0] for c in CASES])
def test_sweep_R_parity(oracle_mod, gpu, name, p):
    """One sweep R(g; u0) with a random g and the assembled u(T)."""
    import torch
    o, g_ = _pair(oracle_mod, gpu, p)
    rng = np.random.default_rng(11)
    g = rng.standard_normal(o.ng) + 1j * rng.standard_normal(o.ng)
    Rg_o = o.apply_R(g, use_u0=True)
    Rg_g, uT_g = g_.apply_R(torch.as_tensor(g, device="cuda"), use_u0=True, want_uT=True)
    assert rel(Rg_g.cpu().numpy(), Rg_o) <= 1e-12
    # u(T) of the same sweep, assembled like the final sweep
    uT_o = np.zeros(p.Nx + 1, np.complex128)
    cnt = np.zeros(p.Nx + 1)
    m = p.Nx // p.N
    for j in range(1, p.N + 1):
        lin = g[(2 * j - 3) * p.NT:(2 * j - 2) * p.NT] if j >= 2 else None
        rin = g[(2 * j - 2) * p.NT:(2 * j - 1) * p.NT] if j <= p.N - 1 else None
        st, _, _, uloc, _ = o.march(j, lin, rin, use_u0=True)
        uT_o[(j - 1) * m:(j - 1) * m + p.Nj] += uloc
        cnt[(j - 1) * m:(j - 1) * m + p.Nj] += 1
    uT_o /= cnt
    assert rel(uT_g.cpu().numpy(), uT_o) <= 1e-12


@pytest.mark.parametrize("name,p", CASES, ids=[c[0] for c in CASES])
def test_interface_operator_parity(oracle_mod, gpu, name, p):
    """d = R(0) and the Toeplitz first columns X^{j,p}."""
    import torch
    o, g_ = _pair(oracle_mod, gpu, p)
    g_.build()
    d_g, X_g = g_.get_interface(0)
    d_o = o.apply_R(None, use_u0=True)
    X_o = o.build_L()
    u0max = np.abs(si.make_u0(p)).max()
    assert rel(d_g.cpu().numpy(), d_o, u0max) <= 1e-12
    assert rel(X_g.cpu().numpy(), X_o) <= 1e-12
    rng = np.random.default_rng(5)
    x = rng.standard_normal(o.ng) + 1j * rng.standard_normal(o.ng)
    y_g = g_.apply_I_minus_L(torch.as_tensor(x, device="cuda"), 0).cpu().numpy()
    y_o = x - o.apply_L(X_o, x)
    assert rel(y_g, y_o) <= 1e-12


@pytest.mark.parametrize("name,p", CASES, ids=[c[0] for c in CASES])
def test_new_algorithm_parity(oracle_mod, gpu, name, p):
    """Algorithm 3 end to end: u(T) within 1e-10, equal GMRES counts."""
    o, g_ = _pair(oracle_mod, gpu, p)
    ro = o.solve()
    st, uT, rg = g_.solve()
    assert ro["status"] == 0 and st == 0
    assert rg["iterations"] == ro["iterations"]
    assert rel(uT, ro["uT"]) <= 1e-10
    assert rel(g_.get_g().cpu().numpy(), ro["g"]) <= 1e-9


@pytest.mark.parametrize("name,p", [CASES[2], CASES[4]], ids=[CASES[2][0], CASES[4][0]])
def test_new_algorithm_parity_cgs2(oracle_mod, gpu, name, p):
    """The CGS2 option (gs_passes = 2) on both sides: equal counts, u(T)."""
    import dataclasses
    p = dataclasses.replace(p, gs_passes=2)
    o, g_ = _pair(oracle_mod, gpu, p)
    ro = o.solve()
    st, uT, rg = g_.solve()
    assert ro["status"] == 0 and st == 0
    assert rg["iterations"] == ro["iterations"]
    assert rel(uT, ro["uT"]) <= 1e-10


SOLVER_CASES = [
    ("new-bicgstab", si.ALG_NEW, si.KRY_BICGSTAB, si.POT_VX),
    ("new-fixed-point", si.ALG_NEW, si.KRY_FIXED_POINT, si.POT_VX),
    ("classical-fixed-point", si.ALG_CLASSICAL, si.KRY_FIXED_POINT, si.POT_VX),
    ("classical-gmres", si.ALG_CLASSICAL, si.KRY_GMRES, si.POT_VX),
    ("classical-bicgstab", si.ALG_CLASSICAL, si.KRY_BICGSTAB, si.POT_VX),
    ("classical-fp-cubic", si.ALG_CLASSICAL, si.KRY_FIXED_POINT, si.POT_CUBIC),
    ("precond-bicgstab", si.ALG_PRECOND, si.KRY_BICGSTAB, si.POT_VTX),
    ("precond-fixed-point", si.ALG_PRECOND, si.KRY_FIXED_POINT, si.POT_VTX),
]


@pytest.mark.parametrize("name,alg,kry,pot", SOLVER_CASES, ids=[c[0] for c in SOLVER_CASES])
def test_solver_variant_parity(oracle_mod, gpu, name, alg, kry, pot):
    """The paper's other interface solvers (Algorithms 1-2, fixed points,
    BiCGStab, readings A20-A22): equal iteration counts, u(T)
    within 1e-10 of the oracle."""
    p = si.config("C1", transmission=si.TC_S02, potential=pot, N=4, algorithm=alg, krylov=kry,
                  u0_kind="soliton" if pot == si.POT_CUBIC else "gaussian")
    o, g_ = _pair(oracle_mod, gpu, p)
    ro = o.solve()
    st, uT, rg = g_.solve()
    info = dict(it=(rg["iterations"], ro["iterations"]), inner=(rg["inner_iterations"], ro["inner_iterations"]),
                st=(st, ro["status"]), err=rel(uT, ro["uT"]))
    print(name, info)
    assert ro["status"] == 0 and st == 0, info
    assert rg["iterations"] == ro["iterations"], info
    assert rel(uT, ro["uT"]) <= 1e-10, info


TC_CASES = [("s03", si.TC_S03), ("s04", si.TC_S04), ("s12", si.TC_S12), ("s14", si.TC_S14),
            ("s22", si.TC_S22), ("s24", si.TC_S24)]


@pytest.mark.parametrize("name,tc", TC_CASES, ids=[c[0] for c in TC_CASES])
@pytest.mark.parametrize("march", ["resident", "stream"])
def test_higher_order_tc_parity(oracle_mod, gpu, name, tc, march):
    """Potential (S0^3, S0^4), gauge (S1^2, S1^4) and Pade (S2^{2,20},
    S2^{4,20}) transmission operators (readings
    A23-A26) through the new algorithm on
    V(x) = -x^2, both march kernels: equal GMRES counts, u(T) within 1e-10."""
    p = si.config("C1", transmission=tc, potential=si.POT_VX, N=4, march_form=int(march == "stream"))
    o, g_ = _pair(oracle_mod, gpu, p)
    ro = o.solve()
    st, uT, rg = g_.solve()
    assert ro["status"] == 0 and st == 0
    assert rg["iterations"] == ro["iterations"], (rg["iterations"], ro["iterations"])
    assert rel(uT, ro["uT"]) <= 1e-10
    d_g, X_g = g_.get_interface(0)
    assert rel(d_g.cpu().numpy(), o.apply_R(np.zeros(o.ng), use_u0=True), 1.0) <= 1e-12
    assert rel(X_g.cpu().numpy(), o.build_L(), 1.0) <= 1e-12


PINV_CASES = [("vtx-gmres", 5, si.POT_VTX, si.KRY_GMRES), ("vtx-bicgstab", 5, si.POT_VTX, si.KRY_BICGSTAB),
              ("nl-fp", 5, si.POT_CUBIC, si.KRY_FIXED_POINT), ("vtx-gmres-N40", 40, si.POT_VTX, si.KRY_GMRES)]


@pytest.mark.parametrize("name,N,pot,kry", PINV_CASES)
def test_pinv_exact_parity(oracle_mod, gpu, name, N, pot, kry):
    """Exact causal P^{-1} (reading A27) in the preconditioned
    algorithms: the oracle's dense lag-0 LU vs the GPU's block-Jacobi sweeps
    (N = 40 has five-cell subdomains, so several sweeps run): equal outer
    iterations, no inner iterations, u(T) within 1e-10."""
    p = si.config("C1", transmission=si.TC_S02, potential=pot, N=N, algorithm=si.ALG_PRECOND, krylov=kry,
                  pinv_exact=1, u0_kind="soliton" if pot == si.POT_CUBIC else "gaussian")
    o, g_ = _pair(oracle_mod, gpu, p)
    ro = o.solve()
    st, uT, rg = g_.solve()
    assert ro["status"] == 0 and st == 0
    assert rg["iterations"] == ro["iterations"], (rg["iterations"], ro["iterations"])
    assert rg["inner_iterations"] == 0 == ro["inner_iterations"]
    assert rel(uT, ro["uT"]) <= 1e-10


@pytest.mark.parametrize("N,tc", [(2, si.TC_ROBIN), (2, si.TC_S02), (4, si.TC_ROBIN)])
def test_pinv_exact_small_chains(oracle_mod, gpu, N, tc):
    """Exact P^{-1} at the ends of its range: one interface (N = 2, no cross
    couplings, no sweeps) and Robin (the 2x2 lag-0 blocks are far from the
    identity), against the oracle's dense lag-0 LU."""
    p = si.config("C1", transmission=tc, potential=si.POT_VTX, N=N, algorithm=si.ALG_PRECOND, pinv_exact=1,
                  robin_p=5.0)
    o, g_ = _pair(oracle_mod, gpu, p)
    ro = o.solve()
    st, uT, rg = g_.solve()
    assert ro["status"] == 0 and st == 0 and rg["iterations"] == ro["iterations"]
    assert rel(uT, ro["uT"]) <= 1e-10


PAPER_COUNT_CASES = [
    # Table 5 (dx = 1e-4): classical fixed point, V = 5tx, N = 100 -> N_nopc = 71
    ("table5-classical-N100", dict(name="C3", N=100, dx=1e-4, algorithm=si.ALG_CLASSICAL,
                                   krylov=si.KRY_FIXED_POINT), 71),
    # the NL table: preconditioned fixed point, |u|^2, N = 100 -> N_pc = 22 (C4 grid)
    ("nl-precond-N100", dict(name="C4", maxit=2000), 22),
    # the NL table's N = 10 row at dx = 1e-5 (N_j = 420,001: the streaming NL march,
    # the exact causal P^{-1}): preconditioned fixed point -> N_pc = 11
    ("nl-precond-N10-fine", dict(name="C4", N=10, dx=1e-5, pinv_exact=1, maxit=2000), 11),
    # the same table's N = 500 and 1000 rows at dx = 1e-5 -> N_pc = 25, 26
    ("nl-precond-N500-fine", dict(name="C4", N=500, dx=1e-5, pinv_exact=1, maxit=2000), 25),
    ("nl-precond-N1000-fine", dict(name="C4", N=1000, dx=1e-5, pinv_exact=1, maxit=2000), 26),
    # Table 7: new algorithm, Robin p = 45, fixed point, N = 500, random g0 -> 1690
    ("table7-robin45-N500", dict(name="C5", transmission=si.TC_ROBIN, robin_p=45.0, krylov=si.KRY_FIXED_POINT,
                                 g0_random=True, maxit=2000), 1690),
]


@pytest.mark.parametrize("name,kw,count", PAPER_COUNT_CASES, ids=[c[0] for c in PAPER_COUNT_CASES])
def test_paper_iteration_counts(gpu, name, kw, count):
    """The GPU path reproduces iteration counts printed in the paper on the
    paper's own experiments at full size (profiles/r01/table*.txt)."""
    kw = dict(kw)
    p = si.config(kw.pop("name"), **kw)
    s = gpu.SWR(p, si.inputs(p))
    s.build()
    st, uT, r = s.solve()
    assert st == 0 and r["iterations"] == count, (r["iterations"], count)


@pytest.mark.parametrize("M", [8, 11, 16])
def test_nl_march_shapes(oracle_mod, gpu, M):
    """The NL march with 8, 11 and 16 rows per thread (the 16-row shape serves
    the largest resident subdomains; each forced on a problem the oracle
    solves; the automatic C4 shape runs in the C4 tests): the preconditioned fixed point for
    |u|^2 with equal outer counts, equal NL fixed-point maxima, u(T) within
    1e-10."""
    p = si.Problem(dx=2e-3, dt=5e-3, N=4, potential=si.POT_CUBIC, algorithm=si.ALG_PRECOND, krylov=si.KRY_FIXED_POINT,
                   u0_kind="soliton", pinv_exact=1, nl_rows_per_thread=M)
    o, g_ = _pair(oracle_mod, gpu, p)
    ro = o.solve()
    st, uT, rg = g_.solve()
    assert ro["status"] == 0 and st == 0
    assert rg["iterations"] == ro["iterations"] and rg["fp_max"] == ro["fp_max"], (rg, ro["iterations"])
    assert rel(uT, ro["uT"]) <= 1e-10


def test_random_g0_and_n1(oracle_mod, gpu):
    p = si.config("C1", transmission=si.TC_S02, potential=si.POT_VX, N=5, g0_random=True)
    o, g_ = _pair(oracle_mod, gpu, p)
    ro = o.solve()
    st, uT, rg = g_.solve()
    assert rg["iterations"] == ro["iterations"] and rel(uT, ro["uT"]) <= 1e-10
    p1 = si.config("C1", N=1, potential=si.POT_VX)
    o1, g1 = _pair(oracle_mod, gpu, p1)
    st, uT, rg = g1.solve()
    assert st == 0 and rg["iterations"] == 0
    assert rel(uT, o1.monodomain()[1]) <= 1e-12


def test_c5_full_size_sampled(oracle_mod, gpu):
    """C5 at full size (N = 500, dx = 1e-5, N_T = 500) in the launch shape
    bench.py times: the d = R(0) traces of sampled subdomains (first, last,
    the Gaussian's support near x = -10, and two random ones) and the probe
    columns X^{j,1}, X^{j,3} of three subdomains against the oracle's marches
    of those subdomains.  Each comparison is relative to the compared
    vector's own norm (floor 1e-3 of the unit impulse), with the bar 1e-10
    raised to 4x the spread between the oracle and its FMA build where the
    problem amplifies rounding beyond it."""
    p = si.config("C5")
    arrays = si.inputs(p)
    g_ = gpu.SWR(p, arrays)
    g_.build()
    d_g, X_g = g_.get_interface(0)
    d_g = d_g.cpu().numpy()
    X_g = X_g.cpu().numpy()
    o = oracle_mod.Oracle(p, arrays)
    of = oracle_mod.Oracle(p, arrays, library=oracle_mod.lib_fma())
    NT = p.NT
    worst = []

    def check(gv, ov, fv, what):
        spread = rel(fv, ov, 1e-3)
        tol = max(1e-10, 4.0 * spread)
        err = rel(gv, ov, 1e-3)
        worst.append((what, err, spread))
        assert err <= tol, (what, err, spread)

    for j in (1, 131, 132, 260, 500):
        st, ol, orr, _, _ = o.march(j, None, None, use_u0=True)
        _, olf, orf, _, _ = of.march(j, None, None, use_u0=True)
        if j >= 2:
            check(d_g[(2 * j - 4) * NT:(2 * j - 3) * NT], ol, olf, ("d left", j))
        if j <= p.N - 1:
            check(d_g[(2 * j - 1) * NT:(2 * j) * NT], orr, orf, ("d right", j))
    e = np.zeros(NT, np.complex128)
    e[0] = 1
    for j in (2, 250, 499):
        st, ol, orr, _, _ = o.march(j, e, None, use_u0=False)
        _, olf, orf, _, _ = of.march(j, e, None, use_u0=False)
        check(X_g[j - 1, 0], ol, olf, ("X1", j))
        check(X_g[j - 1, 2], orr, orf, ("X3", j))
    print("C5 sampled (what, rel err vs oracle, oracle FMA spread):", worst)


def test_c2_full_size_sampled(oracle_mod, gpu):
    """C2 at full size (N = 10, dx = 1e-5: N_j = 420,001, the streaming march)
    in the launch shape the timing uses: d = R(0) traces of subdomains 1, 5
    (the Gaussian's support) against the oracle's marches."""
    p = si.config("C2")
    arrays = si.inputs(p)
    g_ = gpu.SWR(p, arrays)
    g_.build()
    d_g, _ = g_.get_interface(0)
    d_g = d_g.cpu().numpy()
    o = oracle_mod.Oracle(p, arrays)
    NT = p.NT
    for j in (1, 5):
        st, ol, orr, _, _ = o.march(j, None, None, use_u0=True)
        if j >= 2:
            assert rel(d_g[(2 * j - 4) * NT:(2 * j - 3) * NT], ol, 1.0) <= 1e-10
        if j <= p.N - 1:
            assert rel(d_g[(2 * j - 1) * NT:(2 * j) * NT], orr, 1.0) <= 1e-10


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_c3_c4_full_size_sampled(oracle_mod, gpu, name):
    """C3 (V = 5tx: the time-dependent march, N_j = 42,001 in a 15-CTA
    cluster, per-step factors bulk-copied) and C4 (f(u) = |u|^2: the NL march
    with its inner fixed point) at full size: the first sweep d = R(0; u0) of
    the preconditioned algorithms; the traces and u(T) of sampled subdomains
    (the ends and the initial packet's support near x = -10) against the
    oracle's marches.  Bar: 1e-10, raised to 4x the spread between the oracle
    and the same oracle built with FMA contraction where the problem itself
    amplifies rounding beyond it (C3 at dx = 1e-5: the two oracle builds
    differ by 2.1e-9)."""
    p = si.config(name)
    arrays = si.inputs(p)
    g_ = gpu.SWR(p, arrays)
    o = oracle_mod.Oracle(p, arrays)
    of = oracle_mod.Oracle(p, arrays, library=oracle_mod.lib_fma())
    Rg_g, uT_g = g_.apply_R(None, use_u0=True, want_uT=True)
    Rg_g, uT_g = Rg_g.cpu().numpy(), uT_g.cpu().numpy()
    NT, m = p.NT, p.Nx // p.N

    def check(gv, ov, fv, what):
        tol = max(1e-10, 4.0 * rel(fv, ov, 1e-3))
        assert rel(gv, ov, 1e-3) <= tol, (what, rel(gv, ov, 1e-3), tol)

    for j in (1, 27, 28, p.N):
        st, ol, orr, uloc, _ = o.march(j, None, None, use_u0=True)
        st2, olf, orf, ulf, _ = of.march(j, None, None, use_u0=True)
        assert st == 0 and st2 == 0, (j, st, st2)
        if j >= 2:
            check(Rg_g[(2 * j - 4) * NT:(2 * j - 3) * NT], ol, olf, ("left", j))
        if j <= p.N - 1:
            check(Rg_g[(2 * j - 1) * NT:(2 * j) * NT], orr, orf, ("right", j))
        a = (j - 1) * m
        check(uT_g[a + 1:a + p.Nj - 1], uloc[1:-1], ulf[1:-1], ("uT", j))


STREAM_CASES = [
    ("new-s02-N4", si.config("C1", transmission=si.TC_S02, potential=si.POT_VX, N=4)),
    ("new-robin-N5", si.config("C1", transmission=si.TC_ROBIN, potential=si.POT_VX, N=5, robin_p=19.0)),
    ("new-mid-N42", si.Problem(dx=1e-3, dt=5e-3, N=42, potential=si.POT_VX, transmission=si.TC_S02)),
    ("precond-vtx-N4", si.config("C1", transmission=si.TC_S02, potential=si.POT_VTX, algorithm=si.ALG_PRECOND, N=4)),
    # |u|^2: the streaming NL march (k_march_nl_stream), fixed point and GMRES
    ("nl-fp-N4", si.Problem(dx=2e-3, dt=5e-3, N=4, potential=si.POT_CUBIC, algorithm=si.ALG_PRECOND,
                            krylov=si.KRY_FIXED_POINT, u0_kind="soliton", pinv_exact=1)),
    ("nl-robin-N5", si.Problem(dx=1e-2, dt=5e-3, N=5, potential=si.POT_CUBIC, algorithm=si.ALG_PRECOND,
                               krylov=si.KRY_FIXED_POINT, transmission=si.TC_ROBIN, robin_p=19.0,
                               u0_kind="soliton", pinv_exact=1)),
]


@pytest.mark.parametrize("name,p", STREAM_CASES, ids=[c[0] for c in STREAM_CASES])
def test_streaming_march_parity(oracle_mod, gpu, name, p):
    """The streaming march (state through HBM, chains of co-resident CTAs;
    used when a subdomain does not fit a resident cluster, e.g. C2 at
    dx = 1e-5) forced on problems the oracle solves: equal counts, u(T)."""
    import dataclasses
    p = dataclasses.replace(p, march_form=1)
    o, g_ = _pair(oracle_mod, gpu, p)
    ro = o.solve()
    st, uT, rg = g_.solve()
    assert ro["status"] == 0 and st == 0
    assert rg["iterations"] == ro["iterations"], (rg["iterations"], ro["iterations"])
    if p.potential == si.POT_CUBIC:
        assert rg["fp_max"] == ro["fp_max"], (rg["fp_max"], ro["fp_max"])
    assert rel(uT, ro["uT"]) <= 1e-10


def test_streaming_sweep_matches_resident(gpu):
    """One sweep R(g) through both march kernels on a 3-CTA-per-chain
    problem: equal to rounding."""
    import dataclasses
    import torch
    p = si.Problem(dx=1e-3, dt=5e-3, N=10, potential=si.POT_VX, transmission=si.TC_S02)
    arr = si.inputs(p)
    g = torch.randn(p.ng, dtype=torch.complex128, device="cuda")
    a = gpu.SWR(p, arr)
    ra, ua = a.apply_R(g, use_u0=True, want_uT=True)
    b = gpu.SWR(dataclasses.replace(p, march_form=1), arr)
    rb, ub = b.apply_R(g, use_u0=True, want_uT=True)
    assert rel(rb.cpu().numpy(), ra.cpu().numpy()) <= 1e-12
    assert rel(ub.cpu().numpy(), ua.cpu().numpy()) <= 1e-12


def test_cgs_kernel_shapes(oracle_mod, gpu):
    """The fused Gram-Schmidt passes with per-subdomain units (one CTA per
    subdomain, chunked entries with a ragged tail, the three register shapes
    for up to 8 / 16 / 32 basis vectors): the oracle's GMRES iteration count
    and u(T) on a NEW solve with a full restart cycle."""
    p = si.Problem(dx=1e-3, dt=1e-3, N=20, potential=si.POT_VX)
    o, g_ = _pair(oracle_mod, gpu, p)
    ro = o.solve()
    st, uT, rg = g_.solve()
    assert st == 0 and rg["iterations"] == ro["iterations"] > 16, (rg["iterations"], ro["iterations"])
    assert rel(uT, ro["uT"]) <= 1e-10


@pytest.mark.parametrize("mode", ["direct", "fft", "fftsm"])
def test_toeplitz_paths(oracle_mod, gpu, mode):
    """All forms of y = (I - L) x (direct causal convolution; FFT convolution:
    for NF = 1024 the one-warp register four-step kernel (default) or the
    shared-memory radix-4 Stockham kernel) against the oracle's direct
    convolution."""
    import dataclasses
    import torch
    form = {"direct": 1, "fft": 0, "fftsm": 2}[mode]
    for p in (si.Problem(dx=1e-3, dt=5e-3, N=42, potential=si.POT_VX),
              si.Problem(dx=1e-3, dt=1e-3, N=20, potential=si.POT_VX)):   # N_T = 100 and 500
        p = dataclasses.replace(p, toeplitz_form=form)
        o, g_ = _pair(oracle_mod, gpu, p)
        g_.build()
        _, X_g = g_.get_interface(0)
        rng = np.random.default_rng(9)
        x = rng.standard_normal(o.ng) + 1j * rng.standard_normal(o.ng)
        y_g = g_.apply_I_minus_L(torch.as_tensor(x, device="cuda"), 0).cpu().numpy()
        y_o = x - o.apply_L(X_g.cpu().numpy(), x)
        assert rel(y_g, y_o) <= 1e-12, mode


PRECOND_CASES = [
    ("vtx-s02-N4", si.config("C1", transmission=si.TC_S02, potential=si.POT_VTX, algorithm=si.ALG_PRECOND, N=4)),
    ("vtx-robin-N5", si.config("C1", transmission=si.TC_ROBIN, potential=si.POT_VTX, algorithm=si.ALG_PRECOND, N=5,
                               robin_p=5.0)),
    ("vtx-mid-N20", si.Problem(dx=2e-3, dt=5e-3, N=20, potential=si.POT_VTX, algorithm=si.ALG_PRECOND)),
    ("nl-s02-N4", si.config("C1", transmission=si.TC_S02, potential=si.POT_CUBIC, algorithm=si.ALG_PRECOND, N=4,
                            u0_kind="soliton")),
    ("nl-robin-N4", si.config("C1", transmission=si.TC_ROBIN, potential=si.POT_CUBIC, algorithm=si.ALG_PRECOND, N=4,
                              u0_kind="soliton", robin_p=20.0)),
    ("nl-mid-N20", si.Problem(dx=2e-3, dt=5e-3, N=20, potential=si.POT_CUBIC, algorithm=si.ALG_PRECOND,
                              u0_kind="soliton")),
]


@pytest.mark.parametrize("name,p", PRECOND_CASES, ids=[c[0] for c in PRECOND_CASES])
def test_precond_parity(oracle_mod, gpu, name, p):
    """Preconditioned algorithms: GMRES on P^{-1}(I-L)g = P^{-1}d
    for V(t,x) and the preconditioned fixed point for |u|^2; equal outer
    iteration counts and NL fixed-point maxima, u(T) within 1e-10.  The inner
    P^{-1} GMRES solves stop at 1e-12 relative (reading A8), which for these
    operators sits at the rounding floor of (I - L0): the oracle and the same
    oracle source built with FMA contraction (only the rounding differs)
    already disagree on the total inner count by up to 122 steps (vtx-robin-N5).
    The GPU's total must stay within 3x that measured spread of the oracle,
    and equal it where the two oracle builds agree (measured: equal, 0.9 %,
    1 % and 3.5 % apart)."""
    o, g_ = _pair(oracle_mod, gpu, p)
    ro = o.solve()
    rf = oracle_mod.Oracle(p, si.inputs(p), library=oracle_mod.lib_fma()).solve()
    st, uT, rg = g_.solve()
    floor = abs(rf["inner_iterations"] - ro["inner_iterations"])
    info = dict(outer=(rg["iterations"], ro["iterations"]), inner=(rg["inner_iterations"], ro["inner_iterations"]),
                inner_oracle_fma=rf["inner_iterations"], fp=(rg["fp_max"], ro["fp_max"]), err=rel(uT, ro["uT"]),
                st=(st, ro["status"]))
    print(name, info)
    assert ro["status"] == 0 and st == 0, info
    assert rg["iterations"] == ro["iterations"] == rf["iterations"], info
    assert abs(rg["inner_iterations"] - ro["inner_iterations"]) <= max(1, 3 * floor), info
    assert rg["fp_max"] == ro["fp_max"], info
    assert rel(uT, ro["uT"]) <= 1e-10, info


def test_nl_sweep_parity(oracle_mod, gpu):
    """One nonlinear sweep R_nl(g; u0) with a random g (several CTAs)."""
    import torch
    p = si.Problem(dx=1e-3, dt=5e-3, N=20, potential=si.POT_CUBIC, algorithm=si.ALG_PRECOND, u0_kind="soliton")
    o, g_ = _pair(oracle_mod, gpu, p)
    rng = np.random.default_rng(21)
    g = 0.1 * (rng.standard_normal(o.ng) + 1j * rng.standard_normal(o.ng))
    Rg_o = o.apply_R(g, use_u0=True)
    Rg_g, _ = g_.apply_R(torch.as_tensor(g, device="cuda"), use_u0=True)
    assert rel(Rg_g.cpu().numpy(), Rg_o) <= 1e-11


def test_nl_stream_full_size_sampled(oracle_mod, gpu):
    """|u|^2 at the paper's largest NL subdomains (T5 N = 10 at dx = 1e-5:
    N_j = 420,001, beyond the resident NL march, so the streaming NL march
    k_march_nl_stream runs): one sweep R_nl(0; u0); the traces and u(T) of the
    subdomain holding the soliton (j = 3) against the oracle's march.  Bar as
    the other full-size tests: 1e-10, raised to 4x the spread between the
    oracle and its FMA build (the fixed point at dt/dx^2 = 1e7 amplifies
    rounding: the two oracle builds differ by ~1e-9 here)."""
    import torch
    p = si.Problem(dx=1e-5, dt=1e-3, N=10, potential=si.POT_CUBIC, algorithm=si.ALG_PRECOND, u0_kind="soliton")
    arrays = si.inputs(p)
    g_ = gpu.SWR(p, arrays)
    Rg, uT = g_.apply_R(torch.zeros(p.ng, dtype=torch.complex128, device="cuda"), use_u0=True, want_uT=True)
    Rg, uT = Rg.cpu().numpy(), uT.cpu().numpy()
    o = oracle_mod.Oracle(p, arrays)
    of = oracle_mod.Oracle(p, arrays, library=oracle_mod.lib_fma())
    NT, m, j = p.NT, p.Nx // p.N, 3
    st, ol, orr, uloc, _ = o.march(j, None, None, use_u0=True)
    st2, olf, orf, ulf, _ = of.march(j, None, None, use_u0=True)
    assert st == 0 and st2 == 0
    for gv, ov, fv, what in ((Rg[(2 * j - 4) * NT:(2 * j - 3) * NT], ol, olf, "left"),
                             (Rg[(2 * j - 1) * NT:(2 * j) * NT], orr, orf, "right"),
                             (uT[(j - 1) * m + 1:(j - 1) * m + p.Nj - 1], uloc[1:-1], ulf[1:-1], "uT")):
        tol = max(1e-10, 4.0 * rel(fv, ov, 1.0))
        assert rel(gv, ov, 1.0) <= tol, (what, rel(gv, ov, 1.0), rel(fv, ov, 1.0))


EDGE_CASES = [
    ("one-cell-subdomains", si.Problem(a0=-1.0, b0=1.0, T=0.05, dx=0.25, dt=0.01, N=8, potential=si.POT_VX)),
    ("one-step", si.Problem(a0=-2.0, b0=2.0, T=0.01, dx=0.05, dt=0.01, N=4, potential=si.POT_VX)),
    ("two-steps-robin", si.Problem(a0=-2.0, b0=2.0, T=0.02, dx=0.05, dt=0.01, N=5, potential=si.POT_ZERO,
                                   transmission=si.TC_ROBIN, robin_p=3.0)),
    ("N2-fine", si.Problem(a0=-21.0, b0=21.0, T=0.05, dx=1e-2, dt=1e-3, N=2, potential=si.POT_VX)),
    # |u|^2 (the NL march: first and last row in one thread, N_j = 2 and 5) and V(t,x)
    ("nl-one-cell", si.Problem(a0=-1.0, b0=1.0, T=0.05, dx=0.25, dt=0.01, N=8, potential=si.POT_CUBIC,
                               algorithm=si.ALG_PRECOND, krylov=si.KRY_FIXED_POINT, pinv_exact=1)),
    ("nl-one-step", si.Problem(a0=-2.0, b0=2.0, T=0.01, dx=0.1, dt=0.01, N=10, potential=si.POT_CUBIC,
                               algorithm=si.ALG_PRECOND, krylov=si.KRY_FIXED_POINT)),
    ("nl-stream-one-cell", si.Problem(a0=-1.0, b0=1.0, T=0.05, dx=0.25, dt=0.01, N=8, potential=si.POT_CUBIC,
                                      algorithm=si.ALG_PRECOND, krylov=si.KRY_FIXED_POINT, pinv_exact=1,
                                      march_form=1)),
    ("vtx-one-cell", si.Problem(a0=-1.0, b0=1.0, T=0.05, dx=0.25, dt=0.01, N=8, potential=si.POT_VTX,
                                algorithm=si.ALG_PRECOND)),
]


@pytest.mark.parametrize("name,p", EDGE_CASES, ids=[c[0] for c in EDGE_CASES])
def test_edge_cases(oracle_mod, gpu, name, p):
    """Degenerate shapes: one-cell subdomains (N_j = 2), a single time step,
    two steps with Robin, and a long subdomain (N_j = 4201, one CTA) at N = 2;
    the same for the NL marches (resident and streaming) and the
    time-dependent march."""
    x = p.nodes()
    arrays = si.inputs(p)
    arrays["u0"] = np.exp(-(x * x) + 2j * x)
    o, g_ = _pair(oracle_mod, gpu, p, arrays)
    ro = o.solve()
    st, uT, rg = g_.solve()
    assert ro["status"] == 0 and st == 0
    assert rg["iterations"] == ro["iterations"]
    if p.potential == si.POT_CUBIC:
        assert rg["fp_max"] == ro["fp_max"]
    assert rel(uT, ro["uT"]) <= 1e-10


def test_c5_solve_on_the_oracle_operator(oracle_mod, gpu):
    """The north-star configuration's solve stage on a common interface
    operator: the GPU runs Algorithm 3's GMRES(30) and final sweep
    on the oracle's d and L (swr_set_interface, test infrastructure), the
    oracle solves as it stands.  With the build's rounding taken out, the two
    agree to the north-star bar: equal iteration counts, u(T) and g within
    1e-10 relative L2 -- the ~1e-8 of the end-to-end gate is the build's
    rounding (d and L within the oracle's FMA spread) amplified by the
    interface solve, not the solve itself."""
    import os
    p = si.config("C5")
    arrays = si.inputs(p)
    oracle_mod.set_threads(os.cpu_count())
    try:
        o = oracle_mod.Oracle(p, arrays)
        X_o = o.build_L()
        d_o = o.apply_R(None, use_u0=True)
        ro = o.solve()
    finally:
        oracle_mod.set_threads(1)
    s = gpu.SWR(p, arrays)
    s.set_interface(d_o, X_o)
    st, uT, rg = s.solve()
    g_g = s.get_g().cpu().numpy()
    s.close()
    assert st == 0 and ro["status"] == 0
    eu, eg = rel(uT, ro["uT"]), rel(g_g, ro["g"])
    print(f"C5 on the oracle's operator: it {rg['iterations']} / {ro['iterations']}, u(T) {eu:.2e}, g {eg:.2e}")
    assert rg["iterations"] == ro["iterations"]
    assert eu <= 1e-10 and eg <= 1e-10, (eu, eg)


def test_c5_north_star_gate(oracle_mod, gpu):
    """The north-star configuration end to end (C5: N = 500, dx = 1e-5,
    N_T = 500, V = -x^2, NEW + GMRES(30), tol 1e-10 as P:1079), GPU in the
    launch shape bench.py times against the oracle solved on all host cores:
      - equal GMRES iteration counts;
      - the residual estimates of every Arnoldi step agree to 1e-10 of the
        first one (the two Krylov processes track each other to the end);
      - u(T) against the oracle's own rounding floor.  The oracle source built
        with FMA contraction (rounding is the only difference) lands 9.8e-9
        from the default build, at tol 1e-10 and at 1e-12 alike
        (profiles/r02/c5_gate.txt): at this size the method's fp64 result is
        fixed only to ~1e-8 (rounding in the 500-step marches at dt/dx^2 =
        1e7, amplified by the interface solve), so the strict 1e-10 bar is
        below the oracle's own reproducibility.  The GPU (FMA arithmetic) must
        sit within 1.5x that spread of the default build and within a tenth of
        it (measured 4.8e-10) of the FMA build, and be at least as close as
        the oracle to the monodomain solution on the same grid (the exact
        discrete solution the iteration converges to; measured 4.6e-9 vs
        7.0e-9).  DESIGN.md section 2."""
    import os
    p = si.config("C5")
    arrays = si.inputs(p)
    s = gpu.SWR(p, arrays)
    s.build()
    st, uT, rg = s.solve()
    s.close()
    res = {}
    for name, lib in (("oracle", oracle_mod.lib()), ("fma", oracle_mod.lib_fma())):
        oracle_mod.set_threads(os.cpu_count(), lib)
        try:
            res[name] = oracle_mod.Oracle(p, arrays, library=lib).solve()
        finally:
            oracle_mod.set_threads(1, lib)
    ro, rf = res["oracle"], res["fma"]
    assert st == 0 and ro["status"] == 0 and rf["status"] == 0
    assert rg["iterations"] == ro["iterations"] == rf["iterations"], (rg["iterations"], ro["iterations"])
    h_g, h_o = rg["history"], ro["history"]
    assert len(h_g) == len(h_o)
    assert np.abs(h_g - h_o).max() <= 1e-10 * h_o[0]
    spread = rel(rf["uT"], ro["uT"])
    e_o, e_f = rel(uT, ro["uT"]), rel(uT, rf["uT"])
    # the exact discrete solution the iteration converges to: the monodomain
    # march on the same grid (N = 1, no interface problem)
    st_m, um, _ = oracle_mod.Oracle(si.config("C5", N=1), arrays).monodomain()
    m_g, m_o = rel(uT, um), rel(ro["uT"], um)
    print(f"C5 gate: it {rg['iterations']}, u(T) gpu-oracle {e_o:.3e}, gpu-oracle_fma {e_f:.3e}, spread {spread:.3e}; "
          f"to the monodomain solution: gpu {m_g:.3e}, oracle {m_o:.3e}")
    assert e_o <= max(1e-10, 1.5 * spread), (e_o, spread)
    assert e_f <= max(1e-10, 0.1 * spread), (e_f, spread)
    assert st_m == 0 and m_g <= max(1e-10, 1.05 * m_o), (m_g, m_o)


HIGH_TC_FULL = [("s03", si.TC_S03, 20), ("s04", si.TC_S04, 20), ("s12", si.TC_S12, 20), ("s14", si.TC_S14, 20),
                ("s22-m20", si.TC_S22, 20), ("s22-m50", si.TC_S22, 50), ("s22-m100", si.TC_S22, 100),
                ("s24-m20", si.TC_S24, 20), ("s24-m50", si.TC_S24, 50), ("s24-m100", si.TC_S24, 100)]


@pytest.mark.parametrize("name,tc,m", HIGH_TC_FULL, ids=[c[0] for c in HIGH_TC_FULL])
@pytest.mark.parametrize("march", ["resident", "stream"])
def test_higher_order_tc_parity_multi_cta(oracle_mod, gpu, name, tc, m, march):
    """The higher-order and Pade operators on
    subdomains that span a multi-CTA cluster (N_j = 4201 on the paper's
    domain, dx = 1e-3, N = 10, V = -x^2) in both marches, Pade m = 20, 50,
    100: equal GMRES counts, u(T) within 1e-10, d and X within 1e-12."""
    p = si.Problem(dx=1e-3, dt=5e-3, N=10, potential=si.POT_VX, transmission=tc, pade_m=m,
                   march_form=int(march == "stream"))
    o, g_ = _pair(oracle_mod, gpu, p)
    ro = o.solve()
    st, uT, rg = g_.solve()
    assert ro["status"] == 0 and st == 0
    assert rg["iterations"] == ro["iterations"], (rg["iterations"], ro["iterations"])
    assert rel(uT, ro["uT"]) <= 1e-10
    d_g, X_g = g_.get_interface(0)
    assert rel(d_g.cpu().numpy(), o.apply_R(np.zeros(o.ng), use_u0=True), 1.0) <= 1e-12
    assert rel(X_g.cpu().numpy(), o.build_L(), 1.0) <= 1e-12


def test_solve_is_deterministic(gpu):
    """Two solves of the same problem (several CTAs per cluster, GMRES with
    restarts) give bitwise equal u(T), g and residual histories: every
    reduction on the path has a fixed order (no atomics decide a sum)."""
    p = si.Problem(dx=1e-3, dt=5e-3, N=10, potential=si.POT_VX)
    s = gpu.SWR(p, si.inputs(p))
    out = []
    for _ in range(2):
        s.build()
        st, uT, r = s.solve()
        out.append((uT.copy(), s.get_g().cpu().numpy(), r["history"].copy(), r["iterations"]))
    assert out[0][3] == out[1][3]
    for a, b in zip(out[0][:3], out[1][:3]):
        assert np.array_equal(a, b)


@pytest.mark.gpu
def test_update_inputs_equals_fresh_setup(gpu):
    """swr_update_inputs (d depends on u0, L on V through the
    factorisation) gives bitwise the solve of a fresh handle set up with the
    new inputs: host u0 + V_x together (u0's copy on the side stream,
    overlapping V_x's copy and the factorisation), from pinned and pageable
    buffers, and u0 alone."""
    import torch
    p = si.Problem(dx=1e-3, dt=5e-3, N=42, potential=si.POT_VX, transmission=si.TC_S02)
    base = si.inputs(p)
    x = p.nodes()
    u0_b = (2.0 / np.cosh(np.sqrt(2.0) * (x + 5.0)) * np.exp(3j * x)).astype(np.complex128)
    vx_b = (-0.5 * x * x + 0.25 * x).astype(np.float64)
    u0_c = np.exp(-(x - 3.0) ** 2 - 7j * x).astype(np.complex128)

    def fresh(u0, vx):
        arr = dict(base, u0=u0, V_x=vx)
        s = gpu.SWR(p, arr)
        s.build()
        st, uT, r = s.solve()
        s.close()
        return uT.copy(), r["iterations"]

    s = gpu.SWR(p, base)
    s.build()
    s.solve()
    for pinned in (True, False):
        u0h = torch.from_numpy(u0_b).pin_memory().numpy() if pinned else u0_b.copy()
        vxh = torch.from_numpy(vx_b).pin_memory().numpy() if pinned else vx_b.copy()
        s.update_inputs(u0=u0h, V_x=vxh)
        s.build()
        st, uT, r = s.solve()
        ref, it = fresh(u0_b, vx_b)
        assert r["iterations"] == it
        assert np.array_equal(uT, ref)
        # back to the base inputs so the next round changes both again
        s.update_inputs(u0=base["u0"], V_x=base["V_x"])
    s.update_inputs(u0=u0_c)
    s.build()
    st, uT, r = s.solve()
    ref, it = fresh(u0_c, base["V_x"])
    assert r["iterations"] == it and np.array_equal(uT, ref)
    # device inputs (stream-ordered copies on the handle's stream)
    with torch.cuda.stream(s.stream):
        du0 = torch.from_numpy(u0_b).to("cuda", non_blocking=False)
        dvx = torch.from_numpy(vx_b).to("cuda", non_blocking=False)
    torch.cuda.synchronize()
    s.update_inputs(u0=du0, V_x=dvx, on_device=True)
    s.build()
    st, uT, r = s.solve()
    ref, it = fresh(u0_b, vx_b)
    assert r["iterations"] == it and np.array_equal(uT, ref)
    s.close()


@pytest.mark.gpu
def test_factor_flags_nan_pivot(gpu):
    """The factorisation's pivot check (a zero or non-finite pivot of
    A - B) surfaces as SWR_ERR_ZERO_PIVOT at setup and at swr_update_inputs
    (a NaN in V_x poisons the pivots from its row on)."""
    from paper_1503_02564_b200.swr import SWRError
    p = si.Problem(dx=1e-3, dt=5e-3, N=10, potential=si.POT_VX)
    arr = si.inputs(p)
    bad = arr["V_x"].copy()
    bad[len(bad) // 3] = np.nan
    with pytest.raises(SWRError) as e:
        gpu.SWR(p, dict(arr, V_x=bad))
    assert e.value.status == 3
    s = gpu.SWR(p, arr)
    with pytest.raises(SWRError) as e:
        s.update_inputs(V_x=bad)
    assert e.value.status == 3
    s.update_inputs(V_x=arr["V_x"])   # recovers with valid data
    s.build()
    st, uT, r = s.solve()
    assert st == 0 and np.all(np.isfinite(uT))
    s.close()
