"""Measurements behind the oracle pins that must also FAIL on a mutated oracle.

Each function runs one pin's computation with a given oracle library (the
real one, or a build with a deliberate error planted, oracle.lib_mutant(k))
and returns the measured quantity; tests/test_oracle_pins.py asserts the pin
on the real oracle, tests/test_oracle_mutants.py asserts that the same pin
rejects the mutant.  The expected values are closed forms written from the
paper's continuous problem, never from the oracle's discrete formulas.
"""
from __future__ import annotations

import math

import numpy as np

import swr_inputs as si


# ----------------------------------------------------------------------------
# Nonlinear Schrodinger: exact soliton (P:1067 initial datum, eq. P:34 with
# f(u) = |u|^2).  i u_t + u_xx + |u|^2 u = 0 has the travelling soliton
#   u = a sech(a (x - x0 - c t)/sqrt 2) exp(i (c/2 (x - x0) - (c^2/4 - a^2/2) t))
# (direct substitution); a = 2, c = 40, x0 = -10 gives the paper's u0 =
# 2 sech(sqrt 2 (x+10)) e^{20 i (x+10)} and the phase 20 (x+10) - 398 t.
# ----------------------------------------------------------------------------
def soliton_exact(x, t):
    y = x + 10.0
    return 2.0 / np.cosh(math.sqrt(2.0) * (y - 40.0 * t)) * np.exp(1j * (20.0 * y - 398.0 * t))


def nl_soliton_errors(oracle_mod, library=None):
    """Relative L2 error of the oracle's monodomain Duran-Sanz-Serna march
    (with its inner fixed point) against the exact soliton along a
    dt, dx ladder (ratio 2), before the soliton's tails (2 sech(sqrt2 * 12) ~
    1e-7 at the Neumann ends) matter."""
    errs = []
    for f in (1, 2, 4):
        p = si.Problem(a0=-24, b0=4, T=0.02, dx=4e-3 / f, dt=4e-4 / f, N=1, potential=si.POT_CUBIC,
                       u0_kind="soliton")
        o = oracle_mod.Oracle(p, si.inputs(p), library=library)
        st, uT, _ = o.monodomain()
        assert st == 0, st
        ex = soliton_exact(p.nodes(), p.T)
        errs.append(np.linalg.norm(uT - ex) / np.linalg.norm(ex))
    return errs


# ----------------------------------------------------------------------------
# Linear potential V(t, x) = E(t) x (the paper's V = 5tx, has E = 5t).
# With a(t) = int_0^t E, c(t) = int_0^t 2a, b(t) = -int_0^t a^2, the gauge
#   u(x, t) = e^{i (a x + b)} w(x - c, t)
# turns i u_t + u_xx + E x u = 0 into the free equation i w_t + w_xx = 0
# (substitute: the x-terms cancel by a' = E, the w_x terms by c' = 2a).  For
# E = E0 t: a = E0 t^2/2, c = E0 t^3/3, b = -E0^2 t^5/20; w is the free
# Gaussian of the V = 0 pin.
# ----------------------------------------------------------------------------
def free_gaussian(x, t, x0=-10.0, k=20.0):
    """Free Schrodinger (i u_t + u_xx = 0) from exp(-y^2 + i k y), y = x - x0."""
    y = x - x0
    z = 1 + 4j * t
    return z ** -0.5 * np.exp((-(y * y) + 1j * k * y - 1j * k * k * t) / z)


def linear_potential_exact(x, t, E0):
    a, c, b = E0 * t * t / 2.0, E0 * t ** 3 / 3.0, -E0 * E0 * t ** 5 / 20.0
    return np.exp(1j * (a * x + b)) * free_gaussian(x - c, t, x0=0.0, k=0.0)


def linear_potential_errors(oracle_mod, library=None, E0=2000.0):
    """Relative L2 error of the oracle's monodomain Crank-Nicolson march with
    V(t, x) = E0 t x, given as the separable samples tau(t_n) = E0 t_n,
    xi(x_i) = x_i (the oracle forms W_n = (V_n + V_{n-1})/2 itself),
    against the exact solution along a dt, dx ladder (ratio 2)."""
    errs = []
    for f in (1, 2, 4):
        p = si.Problem(a0=-12, b0=12, T=0.05, dx=4e-3 / f, dt=4e-4 / f, N=1, potential=si.POT_VTX)
        x = p.nodes()
        t = np.arange(p.NT + 1) * p.dt
        arrays = {"u0": free_gaussian(x, 0.0, x0=0.0, k=0.0), "V_x": None, "tau": (E0 * t)[None, :].copy(),
                  "xi": x[None, :].copy(), "g0": None}
        o = oracle_mod.Oracle(p, arrays, library=library)
        st, uT, _ = o.monodomain()
        assert st == 0, st
        ex = linear_potential_exact(x, p.T, E0)
        errs.append(np.linalg.norm(uT - ex) / np.linalg.norm(ex))
    return errs


def orders(errs):
    return [math.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]


# ----------------------------------------------------------------------------
# Transmission-operator symbols.  The continuous operators are
#   S0^2 = e^{-i pi/4} d_t^{1/2},  S0^3 = S0^2 - e^{i pi/4} (V/2) I_t^{1/2},
#   S0^4 = S0^3 - i (d_n V / 4) I_t,
#   S1^2 = e^{-i pi/4} e^{i calV} d_t^{1/2} (e^{-i calV} .),
#   S1^4 = S1^2 - i sgn(d_n V) (sqrt|d_n V|/2) e^{i calV} I_t (sqrt|d_n V|/2 e^{-i calV} .).
# Under the trapezoidal (Crank-Nicolson) time discretisation the symbol of
# d_t is s_d(tau) = (2/dt)(1 - tau)/(1 + tau) in the one-step delay tau, so
# d_t^{1/2}, I_t^{1/2}, I_t become s_d^{1/2}, s_d^{-1/2}, s_d^{-1}; for a
# time-independent V = W the gauge factor e^{i W t_n} modulates the sequence,
# i.e. tau -> tau e^{i W dt} (the z-transform's modulation rule), and the
# gauge operators take the potential-free symbols at the modulated tau.
# ----------------------------------------------------------------------------
def tc_symbol(tc, tau, dt, W, dnW):
    def sd(t):
        return (2.0 / dt) * (1.0 - t) / (1.0 + t)

    em, ep = np.exp(-1j * np.pi / 4), np.exp(1j * np.pi / 4)
    if tc in (si.TC_S02, si.TC_S03, si.TC_S04):
        s = sd(tau)
        val = em * np.sqrt(s)
        if tc in (si.TC_S03, si.TC_S04):
            val -= ep * (W / 2.0) / np.sqrt(s)
        if tc == si.TC_S04:
            val -= 1j * (dnW / 4.0) / s
        return val
    if tc in (si.TC_S12, si.TC_S14):
        s = sd(tau * np.exp(1j * W * dt))
        val = em * np.sqrt(s)
        if tc == si.TC_S14:
            val -= 1j * (dnW / 4.0) / s
        return val
    raise ValueError(tc)


def tc_symbol_error(oracle_mod, tc, library=None, nst=400):
    """Max relative distance between the power series sum_n (S v)_n tau^{n-1}
    of the oracle's discrete operator applied to the unit impulse
    v = e_1 (v_0 = 0) and the symbol above, over several W, d_n W and tau."""
    p = si.config("C1", transmission=tc, potential=si.POT_VX)
    o = oracle_mod.Oracle(p, si.inputs(p), library=library)
    v = np.zeros(nst + 1, np.complex128)
    v[1] = 1.0
    worst = 0.0
    for W, dnW in ((0.0, 0.0), (-3.0, 1.7), (2.5, -0.8), (40.0, 6.0)):
        k = o.tc_apply(v, W, dnW)
        for tau in (0.3, -0.5, 0.4j, 0.2 - 0.3j):
            got = np.sum(k * tau ** np.arange(nst))
            ref = tc_symbol(tc, tau, p.dt, W, dnW)
            worst = max(worst, abs(got - ref) / abs(ref))
    return worst


# ----------------------------------------------------------------------------
# S0^2 transparency: reflection of a packet leaving
# subdomain 1 through b_1 with zero incoming flux, against the solution on a
# larger domain.
# ----------------------------------------------------------------------------
def transparency(oracle_mod, tc, library=None, pade_m=20):
    p = si.Problem(a0=-16, b0=4, T=0.2, dx=2e-3, dt=2e-4, N=2, potential=si.POT_ZERO, transmission=tc,
                   robin_p=40.0, pade_m=pade_m)
    o = oracle_mod.Oracle(p, si.inputs(p), library=library)
    st, _, _, uT, _ = o.march(1, None, None, use_u0=True)
    q = si.Problem(a0=-16, b0=24, T=0.2, dx=2e-3, dt=2e-4, N=1, potential=si.POT_ZERO)
    st2, ub, _ = oracle_mod.Oracle(q, si.inputs(q), library=library).monodomain()
    return np.abs(uT - ub[: p.Nj]).max()
