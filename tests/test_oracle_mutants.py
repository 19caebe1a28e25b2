"""The oracle pins catch plausible mistakes: each test builds the oracle with
one deliberate error planted (-DOR_MUTANT=k, hooks in oracle/swr_oracle.c)
and checks that the pin which guards that part of the arithmetic rejects it,
while the real oracle passes the same pin (tests/test_oracle_pins.py).

  k  planted error                                   pin that must fail
  1  NL load b_f with the wrong sign     soliton closed form, order 2
  2  W_n = V_n instead of (V_n + V_{n-1})/2  V = E t x closed form, order 2
  3  S0^3/S0^4 alpha term with the wrong sign        operator symbol
  4  S0^4 gamma term with the wrong sign             operator symbol
  5  S1 gauge phase e^{-i calW} for e^{+i calW}      operator symbol
  6  S1^4 extra term with the wrong sign             operator symbol
  7  sqrt(dt) for sqrt(dt/2) in the alpha term       operator symbol
  8  S0^2 history beta_{n-s-1} for beta_{n-s}        S0^2 transparency
"""
import pytest

import oracle_checks as oc
import swr_inputs as si


def test_nl_load_sign_is_caught(oracle_mod):
    good = oc.orders(oc.nl_soliton_errors(oracle_mod))
    bad_errs = oc.nl_soliton_errors(oracle_mod, oracle_mod.lib_mutant(1))
    bad = oc.orders(bad_errs)
    assert min(good) >= 1.9
    assert min(bad) < 1.0 and bad_errs[-1] > 0.1, (bad, bad_errs)


def test_potential_midpoint_is_caught(oracle_mod):
    good = oc.orders(oc.linear_potential_errors(oracle_mod))
    bad = oc.orders(oc.linear_potential_errors(oracle_mod, oracle_mod.lib_mutant(2)))
    assert min(good) >= 1.9
    assert max(bad) < 1.2, bad   # first order: W_n at t_n is an O(dt) error


@pytest.mark.parametrize("k,tc", [(3, si.TC_S03), (3, si.TC_S04), (4, si.TC_S04), (5, si.TC_S12),
                                  (5, si.TC_S14), (6, si.TC_S14), (7, si.TC_S03)])
def test_operator_coefficients_are_caught(oracle_mod, k, tc):
    assert oc.tc_symbol_error(oracle_mod, tc) <= 1e-13
    assert oc.tc_symbol_error(oracle_mod, tc, oracle_mod.lib_mutant(k)) > 1e-4


def test_history_index_is_caught(oracle_mod):
    assert oc.transparency(oracle_mod, si.TC_S02) <= 1e-4
    assert oc.transparency(oracle_mod, si.TC_S02, oracle_mod.lib_mutant(8)) > 1e-2
