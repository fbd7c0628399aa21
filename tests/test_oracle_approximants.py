"""Pins for the oracle's elementary-function approximants (Tables 1-4).

What pins them (none of these re-types the oracle's code):
* the paper's printed coefficients (tests/golden/paper_tables.txt) must be
  the oracle's tables, digit for digit;
* each approximant's measured max error against the mathematical function it
  approximates (numpy/libm, not the oracle) on a >= 1e6-point grid lies in
  [1.0, 1.2] x the paper's printed eps (Eq. 1);
* an independent Remez exchange (oracle/minimax.py, numpy) re-derives Tables
  1-2 (eps and coefficients within 1e-4 relative) and the printed
  polynomials equioscillate (n+2 alternating extrema, Chebyshev theorem);
* SPEC.md's worked examples and cutoff rules
  (P:163).
"""
import math

import numpy as np
import pytest

import oracle
from oracle import minimax as mm

G = lambda t: 2.0 * np.arcsin(t / np.sqrt(2.0))   # Eq. 7 composite, reading R6
EXPN = lambda z: np.exp(-z)
ENT = lambda z: z * np.log(z)


def test_oracle_tables_are_the_paper_tables(paper_tables):
    pairs = dict(ARCSIN="arcsin", ARCCOS="arccos", EXP_P2="exp_p2", EXP_P3="exp_p3",
                 EXP_P4="exp_p4", EXP_NUM="exp_num", EXP_DEN="exp_den", ENT_NUM="ent_num",
                 ENT_DEN="ent_den")
    for g, o in pairs.items():
        assert list(oracle.coeffs(o)) == paper_tables[g]["values"], g
    t_exp, t_ent, kappa = oracle.coeffs("constants")
    assert t_exp == paper_tables["T_EXP"]["values"][0]
    assert t_ent == paper_tables["T_ENT"]["values"][0]
    assert kappa == paper_tables["KAPPA"]["values"][0]


CERT = [
    # (oracle fn, exact function, golden row)
    ("p_arccos", np.arccos, "ARCCOS"),
    ("p_arcsin", G, "ARCSIN"),
    ("exp_poly2", EXPN, "EXP_P2"),
    ("exp_poly3", EXPN, "EXP_P3"),
    ("exp_poly4", EXPN, "EXP_P4"),
    ("exp_rational", EXPN, "EXP_NUM"),
    ("ent_mm", ENT, "ENT_NUM"),
]


@pytest.mark.parametrize("fn,exact,row", CERT)
def test_certified_error_matches_paper_eps(fn, exact, row, paper_tables):
    a, b = paper_tables[row]["interval"]
    eps_paper = paper_tables[row]["eps"]
    eps, _ = mm.certify(lambda z: oracle.eval_fn(fn, z), exact, a, b, npts=1_000_001)
    # A printed 7-digit table cannot beat the true minimax error by more than
    # rounding; it may exceed it by coefficient rounding (<= 1.2x).
    assert 0.999 * eps_paper <= eps <= 1.2 * eps_paper, (fn, eps, eps_paper)


def test_wrong_readings_fail_certification():
    """The readings R6 (ARCSIN row is g(tau) on [0, 1/sqrt 2]) and R10
    (natural log) are the only ones the printed eps admit."""
    eps_plain_asin, _ = mm.certify(lambda z: oracle.eval_fn("p_arcsin", z), np.arcsin, 0, 0.5)
    assert eps_plain_asin > 0.1
    eps_log10, _ = mm.certify(lambda z: oracle.eval_fn("ent_mm", z), lambda z: z * np.log10(z), 0.05, 1)
    assert eps_log10 > 0.1


def test_composite_arccos_error_and_branch():
    """Eqs. 6-7: composite on [0,1] within 1.2 x max(Table 1 eps); the branch
    at z = 0.5 picks the ARCSIN row (P:97 'for z >= 0.5')."""
    eps, _ = mm.certify(lambda z: oracle.eval_fn("arccos_mm", z), np.arccos, 0.0, 1.0)
    assert eps <= 1.2 * 2.097814e-05
    v = oracle.eval_fn("arccos_mm", [0.5])[0]
    assert v == pytest.approx(float(mm.polyval(oracle.coeffs("arcsin"), np.sqrt(0.5))), abs=0, rel=1e-15)
    # the two rows differ at the branch point by ~3.1e-5 (so the branch matters)
    va = float(mm.polyval(oracle.coeffs("arccos"), 0.5))
    assert abs(va - v) > 3e-5


@pytest.mark.parametrize("deg,row", [(2, "EXP_P2"), (3, "EXP_P3"), (4, "EXP_P4")])
def test_remez_reproduces_table2(deg, row, paper_tables):
    c, eps, _ = mm.remez(EXPN, deg, 0.0, 10.0)
    assert eps == pytest.approx(paper_tables[row]["eps"], rel=1e-4)
    np.testing.assert_allclose(c, paper_tables[row]["values"], rtol=1e-4)


@pytest.mark.parametrize("f,a,b,row", [(np.arccos, 0.0, 0.5, "ARCCOS"),
                                       (G, 0.0, 1 / math.sqrt(2), "ARCSIN")])
def test_remez_reproduces_table1(f, a, b, row, paper_tables):
    c, eps, _ = mm.remez(f, 4, a, b)
    assert eps == pytest.approx(paper_tables[row]["eps"], rel=1e-4)
    np.testing.assert_allclose(c, paper_tables[row]["values"], rtol=1e-4)


def test_remez_trivial_cases():
    c, eps, _ = mm.remez(lambda z: 3 * z + 2, 1, 0.0, 1.0)
    assert eps < 1e-12
    np.testing.assert_allclose(c, [2.0, 3.0], atol=1e-12)


@pytest.mark.parametrize("table,f,a,b", [("arccos", np.arccos, 0, 0.5),
                                         ("arcsin", G, 0, 1 / math.sqrt(2)),
                                         ("exp_p4", EXPN, 0, 10)])
def test_printed_polynomials_equioscillate(table, f, a, b):
    z, e = mm.extrema(oracle.coeffs(table), f, a, b)
    deg = len(oracle.coeffs(table)) - 1
    assert len(z) == deg + 2
    assert np.all(np.sign(e[1:]) == -np.sign(e[:-1]))
    lv = np.abs(e)
    assert (lv.max() - lv.min()) / lv.max() < 0.06


def test_spec_examples():
    # S:121 / S:212 : P_acos(0) = a0
    assert oracle.eval_fn("p_arccos", [0.0])[0] == 1.570786
    # S:213 : z = 1 -> tau = 0 -> a0 of ARCSIN, within eps of acos(1) = 0
    assert oracle.eval_fn("arccos_mm", [1.0])[0] == 2.097797e-05
    # S:214 : arccos(0.25)
    assert abs(oracle.eval_fn("arccos_mm", [0.25])[0] - math.acos(0.25)) < 2.1e-5
    # S:131 : Table 3 at 0 within eps of 1 
    assert abs(oracle.eval_fn("exp_rational", [0.0])[0] - 1.0) < 2.5e-6
    # S:234 : exp approx at 5
    assert abs(oracle.eval_fn("exp_rational", [5.0])[0] - math.exp(-5)) < 2.5e-6
    # S:232 / P:163 : cutoff, 0 outside [0, T]
    assert oracle.eval_fn("exp_rational", [11.0])[0] == 0.0
    assert oracle.eval_fn("exp_poly4", [10.5])[0] == 0.0
    # P:163 : e^{-T} = 4.539993e-05
    assert round(oracle.eval_fn("exp_exact", [10.0])[0], 11) == 4.539993e-05
    # S:133 / S:253 : ENT rational at 1 within eps of 0
    assert abs(oracle.eval_fn("ent_mm", [1.0])[0]) < 1.2 * 7.342477e-07
    # S:254 : ENT at 0.5
    assert abs(oracle.eval_fn("ent_mm", [0.5])[0] - 0.5 * math.log(0.5)) < 1e-6
    # S:252 / P:232 : cutoff below 0.05
    assert oracle.eval_fn("ent_mm", [0.01])[0] == 0.0
    assert oracle.eval_fn("ent_mm", [0.05])[0] != 0.0
    # S:243-244 : exact ENT conventions
    assert oracle.eval_fn("ent_exact", [0.0])[0] == 0.0
    assert oracle.eval_fn("ent_exact", [1 / math.e])[0] == pytest.approx(-1 / math.e, rel=1e-15)


def test_rational_denominators_positive():
    z = np.linspace(0, 10, 200001)
    assert mm.polyval(oracle.coeffs("exp_den"), z).min() > 0.03
    s = np.linspace(0.05, 1, 200001)
    assert mm.polyval(oracle.coeffs("ent_den"), s).min() > 0.03


def test_arccos_mm_monotone():
    """non-increasing within 2 eps slack."""
    z = np.linspace(0, 1, 10001)
    v = oracle.eval_fn("arccos_mm", z)
    assert np.all(np.diff(v) <= 2 * 2.097814e-05)
