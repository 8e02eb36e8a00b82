"""Oracle pins for reading R27: the nodal assembly f_int,k = sum of f_{e,a} over the node's
active incidences (assembly operator A) is evaluated as the exact real sum of
the fp64 contributions rounded once to the nearest fp64, ties to even (oracle/exact_sum.h).

Independent check: Python's fractions.Fraction holds every double exactly, sums exactly, and
float(Fraction) is correctly rounded (round half to even).  Cases are chosen so that the
plausible mistakes fail: a plain sequential sum (cancellation, tiny terms beside a tie),
truncation or round-half-up (ties), a wrong subnormal precision (sums below 2^-1022), a
sign error in the negation path (negative results), a dropped carry (many large terms).
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import cem_inputs as ci
import oracle


def exact(xs):
    return float(sum((Fraction(float(x)) for x in xs), Fraction(0)))


@pytest.mark.parametrize("xs", [
    [],                                                  # empty -> +0.0
    [1.0],
    [1.0, 2.0 ** -53],                                   # tie -> even (1.0)
    [1.0, 2.0 ** -53, 2.0 ** -200],                      # tie broken by a tiny term -> up
    [1.0 + 2.0 ** -52, 2.0 ** -53],                      # tie -> even (up)
    [1.0, -(2.0 ** -54), 2.0 ** -53],                    # below the tie -> 1.0
    [1e16, 1.0, -1e16],                                  # catastrophic cancellation: 1.0
    [1e300, 1e-300, -1e300],                             # 1e-300 exactly
    [-1.0, -(2.0 ** -53)],                               # negative tie -> -1.0
    [-3.5, 1.25, -0.125],
    [5e-324, 5e-324, 5e-324],                            # subnormals
    [2.0 ** -1022, -(2.0 ** -1074)],                     # normal minus a subnormal step
    [2.0 ** -1060, 3 * 2.0 ** -1074, 2.0 ** -1075 * 0],  # subnormal precision
    [1.7976931348623157e308, -1.7976931348623157e308, 1.0],
    [0.1] * 10,                                          # 1.0000000000000000555 -> 1.0
    [1.0, -1.0],                                         # exact zero -> +0.0
])
def test_exact_sum_cases(xs):
    got = oracle.exact_sum(np.array(xs, dtype=np.float64))
    want = exact(xs)
    assert got == want, (xs, got, want)
    if want == 0.0:
        assert math.copysign(1.0, got) == 1.0


def test_exact_sum_random_vs_fractions():
    rng = np.random.default_rng(2027)
    for trial in range(400):
        n = int(rng.integers(1, 40))
        kind = trial % 4
        if kind == 0:      # force-like: comparable magnitudes, cancelling signs
            xs = rng.standard_normal(n) * 10.0 ** rng.integers(-8, 8)
        elif kind == 1:    # wide exponent spread (wave-front tails beside the bulk)
            xs = rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, size=n).astype(float)
        elif kind == 2:    # nearly cancelling pairs plus a residual
            a = rng.standard_normal(n) * 1e3
            xs = np.concatenate([a, -a * (1 + 1e-15 * rng.standard_normal(n)), [1e-9]])
        else:              # many large terms (carry propagation)
            xs = np.full(n, 1.7e308 / 64) * np.where(rng.random(n) < 0.7, 1.0, -1.0)
        xs = np.asarray(xs, dtype=np.float64)
        assert oracle.exact_sum(xs) == exact(xs), (trial, xs)
    # a plain sequential sum differs on some of these (the pin is not vacuous)
    xs = np.array([1.0, 2.0 ** -53, 2.0 ** -200])
    assert (xs[0] + xs[1]) + xs[2] != exact(xs)


def test_exact_sum_order_independent():
    rng = np.random.default_rng(5)
    xs = rng.standard_normal(64) * 10.0 ** rng.integers(-20, 20, size=64).astype(float)
    ref = oracle.exact_sum(xs)
    for _ in range(20):
        assert oracle.exact_sum(rng.permutation(xs)) == ref


def test_exact_sum_nonfinite_propagates():
    assert math.isinf(oracle.exact_sum(np.array([1.0, np.inf, 2.0])))
    assert math.isnan(oracle.exact_sum(np.array([1.0, np.inf, -np.inf])))
    assert math.isnan(oracle.exact_sum(np.array([np.nan, 0.0])))


def test_internal_force_is_exact_assembly():
    """f_int of the oracle = the correctly rounded exact sum of its element contributions over
    each node's active incidences (inactive tets excluded)."""
    p = ci.notched_plate(cells=(5, 3, 2), dims=(0.03, 0.02, 0.01), seed=3, steps=0)
    st = p.tet_state.copy()
    rng = np.random.default_rng(1)
    st[rng.random(st.size) < 0.15] = 0
    p.tet_state = st
    o = oracle.Oracle(p)
    u = rng.standard_normal((p.n_nodes, 3)) * 1e-5
    f = o.internal_force(u)
    fe = o.element_forces()
    inc = [[] for _ in range(p.n_nodes)]
    for e, t in enumerate(p.tets):
        if st[e]:
            for a, k in enumerate(t):
                inc[k].append((e, a))
    for k in range(p.n_nodes):
        for c in range(3):
            assert f[k, c] == exact([fe[e, a, c] for e, a in inc[k]]), (k, c)
    # inactive tets contribute nothing: their slots hold zeros and the incidence filter skips them
    assert np.all(fe[st == 0] == 0.0)
