"""Pins for the oracle's Section 2 maps (penalty, conjugate, prox).

Every check compares the oracle with something other than its own formula:
worked values (tests/golden/penalty_examples.txt, each line cited), the
definition of the proximal operator Eq. (4) minimised numerically,
the definition of the Fenchel conjugate as a brute-force supremum,
and the Moreau decomposition.
"""
import os

import numpy as np
import pytest
from scipy.optimize import minimize_scalar

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "penalty_examples.txt")


def _golden_rows():
    rows = []
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        parts = line.split(None, 6)
        fn, l1, l2, sg, arg, exp = parts[0], *map(float, parts[1:6])
        rows.append((fn, l1, l2, sg, arg, exp, parts[6].strip()))
    return rows


@pytest.mark.parametrize("row", _golden_rows(), ids=lambda r: f"{r[0]}({r[4]})")
def test_golden_values(row):
    fn, l1, l2, sg, arg, exp, cite = row
    if fn == "prox":
        got = oracle.prox(np.array([arg]), sg, l1, l2)[0]
    elif fn == "proxconj":  # argument is u = t/sigma; oracle takes t
        got = oracle.prox_conj(np.array([arg * sg]), sg, l1, l2)[0]
    elif fn == "pstar":
        got = oracle.pstar(np.array([arg]), l1, l2)
    elif fn == "penalty":
        got = oracle.penalty(np.array([arg]), l1, l2)
    else:
        raise AssertionError(fn)
    assert got == pytest.approx(exp, abs=1e-15), cite


def _rand_params(rng, n):
    t = rng.normal(scale=3.0, size=n)
    sigma = np.exp(rng.uniform(np.log(1e-3), np.log(1e3), size=n))
    l1 = np.exp(rng.uniform(np.log(1e-2), np.log(10), size=n))
    l2 = np.exp(rng.uniform(np.log(1e-3), np.log(10), size=n))
    return t, sigma, l1, l2


def test_moreau_identity_10k():
    """x = prox_{σp}(x) + σ·prox_{p*/σ}(x/σ) to 1e-12 relative on 1e4 samples."""
    rng = np.random.default_rng(11)
    t, sigma, l1, l2 = _rand_params(rng, 10_000)
    L = oracle.lib()
    err = 0.0
    for i in range(len(t)):
        p = L.orc_prox(t[i], sigma[i], l1[i], l2[i])
        q = L.orc_prox_conj(t[i], sigma[i], l1[i], l2[i])
        err = max(err, abs(p + sigma[i] * q - t[i]) / max(1.0, abs(t[i])))
    assert err <= 1e-12


def test_prox_is_argmin_of_definition():
    """Eq. (6) left equals argmin_u p(u) + (u − t)²/(2σ) (definition Eq. (4))."""
    rng = np.random.default_rng(5)
    t, sigma, l1, l2 = _rand_params(rng, 200)
    for i in range(len(t)):
        f = lambda u: l1[i] * abs(u) + 0.5 * l2[i] * u * u + (u - t[i]) ** 2 / (2 * sigma[i])
        lo, hi = -abs(t[i]) - 1, abs(t[i]) + 1
        res = minimize_scalar(f, bounds=(lo, hi), method="bounded", options={"xatol": 1e-12})
        p = oracle.lib().orc_prox(t[i], sigma[i], l1[i], l2[i])
        # compare objective values (the argmin of a strongly convex 1-D function)
        assert f(p) <= f(res.x) + 1e-10 * max(1.0, abs(f(res.x)))
        assert abs(p - res.x) <= 1e-5 * max(1.0, abs(t[i]))


def test_prox_conj_is_argmin_of_definition():
    """Eq. (6) right equals argmin_v p*(v)/σ + ½(v − t/σ)² (Eq. (4) applied to p*/σ), with p*
    taken from its definition as a supremum (not from Prop. 1)."""
    rng = np.random.default_rng(6)
    t, sigma, l1, l2 = _rand_params(rng, 60)
    for i in range(len(t)):
        s, a, c = sigma[i], l1[i], l2[i]

        def pstar_def(v):  # sup_x v x − a|x| − c x²/2, closed in 1-D: attained at soft(v,a)/c
            xs = np.linspace(-2 * (abs(v) + 1) / c, 2 * (abs(v) + 1) / c, 20001)
            vals = v * xs - a * np.abs(xs) - 0.5 * c * xs * xs
            j = int(np.argmax(vals))
            # refine around the grid maximiser
            r = minimize_scalar(lambda x: -(v * x - a * abs(x) - 0.5 * c * x * x),
                                bounds=(xs[max(j - 1, 0)], xs[min(j + 1, len(xs) - 1)]), method="bounded",
                                options={"xatol": 1e-13})
            return max(vals[j], -r.fun)

        u = t[i] / s
        f = lambda v: pstar_def(v) / s + 0.5 * (v - u) ** 2
        q = oracle.lib().orc_prox_conj(t[i], s, a, c)
        res = minimize_scalar(f, bounds=(-abs(u) - a - 1, abs(u) + a + 1), method="bounded",
                              options={"xatol": 1e-11})
        assert f(q) <= f(res.x) + 1e-8 * max(1.0, abs(f(res.x)))


def test_pstar_matches_grid_supremum():
    """Prop. 1 vs the conjugate's definition sup_x z x − p(x) on a dense grid, within 1e-4."""
    xs = np.linspace(-60, 60, 1_200_001)
    rng = np.random.default_rng(7)
    for _ in range(40):
        l1 = rng.uniform(0.1, 3)
        l2 = rng.uniform(0.2, 3)
        z = rng.uniform(-8, 8)
        sup = np.max(z * xs - l1 * np.abs(xs) - 0.5 * l2 * xs * xs)
        assert abs(oracle.pstar(np.array([z]), l1, l2) - sup) <= 1e-4


def test_pstar_lasso_indicator():
    """λ2 = 0: p* is the indicator of ‖z‖∞ ≤ λ1 (Eq. (2))."""
    assert oracle.pstar(np.array([0.5, -1.0]), 1.0, 0.0) == 0.0
    assert oracle.pstar(np.array([0.5, -1.5]), 1.0, 0.0) == np.inf


def test_fenchel_young():
    """p(x) + p*(z) ≥ zᵀx, with equality at z = λ1 sign(x) + λ2 x (subgradient),."""
    rng = np.random.default_rng(8)
    for _ in range(200):
        n = 7
        l1, l2 = rng.uniform(0.1, 2), rng.uniform(0.1, 2)
        x = rng.normal(size=n)
        z = rng.normal(scale=3, size=n)
        assert oracle.penalty(x, l1, l2) + oracle.pstar(z, l1, l2) >= z @ x - 1e-12
        zs = l1 * np.sign(x) + l2 * x
        lhs = oracle.penalty(x, l1, l2) + oracle.pstar(zs, l1, l2)
        assert lhs == pytest.approx(zs @ x, rel=1e-10, abs=1e-12)


def test_prox_lipschitz_monotone():
    """prox_{σp} is 1/(1+σλ2)-Lipschitz and nondecreasing."""
    rng = np.random.default_rng(9)
    t = np.sort(rng.normal(scale=5, size=2000))
    for sigma, l1, l2 in [(1.0, 1.0, 1.0), (0.01, 3.0, 0.5), (50.0, 0.2, 2.0)]:
        p = oracle.prox(t, sigma, l1, l2)
        assert np.all(np.diff(p) >= 0)
        assert np.all(np.abs(np.diff(p)) <= np.diff(t) / (1 + sigma * l2) * (1 + 1e-12) + 1e-15)
