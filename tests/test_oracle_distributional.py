"""Pins for the C51 machinery of the oracle (a9, a10): SPEC worked examples, mass, mean
preservation, monotone shift, brute-force hat form, exact landing, CE closed forms."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


def _proj(case, shift=0.0):
    vmin, vmax, n = case["support"]
    p = np.array([case["probs"]], float)
    return O.categorical_project(p, np.array([case["r"]]), np.array([float(case["not_done"])]),
                                 case["gamma"], np.array([shift]), vmin, vmax)[0]


@pytest.mark.parametrize("key", ["project_gamma0", "project_hand", "project_terminal"])
def test_projection_spec_examples(key):
    c = GOLD[key]
    assert np.abs(_proj(c) - np.array(c["expected"])).max() < 1e-12


@pytest.mark.parametrize("key", ["support_a", "support_b", "support_c"])
def test_support_spec274(key):
    c = GOLD[key]
    z, dz = O.make_support(c["v_min"], c["v_max"], c["n"])
    if "atoms" in c:
        assert np.allclose(z, c["atoms"], atol=0)
    if "dz" in c:
        assert dz == c["dz"]
    if "atom37" in c:
        assert z[37] == c["atom37"]


def test_support_invalid_spec272():
    with pytest.raises(ValueError):
        O.make_support(1.0, -1.0, 5)
    with pytest.raises(ValueError):
        O.make_support(-1.0, 1.0, 1)


@pytest.mark.parametrize("key", ["expected_value_sym", "expected_value_point"])
def test_expected_value_spec292(key):
    c = GOLD[key]
    z, _ = O.make_support(*c["support"])
    assert abs(O.expected_value(np.array(c["probs"], float), z) - c["expected"]) < 1e-15


def _rand_case(rng, B, N):
    p = rng.dirichlet(np.ones(N), size=B)
    r = rng.uniform(-1, 1, B)
    nd = (rng.uniform(size=B) > 0.2).astype(float)
    sh = rng.uniform(-2, 2, B)
    return p, r, nd, sh


def test_projection_mass_spec306():
    rng = np.random.default_rng(0)
    p, r, nd, sh = _rand_case(rng, 200, 51)
    m = O.categorical_project(p, r * 20, nd, 0.99, sh, -10.0, 10.0)
    assert np.abs(m.sum(axis=1) - 1).max() < 1e-12
    assert (m >= 0).all()


def test_projection_mean_preserving_spec307():
    rng = np.random.default_rng(1)
    N = 51
    z, _ = O.make_support(-10.0, 10.0, N)
    p = np.zeros((50, N))
    p[:, 15:36] = rng.dirichlet(np.ones(21), size=50)  # support well inside
    r = rng.uniform(-1, 1, 50)
    m = O.categorical_project(p, r, np.ones(50), 0.9, np.zeros(50), -10.0, 10.0)
    assert np.abs(m @ z - (r + 0.9 * (p @ z))).max() < 1e-12


def test_projection_monotone_shift_spec308():
    rng = np.random.default_rng(2)
    N = 51
    z, _ = O.make_support(-10.0, 10.0, N)
    p = np.zeros((20, N))
    p[:, 20:31] = rng.dirichlet(np.ones(11), size=20)
    r = rng.uniform(-1, 1, 20)
    delta = 0.37
    m0 = O.categorical_project(p, r, np.ones(20), 0.95, np.zeros(20), -10.0, 10.0)
    m1 = O.categorical_project(p, r + delta, np.ones(20), 0.95, np.zeros(20), -10.0, 10.0)
    assert np.abs((m1 - m0) @ z - delta).max() < 1e-12


def test_projection_vs_hat_form_spec309():
    """Brute force, independent formulation: m_k = sum_j p_j max(0, 1 - |b_j - k|)."""
    rng = np.random.default_rng(3)
    for _ in range(1000):
        N = int(rng.integers(2, 8))
        vmin = float(rng.uniform(-3, 0))
        vmax = vmin + float(rng.uniform(0.5, 4))
        p, r, nd, sh = _rand_case(rng, 1, N)
        g = float(rng.uniform(0, 1))
        m = O.categorical_project(p, r * 3, nd, g, sh, vmin, vmax)[0]
        z = np.linspace(vmin, vmax, N)
        gj = np.clip(r[0] * 3 + nd[0] * g * (z - sh[0]), vmin, vmax)
        bj = (gj - vmin) / ((vmax - vmin) / (N - 1))
        hat = np.array([sum(p[0, j] * max(0.0, 1 - abs(bj[j] - k)) for j in range(N)) for k in range(N)])
        assert np.abs(m - hat).max() < 1e-9


def test_projection_exact_landing_dyadic():
    c = GOLD["exact_landing_dyadic"]
    vmin, vmax, n = c["support"]
    z, dz = O.make_support(vmin, vmax, n)
    p = np.zeros((1, n))
    p[0, int(np.where(z == c["point_mass_atom_value"])[0][0])] = 1.0
    m = O.categorical_project(p, np.array([c["r"]]), np.array([1.0]), c["gamma"], np.array([c["alpha_logp"]]),
                              vmin, vmax)[0]
    k = int(np.where(z == c["expected_atom_value"])[0][0])
    assert m[k] == 1.0 and m.sum() == 1.0


def test_projection_entropy_fold_spec315():
    """Shifting atoms by alpha log pi equals folding it into the reward:
    r' = r - not_done gamma alpha log pi (Q21)."""
    rng = np.random.default_rng(4)
    p, r, nd, sh = _rand_case(rng, 30, 21)
    a = O.categorical_project(p, r, nd, 0.97, sh, -5.0, 5.0)
    b = O.categorical_project(p, r - nd * 0.97 * sh, nd, 0.97, np.zeros(30), -5.0, 5.0)
    assert np.abs(a - b).max() < 1e-9


def test_projection_linear_in_p_q20():
    """Averaging head probabilities then projecting == averaging projected targets."""
    rng = np.random.default_rng(5)
    p1, r, nd, sh = _rand_case(rng, 10, 11)
    p2 = rng.dirichlet(np.ones(11), size=10)
    mix = O.categorical_project(0.5 * (p1 + p2), r, nd, 0.9, sh, -3.0, 3.0)
    sep = 0.5 * (O.categorical_project(p1, r, nd, 0.9, sh, -3.0, 3.0) + O.categorical_project(p2, r, nd, 0.9, sh, -3.0, 3.0))
    assert np.abs(mix - sep).max() < 1e-12


def test_identical_point_mass_heads_spec354():
    z, _ = O.make_support(-10.0, 10.0, 51)
    p = np.zeros((1, 51))
    p[0, 30] = 1.0
    m = O.categorical_project(p, np.array([0.5]), np.array([1.0]), 0.99, np.array([0.0]), -10.0, 10.0)[0]
    g = 0.5 + 0.99 * z[30]
    assert abs(m @ z - g) < 1e-12 and np.count_nonzero(m) == 2


def test_ce_uniform_is_log_n_spec301():
    for n in (3, 51, 101):
        m = np.full((4, n), 1.0 / n)
        assert abs(O.cross_entropy(m, np.zeros((4, n))) - math.log(n)) < 1e-12


def test_ce_grad_fd_spec303():
    rng = np.random.default_rng(6)
    logits = rng.standard_normal((4, 7))
    m = rng.dirichlet(np.ones(7), size=4)
    an = (O.softmax(logits) - m) / 4
    h = 1e-6
    for b in range(4):
        for k in range(7):
            lp, lm = logits.copy(), logits.copy()
            lp[b, k] += h
            lm[b, k] -= h
            num = (O.cross_entropy(m, lp) - O.cross_entropy(m, lm)) / (2 * h)
            assert abs(num - an[b, k]) < 1e-8


def test_ce_perfect_prediction_limit_spec302():
    logits = np.array([[0.0, 60.0, 0.0]])
    assert O.cross_entropy(np.array([[0.0, 1.0, 0.0]]), logits) < 1e-20


def test_softmax_rows_sum_spec220():
    x = np.random.default_rng(7).standard_normal((9, 101)) * 10
    assert np.abs(O.softmax(x).sum(axis=1) - 1).max() < 1e-12
