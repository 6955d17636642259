"""Pins for the oracle's float layers: conv (direct vs im2col), LN statistics,
finite-difference backward of every layer, tanh-Gaussian closed form + density."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


def fd_check(f, x, analytic, n_probe=12, h=1e-6, rtol=2e-6, seed=0):
    """Central differences of scalar f at n_probe random coordinates of x (in place)."""
    rng = np.random.default_rng(seed)
    flat = x.reshape(-1)
    an = analytic.reshape(-1)
    scale = max(np.abs(an).max(), 1e-12)
    for i in rng.choice(flat.size, min(n_probe, flat.size), replace=False):
        old = flat[i]
        flat[i] = old + h
        fp = f()
        flat[i] = old - h
        fm = f()
        flat[i] = old
        num = (fp - fm) / (2 * h)
        assert abs(num - an[i]) <= rtol * scale + 1e-9, (i, num, an[i])


def test_conv_direct_vs_im2col():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 3, 16, 16))
    w = rng.standard_normal((4, 3, 3, 3))
    b = rng.standard_normal(4)
    for stride in (1, 2):
        y, _ = O.conv2d_fwd(x, w, b, stride)
        assert np.abs(y - O.conv2d_direct(x, w, b, stride)).max() < 1e-12
    assert y.shape == (2, 4, 7, 7)


def test_conv_bwd_fd():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((2, 3, 9, 9))
    w = rng.standard_normal((4, 3, 3, 3))
    b = rng.standard_normal(4)
    R = rng.standard_normal((2, 4, 4, 4))
    f = lambda: float((O.conv2d_fwd(x, w, b, 2)[0] * R).sum())
    _, cache = O.conv2d_fwd(x, w, b, 2)
    dw, db, dx = O.conv2d_bwd(R, cache)
    fd_check(f, w, dw)
    fd_check(f, b, db)
    fd_check(f, x, dx)


def _enc_params(C, rng):
    return {"enc.conv1.w": rng.uniform(-0.3, 0.3, (C, 3, 3, 3)), "enc.conv1.b": rng.uniform(-0.1, 0.1, C),
            "enc.conv2.w": rng.uniform(-0.3, 0.3, (C, C, 3, 3)), "enc.conv2.b": rng.uniform(-0.1, 0.1, C)}


def test_encoder_shapes_and_bwd_fd():
    rng = np.random.default_rng(2)
    p = _enc_params(4, rng)
    x = rng.uniform(0, 1, (3, 3, 16, 16))
    h, cache = O.encoder_fwd(p, x)
    assert h.shape == (3, 4 * 25)
    R = rng.standard_normal(h.shape)
    f = lambda: float((O.encoder_fwd(p, x)[0] * R).sum())
    g = O.encoder_bwd(R, cache)
    for k in p:
        fd_check(f, p[k], g[k])


def test_layernorm_stats_spec225():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((16, 50)) * 3 + 2
    y, (xh, rstd, g) = O.layernorm_fwd(x, np.ones(50), np.zeros(50), 1e-5)
    assert np.abs(xh.mean(axis=1)).max() < 1e-12
    assert np.abs(xh.var(axis=1) - 1).max() < 1e-5


def test_layernorm_bwd_fd():
    rng = np.random.default_rng(4)
    x = rng.standard_normal((5, 9))
    g = rng.uniform(0.5, 1.5, 9)
    b = rng.standard_normal(9)
    R = rng.standard_normal((5, 9))
    f = lambda: float((O.layernorm_fwd(x, g, b, 1e-5)[0] * R).sum())
    _, cache = O.layernorm_fwd(x, g, b, 1e-5)
    dx, dg, db = O.layernorm_bwd(R, cache)
    fd_check(f, x, dx)
    fd_check(f, g, dg)
    fd_check(f, b, db)


def _mlp_params(prefix, n_in, hid, n_out, rng):
    return {f"{prefix}.l1.w": rng.uniform(-0.5, 0.5, (hid, n_in)), f"{prefix}.l1.b": rng.uniform(-0.1, 0.1, hid),
            f"{prefix}.ln1.g": rng.uniform(0.7, 1.3, hid), f"{prefix}.ln1.b": rng.uniform(-0.2, 0.2, hid),
            f"{prefix}.l2.w": rng.uniform(-0.5, 0.5, (hid, hid)), f"{prefix}.l2.b": rng.uniform(-0.1, 0.1, hid),
            f"{prefix}.ln2.g": rng.uniform(0.7, 1.3, hid), f"{prefix}.ln2.b": rng.uniform(-0.2, 0.2, hid),
            f"{prefix}.l3.w": rng.uniform(-0.5, 0.5, (n_out, hid)), f"{prefix}.l3.b": rng.uniform(-0.1, 0.1, n_out)}


def test_mlp_bwd_fd():
    rng = np.random.default_rng(5)
    p = _mlp_params("q", 7, 16, 5, rng)
    x = rng.standard_normal((4, 7))
    R = rng.standard_normal((4, 5))
    f = lambda: float((O.mlp_fwd(p, "q", x, 1e-5)[0] * R).sum())
    _, cache = O.mlp_fwd(p, "q", x, 1e-5)
    g, dx = O.mlp_bwd(R, cache, "q", p)
    for k in p:
        fd_check(f, p[k], g[k])
    fd_check(f, x, dx)


def test_projection_bwd_fd():
    rng = np.random.default_rng(6)
    p = {"c.proj.w": rng.uniform(-0.3, 0.3, (8, 20)), "c.proj.b": rng.uniform(-0.1, 0.1, 8),
         "c.proj.ln.g": rng.uniform(0.7, 1.3, 8), "c.proj.ln.b": rng.uniform(-0.2, 0.2, 8)}
    h = rng.standard_normal((4, 20))
    R = rng.standard_normal((4, 8))
    f = lambda: float((O.projection_fwd(p, "c", h, 1e-5)[0] * R).sum())
    z, cache = O.projection_fwd(p, "c", h, 1e-5)
    assert np.abs(z).max() < 1
    g, dh = O.projection_bwd(R, cache, "c", p, need_dh=True)
    for k in p:
        fd_check(f, p[k], g[k])
    fd_check(f, h, dh)


# ---- tanh-Gaussian (a7) --------------------------------------------------------------
def test_logprob_u0_spec202():
    g = GOLD["logprob_u0"]
    lo, hi = -5.0, 2.0
    # choose l with log sigma = 0: lo + (hi-lo)/2 (tanh l + 1) = 0
    l = math.atanh(-2 * lo / (hi - lo) - 1)
    out = np.array([[g["mu"], l]])
    a, logp, _ = O.tanh_gaussian_fwd(out, np.zeros((1, 1)), lo, hi)
    assert a[0, 0] == 0.0
    assert abs(logp[0] - g["expected"]) < g["tol"]
    assert abs(logp[0] - (-0.5 * math.log(2 * math.pi) - math.log(1 + 1e-6))) < 1e-12


def test_log_std_bounds_spec228():
    out = np.array([[0.0, -1e3], [0.0, 1e3], [0.0, 0.0]])
    _, _, (eps, tl, std, a, lo, hi) = O.tanh_gaussian_fwd(out, np.zeros((3, 1)), -5.0, 2.0)
    assert np.all(std >= math.exp(-5) - 1e-15) and np.all(std <= math.exp(2) + 1e-12)


def test_action_is_tanh_u_spec203():
    rng = np.random.default_rng(8)
    out = rng.standard_normal((6, 4))
    eps = rng.standard_normal((6, 2))
    a, _, (e, tl, std, aa, lo, hi) = O.tanh_gaussian_fwd(out, eps, -5.0, 2.0)
    assert np.array_equal(a, np.tanh(out[:, :2] + std * eps))


def test_tanh_gaussian_density_spec204():
    """Monte Carlo: histogram of a = tanh(mu + sigma eps) vs exp(log pi(a)), TV < 0.01."""
    mu, log_std = 0.3, math.log(0.6)
    lo, hi = -5.0, 2.0
    l = math.atanh((log_std - lo) * 2 / (hi - lo) - 1)
    n = 1_000_000
    eps = np.random.default_rng(9).standard_normal((n, 1))
    a, _, _ = O.tanh_gaussian_fwd(np.tile([[mu, l]], (n, 1)), eps, lo, hi)
    edges = np.linspace(-1, 1, 201)
    hist, _ = np.histogram(a[:, 0], bins=edges)
    emp = hist / n
    # density on a fine grid inside each bin: invert a -> eps, evaluate log pi (with the 1e-6)
    fine = np.linspace(-1, 1, 200 * 50 + 1)[1:-1]
    u = np.arctanh(fine)
    e = (u - mu) / math.exp(log_std)
    _, logp, _ = O.tanh_gaussian_fwd(np.tile([[mu, l]], (fine.size, 1)), e[:, None], lo, hi)
    dens = np.exp(logp)
    prob = np.zeros(200)
    idx = np.minimum(((fine + 1) / 2 * 200).astype(int), 199)
    np.add.at(prob, idx, dens * (fine[1] - fine[0]))
    tv = 0.5 * np.abs(prob - emp).sum()
    assert tv < 0.01, tv


def test_tanh_gaussian_bwd_fd():
    rng = np.random.default_rng(10)
    out = rng.standard_normal((5, 6)) * 0.7
    eps = rng.standard_normal((5, 3))
    Ra = rng.standard_normal((5, 3))
    Rl = rng.standard_normal(5)

    def f():
        a, lp, _ = O.tanh_gaussian_fwd(out, eps, -5.0, 2.0)
        return float((a * Ra).sum() + (lp * Rl).sum())
    _, _, cache = O.tanh_gaussian_fwd(out, eps, -5.0, 2.0)
    fd_check(f, out, O.tanh_gaussian_bwd(Ra, Rl, cache))
