"""Pins for the oracle's optimiser steps and the composed update: Adam / Polyak closed
forms, finite-difference gradients of L_Q, L_pi and L_alpha on tiny nets, stop-gradient
and gradient-partition invariants, the alpha fixed point and the data-parallel (Q33)
equivalence."""
import copy
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import squint_inputs as SI

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))

TINY = dict(img_c=3, img_h=16, img_w=16, pad=2, conv_ch=4, latent=8, proprio_dim=3, action_dim=2,
            critic_hidden=16, actor_hidden=16, n_atoms=7, v_min=-2.0, v_max=2.0, batch=3)


def tiny_setup(seed=0, perturb=True, **over):
    d = O.Dims(**dict(TINY, **over))
    hp = O.HParams(target_entropy=-float(d.action_dim))
    specs = O.param_specs(d)
    vals = SI.make_params(specs, seed=seed + 1, perturb=perturb)
    st = O.init_state(specs, vals)
    R = SI.make_replay(50, TINY if not over else dict(TINY, **over), seed=seed)
    return d, hp, specs, st, R


# ---- Adam / Polyak --------------------------------------------------------------------
def test_adam_first_step_closed_form():
    rng = np.random.default_rng(0)
    g = rng.standard_normal(100)
    p0 = rng.standard_normal(100)
    p1, m, v = O.adam_step(p0, g, np.zeros(100), np.zeros(100), 1, 3e-4, 0.9, 0.999, 1e-8)
    assert np.abs((p1 - p0) - (-3e-4 * g / (np.abs(g) + 1e-8))).max() < 1e-15


def test_adam_constant_gradient_k_steps():
    """Constant g: m_hat = g and v_hat = g^2 at every t, so k steps move -k lr g/(|g|+eps)."""
    g = np.array([0.3, -2.0, 1e-3])
    p = np.zeros(3)
    m = np.zeros(3)
    v = np.zeros(3)
    for t in range(1, 4):
        p, m, v = O.adam_step(p, g, m, v, t, 1e-2, 0.9, 0.999, 1e-8)
    assert np.abs(p - (-3 * 1e-2 * g / (np.abs(g) + 1e-8))).max() < 1e-14


def test_polyak_spec388():
    for c in GOLD["ema"]["cases"]:
        tau = 1.0 - c["rho"]
        assert O.polyak(np.array(c["target"]), np.array(c["online"]), tau) == c["expected"]


def test_polyak_k_step_closed_form():
    rng = np.random.default_rng(1)
    th, tb = rng.standard_normal(50), rng.standard_normal(50)
    tau, k = 0.005, 37
    x = tb.copy()
    for _ in range(k):
        x = O.polyak(x, th, tau)
    assert np.abs(x - (th + (1 - tau) ** k * (tb - th))).max() < 1e-13


# ---- finite differences through the composed losses -------------------------------
def _batch(d, R, seed=5):
    idx = SI.make_indices(1, d.batch, 50, seed=seed)[0]
    sh = SI.make_shifts(1, d.batch, d.pad, seed=seed)[0]
    eps = SI.make_eps(1, d.batch, d.action_dim, seed=seed)[0]
    O_ = O.shift_images(R["obs"][idx], sh[:, 0], sh[:, 1], d.pad)
    On = O.shift_images(R["next_obs"][idx], sh[:, 2], sh[:, 3], d.pad)
    f = lambda k: R[k][idx].astype(np.float64)
    return dict(O=O_, On=On, s=f("proprio"), sn=f("next_proprio"), a=f("action"), r=f("reward"),
                done=R["done"][idx], eps=eps.astype(np.float64))


def _fd(f, arr, an, n=6, h=1e-6, seed=0):
    rng = np.random.default_rng(seed)
    flat, a = arr.reshape(-1), an.reshape(-1)
    sc = max(np.abs(a).max(), 1e-10)
    for i in rng.choice(flat.size, min(n, flat.size), replace=False):
        old = flat[i]
        flat[i] = old + h
        fp = f()
        flat[i] = old - h
        fm = f()
        flat[i] = old
        assert abs((fp - fm) / (2 * h) - a[i]) <= 1e-5 * sc + 1e-9, (i, (fp - fm) / (2 * h), a[i])


def test_critic_loss_fd_all_tensors():
    d, hp, specs, st, R = tiny_setup()
    b = _batch(d, R)
    hn, _ = O.encoder_fwd(st["critic"], O.normalize_pixels(b["On"]))
    m, _ = O.target_distribution(d, hp, st["target"], st["actor"], hn, b["sn"], b["r"], b["done"], b["eps"][0], 0.7)
    crit = st["critic"]
    f = lambda: O.critic_loss_and_grads(d, hp, crit, b["O"], b["s"], b["a"], m, 1.0 / d.batch)[0]
    L, g, _ = O.critic_loss_and_grads(d, hp, crit, b["O"], b["s"], b["a"], m, 1.0 / d.batch)
    assert abs(L - sum(O.cross_entropy(m, O.mlp_fwd(crit, f"critic.q{i}", np.concatenate(
        [O.projection_fwd(crit, "critic", O.encoder_fwd(crit, O.normalize_pixels(b["O"]))[0], 1e-5)[0],
         b["s"], b["a"]], 1), 1e-5)[0]) for i in (1, 2))) < 1e-12
    assert set(g) == {n for grp, n, *_ in specs if grp == "critic"}
    for k in sorted(g):
        _fd(f, crit[k], g[k])


def test_critic_grad_zero_at_target_spec361():
    """If head 1's predicted distribution equals the target m, head 1 gets zero gradient
    while head 2 (different prediction) does not (S:361, S:222 head independence)."""
    d, hp, specs, st, R = tiny_setup(seed=11)
    b = _batch(d, R)
    crit = st["critic"]
    h, _ = O.encoder_fwd(crit, O.normalize_pixels(b["O"]))
    zq, _ = O.projection_fwd(crit, "critic", h, hp.ln_eps)
    l1, _ = O.mlp_fwd(crit, "critic.q1", np.concatenate([zq, b["s"], b["a"]], 1), hp.ln_eps)
    m = O.softmax(l1)
    _, g, _ = O.critic_loss_and_grads(d, hp, crit, b["O"], b["s"], b["a"], m, 1.0 / d.batch)
    for k in [n for n in g if n.startswith("critic.q1.")]:
        assert np.abs(g[k]).max() < 1e-15, k
    assert np.abs(g["critic.q2.l3.w"]).max() > 1e-6


def test_actor_loss_fd_and_stopgrad():
    d, hp, specs, st, R = tiny_setup(seed=2)
    b = _batch(d, R)
    h, _ = O.encoder_fwd(st["critic"], O.normalize_pixels(b["O"]))
    act = st["actor"]
    crit = st["critic"]

    def f():
        a, lp, c = O.actor_forward(d, hp, act, h, b["s"], b["eps"][1])
        return O.actor_loss_and_grads(d, hp, crit, act, h, b["s"], a, lp, c, 0.3, 1.0 / d.batch)[0]
    a, lp, c = O.actor_forward(d, hp, act, h, b["s"], b["eps"][1])
    L, g, q = O.actor_loss_and_grads(d, hp, crit, act, h, b["s"], a, lp, c, 0.3, 1.0 / d.batch)
    # gradient partition: only phi receives gradient from L_pi
    assert set(g) == {n for grp, n, *_ in specs if grp == "actor"}
    for k in sorted(g):
        _fd(f, act[k], g[k])


def test_alpha_grad_fd_fixed_point_direction_spec379():
    hp = O.HParams(target_entropy=-6.0)
    for la in (-1.0, 0.0, 0.4):
        for ml in (-8.0, 6.0, 2.5):
            L, g = O.alpha_loss_and_grad(hp, la, ml)
            h = 1e-6
            num = (O.alpha_loss_and_grad(hp, la + h, ml)[0] - O.alpha_loss_and_grad(hp, la - h, ml)[0]) / (2 * h)
            assert abs(num - g) < 1e-8
    # fixed point: entropy == target -> zero gradient
    assert O.alpha_loss_and_grad(hp, 0.2, 6.0)[1] == 0.0
    # entropy below target (mean log pi > -H_t... i.e. H = -mean log pi < H_t) -> alpha rises
    Hhat = -7.0  # below target -6
    g = O.alpha_loss_and_grad(hp, 0.0, -Hhat)[1]
    la, *_ = O.adam_step(np.array([0.0]), np.array([g]), np.zeros(1), np.zeros(1), 1, 1e-3, 0.9, 0.999, 1e-8)
    assert la[0] > 0.0
    Hhat = -5.0  # above target -> alpha falls
    g = O.alpha_loss_and_grad(hp, 0.0, -Hhat)[1]
    la, *_ = O.adam_step(np.array([0.0]), np.array([g]), np.zeros(1), np.zeros(1), 1, 1e-3, 0.9, 0.999, 1e-8)
    assert la[0] < 0.0


def _run_update(d, hp, st, R, utd=1, seed=5):
    idx = SI.make_indices(utd, d.batch, 50, seed=seed)
    sh = SI.make_shifts(utd, d.batch, d.pad, seed=seed)
    eps = SI.make_eps(utd, d.batch, d.action_dim, seed=seed)
    return O.update(d, hp, R, idx, sh, eps, st)


def test_update_gradient_partition_spec393():
    d, hp, specs, st, R = tiny_setup(seed=3)
    for zero in ("lr_critic", "lr_actor", "lr_alpha"):
        hp2 = copy.deepcopy(hp)
        setattr(hp2, zero, 0.0)
        st2, met = _run_update(d, hp2, st, R)
        grp = {"lr_critic": "critic", "lr_actor": "actor", "lr_alpha": "alpha"}[zero]
        if grp == "alpha":
            assert st2["log_alpha"] == st["log_alpha"]
        else:
            for k in st[grp]:
                assert np.array_equal(st2[grp][k], st[grp][k]), k
        assert np.isfinite(met).all()


def test_update_encoder_moves_spec362_and_target_polyak():
    d, hp, specs, st, R = tiny_setup(seed=4)
    st2, met = _run_update(d, hp, st, R)
    assert met[0, 0] > 0
    assert np.abs(st2["critic"]["enc.conv1.w"] - st["critic"]["enc.conv1.w"]).max() > 0
    for k in st["target"]:
        exp = (1 - hp.tau) * st["target"][k] + hp.tau * st2["critic"][k]
        assert np.abs(st2["target"][k] - exp).max() < 1e-15
    assert st2["step"] == [1, 1, 1]


def test_target_detach_spec394():
    """Perturbing the target nets changes L_Q but the critic gradient is taken with m
    fixed: d m / d theta_bar never enters (checked by FD with m recomputed vs frozen)."""
    d, hp, specs, st, R = tiny_setup(seed=6)
    b = _batch(d, R)
    hn, _ = O.encoder_fwd(st["critic"], O.normalize_pixels(b["On"]))
    m, _ = O.target_distribution(d, hp, st["target"], st["actor"], hn, b["sn"], b["r"], b["done"], b["eps"][0], 1.0)
    tgt2 = copy.deepcopy(st["target"])
    tgt2["critic.q1.l3.b"][3] += 0.5  # one atom (a uniform shift is softmax-invariant)
    m2, _ = O.target_distribution(d, hp, tgt2, st["actor"], hn, b["sn"], b["r"], b["done"], b["eps"][0], 1.0)
    L1 = O.critic_loss_and_grads(d, hp, st["critic"], b["O"], b["s"], b["a"], m, 1 / d.batch)[0]
    L2 = O.critic_loss_and_grads(d, hp, st["critic"], b["O"], b["s"], b["a"], m2, 1 / d.batch)[0]
    assert L1 != L2
    assert np.abs(m2.sum(1) - 1).max() < 1e-12


def test_dp_shard_equivalence_q33():
    """Sum over 2 shards of per-shard grads (scale 1/B_global) == full-batch grads."""
    d, hp, specs, st, R = tiny_setup(seed=7, batch=4)
    b = _batch(d, R)
    hn, _ = O.encoder_fwd(st["critic"], O.normalize_pixels(b["On"]))
    m, _ = O.target_distribution(d, hp, st["target"], st["actor"], hn, b["sn"], b["r"], b["done"], b["eps"][0], 1.0)
    Lf, gf, _ = O.critic_loss_and_grads(d, hp, st["critic"], b["O"], b["s"], b["a"], m, 1 / 4)
    tot = {k: 0.0 for k in gf}
    Ls = 0.0
    for sl in (slice(0, 2), slice(2, 4)):
        L, g, _ = O.critic_loss_and_grads(d, hp, st["critic"], b["O"][sl], b["s"][sl], b["a"][sl], m[sl], 1 / 4)
        Ls += L
        for k in g:
            tot[k] = tot[k] + g[k]
    assert abs(Ls - Lf) < 1e-12
    for k in gf:
        assert np.abs(tot[k] - gf[k]).max() < 1e-12


def test_update_utd_is_sequential_q30():
    d, hp, specs, st, R = tiny_setup(seed=8)
    idx = SI.make_indices(2, d.batch, 50, seed=9)
    sh = SI.make_shifts(2, d.batch, d.pad, seed=9)
    eps = SI.make_eps(2, d.batch, d.action_dim, seed=9)
    s2, m2 = O.update(d, hp, R, idx, sh, eps, st)
    sa, ma = O.update(d, hp, R, idx[:1], sh[:1], eps[:1], st)
    sb, mb = O.update(d, hp, R, idx[1:], sh[1:], eps[1:], sa)
    assert np.array_equal(m2, np.concatenate([ma, mb]))
    for k in s2["critic"]:
        assert np.array_equal(s2["critic"][k], sb["critic"][k])


def test_act_mean_action_and_sample():
    d, hp, specs, st, R = tiny_setup(seed=9)
    frames = SI.make_frames(3, 128, seed=1)
    prop = np.random.default_rng(0).standard_normal((3, d.proprio_dim))
    a0, lp0, small = O.act(d, hp, st["critic"], st["actor"], frames, prop)
    assert (small == O.area_downsample(frames, 8)).all()
    assert np.all(np.abs(a0) < 1)
    e = np.random.default_rng(1).standard_normal((3, d.action_dim))
    a1, lp1, _ = O.act(d, hp, st["critic"], st["actor"], frames, prop, e)
    assert not np.allclose(a0, a1)


# ---- f3: CDQ-min target ------------------------------------------------
def _cdq_target(d, st, b, mode, alpha0=0.7):
    hp = O.HParams(target_entropy=-float(d.action_dim), target_mode=mode)
    hn, _ = O.encoder_fwd(st["critic"], O.normalize_pixels(b["On"]))
    return O.target_distribution(d, hp, st["target"], st["actor"], hn, b["sn"], b["r"], b["done"], b["eps"][0],
                                 alpha0)


def test_cdq_identical_heads_equals_average_spec395():
    d, hp, specs, st, R = tiny_setup(seed=11)
    for k in list(st["target"]):
        if k.startswith("critic.q2"):
            st["target"][k] = st["target"][k.replace("critic.q2", "critic.q1")].copy()
    b = _batch(d, R)
    m0, _ = _cdq_target(d, st, b, 0)
    m1, _ = _cdq_target(d, st, b, 1)
    assert np.array_equal(m0, m1)


def test_cdq_target_mean_is_min_head_mean_spec395():
    """Wide support (no clipping): the projection keeps the mean, so the CDQ target's mean is
    r + (1-d) gamma min_i E_i (alpha = 0) and never exceeds the average target's mean."""
    d, hp, specs, st, R = tiny_setup(seed=12, v_min=-60.0, v_max=60.0)
    b = _batch(d, R)
    b["r"] = 0.5 * b["r"]  # r + gamma z_j stays inside [-60, 60]
    z, _ = O.make_support(d.v_min, d.v_max, d.n_atoms)
    m0, _ = _cdq_target(d, st, b, 0, alpha0=0.0)  # no entropy shift: no atom leaves the support
    m1, _ = _cdq_target(d, st, b, 1, alpha0=0.0)
    # the heads' own expectations, from a separate forward of the target nets
    hn, _ = O.encoder_fwd(st["critic"], O.normalize_pixels(b["On"]))
    zpn, _ = O.projection_fwd(st["actor"], "actor", hn, 1e-5)
    out_n, _ = O.mlp_fwd(st["actor"], "actor", np.concatenate([zpn, b["sn"]], 1), 1e-5)
    an, _, _ = O.tanh_gaussian_fwd(out_n, b["eps"][0], -5.0, 2.0)
    zq, _ = O.projection_fwd(st["target"], "critic", hn, 1e-5)
    x0 = np.concatenate([zq, b["sn"], an], 1)
    E = [O.softmax(O.mlp_fwd(st["target"], f"critic.q{i}", x0, 1e-5)[0]) @ z for i in (1, 2)]
    nd = 1.0 - b["done"].astype(np.float64)
    want = b["r"] + nd * 0.99 * np.minimum(E[0], E[1])
    assert np.abs(m1 @ z - want).max() < 1e-9
    assert (m1 @ z <= m0 @ z + 1e-12).all()
    assert (E[0] != E[1]).all()  # distinct heads: the selection is exercised


def test_cdq_picks_lower_mean_head_hand_case():
    z = np.linspace(-10, 10, 21)
    p1 = np.zeros((3, 21)); p2 = np.zeros((3, 21))
    p1[0, 15] = p2[0, 5] = 1.0      # head 2 lower
    p1[1, 4] = p2[1, 16] = 1.0      # head 1 lower
    p1[2, 10] = p2[2, 10] = 1.0     # tie -> head 1
    p2[2, 10] = 0.5; p2[2, 9] = 0.25; p2[2, 11] = 0.25  # same mean, different spread
    out = O.target_probs(p1, p2, z, 1)
    assert np.array_equal(out[0], p2[0]) and np.array_equal(out[1], p1[1]) and np.array_equal(out[2], p1[2])
    assert np.array_equal(O.target_probs(p1, p2, z, 0), 0.5 * (p1 + p2))


# ---- f3: scalar MSE critic (Eqs. 1-2, Algorithm 1 lines 13, 15, 22) ---------------------
def test_mse_critic_loss_fd_all_tensors():
    d, hp, specs, st, R = tiny_setup(seed=21, critic_kind=1)
    assert st["critic"]["critic.q1.l3.w"].shape == (1, d.critic_hidden)
    b = _batch(d, R)
    y = np.random.default_rng(0).standard_normal(d.batch)
    crit = st["critic"]
    f = lambda: O.critic_loss_and_grads(d, hp, crit, b["O"], b["s"], b["a"], y, 1.0 / d.batch)[0]
    L, g, _ = O.critic_loss_and_grads(d, hp, crit, b["O"], b["s"], b["a"], y, 1.0 / d.batch)
    assert set(g) == {n for grp, n, *_ in specs if grp == "critic"}
    for k in sorted(g):
        _fd(f, crit[k], g[k])


def test_mse_loss_and_zero_grad_at_target():
    """L = sum_i mean_b (Q_i - y)^2 (Eq. 2); with y = Q_1 head 1 gets no gradient, head 2 does."""
    d, hp, specs, st, R = tiny_setup(seed=22, critic_kind=1)
    b = _batch(d, R)
    crit = st["critic"]
    h, _ = O.encoder_fwd(crit, O.normalize_pixels(b["O"]))
    zq, _ = O.projection_fwd(crit, "critic", h, hp.ln_eps)
    x0 = np.concatenate([zq, b["s"], b["a"]], 1)
    q1 = O.mlp_fwd(crit, "critic.q1", x0, hp.ln_eps)[0][:, 0]
    q2 = O.mlp_fwd(crit, "critic.q2", x0, hp.ln_eps)[0][:, 0]
    y = q1.copy()
    L, g, _ = O.critic_loss_and_grads(d, hp, crit, b["O"], b["s"], b["a"], y, 1.0 / d.batch)
    assert abs(L - ((q2 - y) ** 2).mean()) < 1e-12
    for k in [n for n in g if n.startswith("critic.q1.")]:
        assert np.abs(g[k]).max() < 1e-15, k
    assert np.abs(g["critic.q2.l3.w"]).max() > 1e-6
    # d L / d b3 of head 2 = 2 mean(Q_2 - y) (the output bias enters Q_2 with slope 1)
    assert abs(g["critic.q2.l3.b"][0] - 2 * (q2 - y).mean()) < 1e-12


@pytest.mark.parametrize("mode", [0, 1])
def test_mse_target_constant_heads_closed_form(mode):
    """Target heads with zero output weights: Qbar_i = c_i, so y = r + (1-d) gamma (c - alpha
    log pi') with c = (c1 + c2)/2 (Algorithm 1 line 13) or min(c1, c2) (CDQ)."""
    d, hp, specs, st, R = tiny_setup(seed=23, critic_kind=1)
    hp = O.HParams(target_entropy=-float(d.action_dim), target_mode=mode)
    b = _batch(d, R)
    b["done"] = np.array([0, 1, 0], np.uint8)
    for i, c in ((1, 1.7), (2, -0.4)):
        st["target"][f"critic.q{i}.l3.w"][:] = 0.0
        st["target"][f"critic.q{i}.l3.b"][:] = c
    hn, _ = O.encoder_fwd(st["critic"], O.normalize_pixels(b["On"]))
    y, logpn = O.target_value(d, hp, st["target"], st["actor"], hn, b["sn"], b["r"], b["done"], b["eps"][0], 0.3)
    zpn, _ = O.projection_fwd(st["actor"], "actor", hn, hp.ln_eps)
    out, _ = O.mlp_fwd(st["actor"], "actor", np.concatenate([zpn, b["sn"]], 1), hp.ln_eps)
    _, lp, _ = O.tanh_gaussian_fwd(out, b["eps"][0], hp.log_std_min, hp.log_std_max)
    c = 0.65 if mode == 0 else -0.4
    want = b["r"] + np.array([1.0, 0.0, 1.0]) * hp.gamma * (c - 0.3 * lp)
    assert np.abs(y - want).max() < 1e-12
    assert y[1] == b["r"][1]


def test_mse_actor_loss_fd():
    d, hp, specs, st, R = tiny_setup(seed=24, critic_kind=1)
    b = _batch(d, R)
    h, _ = O.encoder_fwd(st["critic"], O.normalize_pixels(b["O"]))
    act, crit = st["actor"], st["critic"]

    def f():
        a, lp, c = O.actor_forward(d, hp, act, h, b["s"], b["eps"][1])
        return O.actor_loss_and_grads(d, hp, crit, act, h, b["s"], a, lp, c, 0.3, 1.0 / d.batch)[0]
    a, lp, c = O.actor_forward(d, hp, act, h, b["s"], b["eps"][1])
    L, g, q = O.actor_loss_and_grads(d, hp, crit, act, h, b["s"], a, lp, c, 0.3, 1.0 / d.batch)
    # L_pi = mean_b [alpha log pi - (Q1 + Q2)/2] with Q_i the heads' outputs (line 22)
    zq, _ = O.projection_fwd(crit, "critic", h, hp.ln_eps)
    x0 = np.concatenate([zq, b["s"], a], 1)
    qm = 0.5 * sum(O.mlp_fwd(crit, f"critic.q{i}", x0, hp.ln_eps)[0][:, 0] for i in (1, 2))
    assert abs(L - (0.3 * lp - qm).mean()) < 1e-12
    for k in sorted(g):
        _fd(f, act[k], g[k])
