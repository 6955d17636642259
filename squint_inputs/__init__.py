"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method: only problem sizes (BASELINE.json
configs[0..4]) and seeded random draws shaped like the paper's workloads (SURVEY.md
§8(d)).  Both ``oracle/`` and ``paper_2602_21203_b200/`` are fed from here;
neither imports the other, and this module imports neither.

Seeds: data 0, params 1, idx/shift 2 (+1000*rank), noise 3.
"""
from __future__ import annotations

import numpy as np

# ---- configs (BASELINE.json configs[0..4]) -------------------------------------------
_BASE_DIMS = dict(img_c=3, img_h=16, img_w=16, pad=2, conv_ch=32, latent=50, proprio_dim=12,
                  action_dim=6, critic_hidden=256, actor_hidden=256, n_atoms=51, v_min=-10.0,
                  v_max=10.0, batch=32)
_BASE_HP = dict(gamma=0.99, tau=0.005, lr_critic=3e-4, lr_actor=3e-4, lr_alpha=3e-4, beta1=0.9,
                beta2=0.999, adam_eps=1e-8, target_entropy=-6.0, ln_eps=1e-5, log_std_min=-5.0,
                log_std_max=2.0)

CONFIGS = {
    # c0: tiny single update, fp32, replay 1000, B 32, 51 atoms [-10, 10]
    "c0": dict(dims=dict(_BASE_DIMS), hp=dict(_BASE_HP), capacity=1000, utd=1, precision="fp32"),
    # c1: squint insert, 1024 frames 3x128x128 -> 1M ring
    "c1": dict(n_frames=1024, frame_hw=128, factor=8, capacity=1_000_000),
    # c2: standard update, 1M ring, B 512, UTD 4, 101 atoms [-20, 20], bf16 tensor cores
    "c2": dict(dims=dict(_BASE_DIMS, n_atoms=101, v_min=-20.0, v_max=20.0, batch=512), hp=dict(_BASE_HP),
               capacity=1_000_000, utd=4, precision="bf16"),
    # c3: large-batch DP, global B 4096, C 64, critic 512-512, 101 atoms
    "c3": dict(dims=dict(_BASE_DIMS, conv_ch=64, critic_hidden=512, n_atoms=101, v_min=-20.0, v_max=20.0,
                         batch=4096), hp=dict(_BASE_HP), capacity=1_000_000, utd=1, precision="bf16"),
    # c4: rollout act, 4096 envs, 3x128x128 frames
    "c4": dict(n_frames=4096, frame_hw=128, factor=8),
}


def dims_of(name, **over):
    d = dict(CONFIGS[name]["dims"])
    d.update(over)
    return d


def hp_of(name, **over):
    h = dict(CONFIGS[name]["hp"])
    h.update(over)
    return h


def _rng(seed, rank=0):
    return np.random.Generator(np.random.PCG64(seed + 1000 * rank))


# ---- replay ring contents ---------------------------------------------------------------
def make_replay(capacity, dims, seed=0, size=None):
    """SoA ring: obs/next_obs u8 [cap,3,16,16] uniform 0-255, proprio/next N(0,1) f32,
    action U[-1,1] f32, reward U[0,1] f32, done Bernoulli(0.01) u8 (BASELINE configs[0])."""
    g = _rng(seed)
    c, h, w = dims["img_c"], dims["img_h"], dims["img_w"]
    P, A = dims["proprio_dim"], dims["action_dim"]
    R = {
        "obs": g.integers(0, 256, (capacity, c, h, w), dtype=np.uint8),
        "next_obs": g.integers(0, 256, (capacity, c, h, w), dtype=np.uint8),
        "proprio": g.standard_normal((capacity, P), dtype=np.float32),
        "next_proprio": g.standard_normal((capacity, P), dtype=np.float32),
        "action": g.uniform(-1.0, 1.0, (capacity, A)).astype(np.float32),
        "reward": g.uniform(0.0, 1.0, capacity).astype(np.float32),
        "done": (g.uniform(0.0, 1.0, capacity) < 0.01).astype(np.uint8),
    }
    R["capacity"] = capacity
    R["size"] = capacity if size is None else size
    return R


def make_indices(utd, batch, size, seed=2, rank=0):
    """Uniform with replacement in [0, size)."""
    return _rng(seed, rank).integers(0, size, (utd, batch), dtype=np.int64)


def make_shifts(utd, batch, pad, seed=2, rank=0):
    """(dx, dy, dx', dy') per sample, each uniform in {0..2 pad} (Q5)."""
    return _rng(seed + 500, rank).integers(0, 2 * pad + 1, (utd, batch, 4), dtype=np.uint8)


def make_eps(utd, batch, action_dim, seed=3, rank=0):
    """N(0,1) noise [utd, 2, B, A]: [:,0] next-state sample, [:,1] current (Q32)."""
    return _rng(seed, rank).standard_normal((utd, 2, batch, action_dim), dtype=np.float32)


def make_params(specs, seed=1, perturb=False):
    """U(+-1/sqrt(fan_in)) weights and biases, LN (1, 0), log alpha 0, target = online.

    ``perturb`` (parity tests only): LN affine g = 1 + U(+-0.25), beta = U(+-0.25),
    target = online + U(+-0.02), log alpha = U(-1, 0) -- so that a swapped or skipped
    tensor cannot hide behind the symmetric defaults."""
    g = _rng(seed)
    vals = {}
    for grp, name, shape, kind, fan_in in specs:
        if grp == "target":
            continue
        if kind in ("w", "b"):
            bound = 1.0 / np.sqrt(fan_in)
            v = g.uniform(-bound, bound, shape)
        elif kind == "g":
            v = np.ones(shape) + (g.uniform(-0.25, 0.25, shape) if perturb else 0.0)
        elif kind == "beta":
            v = g.uniform(-0.25, 0.25, shape) if perturb else np.zeros(shape)
        elif kind == "zero":
            v = g.uniform(-1.0, 0.0, shape) if perturb else np.zeros(shape)
        else:
            raise ValueError(kind)
        vals[(grp, name)] = v.astype(np.float32)
    for grp, name, shape, kind, fan_in in specs:
        if grp == "target":
            v = vals[("critic", name)].astype(np.float64)
            if perturb:
                v = v + g.uniform(-0.02, 0.02, shape)
            vals[(grp, name)] = v.astype(np.float32)
    return vals


def specs_from_layout(layout):
    """(group, name, shape, kind, fan_in) from (group_name, name, shape) triples, by naming
    convention: *.w weights (fan_in = prod(shape[1:])), *.b biases of the matching *.w,
    *.ln*.g / *.ln*.b LayerNorm gain / bias, log_alpha."""
    shapes = {(g, n): s for g, n, s in layout}
    out = []
    for g, n, s in layout:
        if n == "log_alpha":
            out.append((g, n, s, "zero", 0))
        elif ".ln" in n and n.endswith(".g"):
            out.append((g, n, s, "g", 0))
        elif ".ln" in n and n.endswith(".b"):
            out.append((g, n, s, "beta", 0))
        elif n.endswith(".w"):
            out.append((g, n, s, "w", int(np.prod(s[1:]))))
        elif n.endswith(".b"):
            ws = shapes[(g, n[:-2] + ".w")]
            out.append((g, n, s, "b", int(np.prod(ws[1:]))))
        else:
            raise ValueError(n)
    return out


def make_adam_prewarm(specs, seed=4, step=10):
    """Pre-warmed Adam moments (Q27): m ~ N(0, 1e-3^2), v ~ U(1e-6, 1e-5), step 10."""
    g = _rng(seed)
    m, v = {}, {}
    for grp, name, shape, kind, fan_in in specs:
        if grp in ("critic", "actor", "alpha"):
            m[(grp, name)] = (1e-3 * g.standard_normal(shape)).astype(np.float32)
            v[(grp, name)] = g.uniform(1e-6, 1e-5, shape).astype(np.float32)
    return m, v, [step, step, step]


def make_frames(n, hw=128, seed=0, channels=3):
    """u8 [n, 3, hw, hw]: U{0..255} plus a smooth low-frequency field f (Q3):
    f = per-frame, per-channel bilinear upsample of a 9x9 grid of U[-64, 64]."""
    g = _rng(seed)
    base = g.integers(0, 256, (n, channels, hw, hw), dtype=np.int16)
    grid = g.uniform(-64.0, 64.0, (n, channels, 9, 9)).astype(np.float32)
    t = np.linspace(0.0, 8.0, hw, dtype=np.float32)
    i0 = np.minimum(t.astype(np.int64), 7)
    fr = t - i0
    rows = grid[:, :, i0, :] * (1 - fr)[None, None, :, None] + grid[:, :, i0 + 1, :] * fr[None, None, :, None]
    field = rows[:, :, :, i0] * (1 - fr) + rows[:, :, :, i0 + 1] * fr
    return np.ascontiguousarray(np.clip(base + np.rint(field).astype(np.int16), 0, 255).astype(np.uint8))


def make_jitter(n, seed=5, lo=0.6, hi=1.4):
    """f32 [n, 3] colour-jitter factors (brightness, contrast, saturation), each U[lo, hi]
    (S:31-34 intervals; the paper gives no ranges -- reading R-jit)."""
    return _rng(seed + 11).uniform(lo, hi, (n, 3)).astype(np.float32)


def make_slots(n, capacity, seed=2):
    """Distinct write slots (Q4)."""
    return _rng(seed).choice(capacity, n, replace=False).astype(np.int64)


def make_proprio(n, dim=12, seed=3):
    return _rng(seed + 7).standard_normal((n, dim), dtype=np.float32)
