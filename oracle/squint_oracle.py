"""Squint CPU oracle, float64 NumPy.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Citations: ``P:n`` = PAPER.md line n, ``S:n`` = SPEC.md line n, ``Qn`` = the reading
numbered n in SURVEY.md §8(c) / DESIGN.md §3.

Every function follows the paper's definition in its own order; library primitives used
as single steps are ``@`` (matmul), ``np.tanh``/``np.exp``/``np.log`` and ``np.rint``.
Nothing here is blocked, fused or reordered for speed.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "Dims", "HParams", "LOG_2PI", "param_specs", "area_downsample", "area_downsample_loops",
    "shift_images", "normalize_pixels", "conv2d_fwd", "conv2d_bwd", "conv2d_direct",
    "encoder_fwd", "encoder_bwd", "layernorm_fwd", "layernorm_bwd", "linear_fwd",
    "projection_fwd", "projection_bwd", "mlp_fwd", "mlp_bwd", "tanh_gaussian_fwd",
    "tanh_gaussian_bwd", "softmax", "log_softmax", "make_support", "categorical_project",
    "expected_value", "cross_entropy", "adam_step", "polyak", "target_distribution",
    "critic_loss_and_grads", "actor_forward", "alpha_loss_and_grad", "actor_loss_and_grads",
    "update", "act", "insert", "soft_update", "init_state", "target_probs", "target_value", "GREY_W", "grey_u8", "color_jitter",
    "insert_ex",
]

LOG_2PI = math.log(2.0 * math.pi)
SQUASH_EPS = 1e-6  # Q14 / S:199


@dataclass
class Dims:
    """Problem shape (SURVEY §8(b) squint_dims; BASELINE.json configs)."""
    img_c: int = 3
    img_h: int = 16
    img_w: int = 16
    pad: int = 2
    conv_ch: int = 32
    latent: int = 50
    proprio_dim: int = 12
    action_dim: int = 6
    critic_hidden: int = 256
    actor_hidden: int = 256
    n_atoms: int = 51
    v_min: float = -10.0
    v_max: float = 10.0
    batch: int = 32
    critic_kind: int = 0  # 0: distributional C51; 1: scalar MSE critic (Eqs. 1-2, Algorithm 1; f3)

    @property
    def head_out(self):  # critic head width: n_atoms logits, or one Q value
        return 1 if self.critic_kind == 1 else self.n_atoms

    @property
    def conv1_out(self):  # conv 3x3 stride 2 valid (Q7): 16 -> 7
        return (self.img_h - 3) // 2 + 1

    @property
    def conv2_out(self):  # conv 3x3 stride 1 valid (Q7): 7 -> 5
        return self.conv1_out - 2

    @property
    def flat(self):
        return self.conv_ch * self.conv2_out * self.conv2_out


@dataclass
class HParams:
    """Hyper-parameters (BASELINE.json configs[0]; Q15, Q26, Q28, Q13)."""
    gamma: float = 0.99
    tau: float = 0.005
    lr_critic: float = 3e-4
    lr_actor: float = 3e-4
    lr_alpha: float = 3e-4
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    target_entropy: float = -6.0
    target_mode: int = 0  # 0: average of the twin target heads (Q20); 1: CDQ-min (f3)
    ln_eps: float = 1e-5
    log_std_min: float = -5.0
    log_std_max: float = 2.0


# --------------------------------------------------------------------------------------
# Parameters.  Names are the ones the C-ABI layout reports; the tests check agreement.
# --------------------------------------------------------------------------------------
def _mlp_specs(prefix, n_in, hidden, n_out):
    return [
        (f"{prefix}.l1.w", (hidden, n_in), "w", n_in), (f"{prefix}.l1.b", (hidden,), "b", n_in),
        (f"{prefix}.ln1.g", (hidden,), "g", 0), (f"{prefix}.ln1.b", (hidden,), "beta", 0),
        (f"{prefix}.l2.w", (hidden, hidden), "w", hidden), (f"{prefix}.l2.b", (hidden,), "b", hidden),
        (f"{prefix}.ln2.g", (hidden,), "g", 0), (f"{prefix}.ln2.b", (hidden,), "beta", 0),
        (f"{prefix}.l3.w", (n_out, hidden), "w", hidden), (f"{prefix}.l3.b", (n_out,), "b", hidden),
    ]


def _proj_specs(prefix, flat, latent):
    return [
        (f"{prefix}.proj.w", (latent, flat), "w", flat), (f"{prefix}.proj.b", (latent,), "b", flat),
        (f"{prefix}.proj.ln.g", (latent,), "g", 0), (f"{prefix}.proj.ln.b", (latent,), "beta", 0),
    ]


def param_specs(d: Dims):
    """(group, name, shape, init kind, fan_in) for every parameter tensor.

    Groups: "critic" = encoder psi + critic projection + twin heads theta_1, theta_2
    (the encoder is trained only by the critic loss); "target" = EMA copy of
    the critic tensors except the encoder (Q28); "actor" = actor projection + MLP
    phi (Q8); "alpha" = log alpha (Q16).
    """
    C = d.conv_ch
    enc = [
        ("enc.conv1.w", (C, d.img_c, 3, 3), "w", d.img_c * 9), ("enc.conv1.b", (C,), "b", d.img_c * 9),
        ("enc.conv2.w", (C, C, 3, 3), "w", C * 9), ("enc.conv2.b", (C,), "b", C * 9),
    ]
    n_in_q = d.latent + d.proprio_dim + d.action_dim   # Q11
    n_in_pi = d.latent + d.proprio_dim                  # Q12
    critic_tail = (_proj_specs("critic", d.flat, d.latent)
                   + _mlp_specs("critic.q1", n_in_q, d.critic_hidden, d.head_out)
                   + _mlp_specs("critic.q2", n_in_q, d.critic_hidden, d.head_out))
    actor = (_proj_specs("actor", d.flat, d.latent)
             + _mlp_specs("actor", n_in_pi, d.actor_hidden, 2 * d.action_dim))
    out = [("critic",) + s for s in enc + critic_tail]
    out += [("target",) + s for s in critic_tail]
    out += [("actor",) + s for s in actor]
    out += [("alpha", "log_alpha", (1,), "zero", 0)]
    return out


# --------------------------------------------------------------------------------------
# a1: squint (area downsample); Q1 round-half-to-even.
# --------------------------------------------------------------------------------------
def area_downsample(frames: np.ndarray, factor: int) -> np.ndarray:
    """frames u8 [N, C, H, W] -> u8 [N, C, H/f, W/f]; q = round_half_even(block sum / f^2).

    S/f^2 is an exact float64 quotient whenever it is a tie (S, f^2 < 2^53), so ``np.rint``
    (IEEE round-half-to-even) gives the exact RHE of the exact block mean (Q1)."""
    n, c, h, w = frames.shape
    if h % factor or w % factor:
        raise ValueError("frame size not divisible by factor (S:41)")
    s = frames.astype(np.int64).reshape(n, c, h // factor, factor, w // factor, factor).sum(axis=(3, 5))
    return np.rint(s / float(factor * factor)).astype(np.uint8)


def area_downsample_loops(img: np.ndarray, factor: int) -> np.ndarray:
    """Nested-loop block mean on one [C, H, W] image, Python ints + Fraction-free RHE."""
    c, h, w = img.shape
    out = np.zeros((c, h // factor, w // factor), np.uint8)
    n = factor * factor
    for ch in range(c):
        for i in range(h // factor):
            for j in range(w // factor):
                s = 0
                for a in range(factor):
                    for b in range(factor):
                        s += int(img[ch, i * factor + a, j * factor + b])
                q, r = divmod(s, n)
                if 2 * r > n or (2 * r == n and q % 2 == 1):
                    q += 1
                out[ch, i, j] = q
    return out


def insert(frames, factor, slots, ring):
    """squint_insert: ring[slot[f]] = area_downsample(frames[f]) (Q4 distinct slots)."""
    ring = ring.copy()
    ring[np.asarray(slots)] = area_downsample(frames, factor)
    return ring


# --------------------------------------------------------------------------------------
# f4: renderer-side insert variants.  Colour jitter: P:267 names "lighting
# and color jitter alterations" and nothing more; S:55-63 fixes three factors (brightness,
# contrast, saturation) with a [1, 1] identity, clamping to [0, 255], and S:84 applies the
# jitter to the full-resolution frame before squinting.  The formulas and their order are
# reading R-jit: single-precision arithmetic with every product and sum
# rounded on its own and an 8-bit image after every step, because the integer pixel values
# the jitter produces are decided in the kernel's precision (the paper fixes none).
# --------------------------------------------------------------------------------------
GREY_W = (np.float32(0.2989), np.float32(0.587), np.float32(0.114))  # R-jit: Rec. 601 luma weights


def _u8(x):
    """u8(v) = truncate(clamp(v, 0, 255)) of a float32 array."""
    return np.clip(x, np.float32(0), np.float32(255)).astype(np.uint8)


def grey_u8(img):
    """grey(x) = u8((0.2989 R + 0.587 G) + 0.114 B) of a u8 [3, H, W] image, float32, left to right."""
    r, g, b = (img[k].astype(np.float32) for k in range(3))
    return _u8((GREY_W[0] * r + GREY_W[1] * g) + GREY_W[2] * b)


def color_jitter(frames, factors):
    """frames u8 [N, 3, H, W], factors float32 [N, 3] = (brightness b, contrast c, saturation s).

    Per frame, in this order (R-jit):
      x1 = u8(b x)
      m  = (sum over pixels of grey(x1)) / (H W)        (the integer sum is exact in float32)
      x2 = u8(c x1 + (1 - c) m)
      x3 = u8(s x2 + (1 - s) grey(x2))
    """
    frames = np.asarray(frames)
    factors = np.asarray(factors, np.float32)
    out = np.empty_like(frames)
    one = np.float32(1)
    for k in range(frames.shape[0]):
        b, c, s = factors[k]
        x1 = _u8(b * frames[k].astype(np.float32))
        m = np.float32(int(grey_u8(x1).astype(np.int64).sum())) / np.float32(x1.shape[1] * x1.shape[2])
        x2 = _u8(c * x1.astype(np.float32) + (one - c) * m)
        g2 = grey_u8(x2).astype(np.float32)
        out[k] = _u8(s * x2.astype(np.float32) + (one - s) * g2[None])
    return out


def insert_ex(frames, factor, slots, ring, hwc=False, jitter=None):
    """squint_insert_ex: HWC frames are read as their CHW transpose; the optional jitter
    runs on the full-resolution frame before the squint; then ``insert``."""
    x = np.ascontiguousarray(np.asarray(frames).transpose(0, 3, 1, 2)) if hwc else np.asarray(frames)
    if jitter is not None:
        x = color_jitter(x, jitter)
    return insert(x, factor, slots, ring)


def normalize_pixels(u8):
    """x = u / 255 (Q6)."""
    return u8.astype(np.float64) / 255.0


# --------------------------------------------------------------------------------------
# a4: random shift (DrQ lineage P:86; Q5): replicate pad p, crop at (dx, dy).
# --------------------------------------------------------------------------------------
def shift_images(imgs: np.ndarray, dx: np.ndarray, dy: np.ndarray, pad: int) -> np.ndarray:
    """out[b, c, y, x] = imgs[b, c, clamp(y + dy_b - p), clamp(x + dx_b - p)]  (u8, exact)."""
    b, c, h, w = imgs.shape
    out = np.empty_like(imgs)
    for k in range(b):
        ys = np.clip(np.arange(h) + int(dy[k]) - pad, 0, h - 1)
        xs = np.clip(np.arange(w) + int(dx[k]) - pad, 0, w - 1)
        out[k] = imgs[k][:, ys][:, :, xs]
    return out


# --------------------------------------------------------------------------------------
# a5: encoder f_psi (Q7): conv3x3 s2 -> ReLU -> conv3x3 s1 -> ReLU -> flatten
# --------------------------------------------------------------------------------------
def _im2col(x, k, stride):
    b, c, h, w = x.shape
    ho, wo = (h - k) // stride + 1, (w - k) // stride + 1
    cols = np.empty((b, ho, wo, c, k, k))
    for ki in range(k):
        for kj in range(k):
            cols[:, :, :, :, ki, kj] = x[:, :, ki:ki + stride * (ho - 1) + 1:stride,
                                         kj:kj + stride * (wo - 1) + 1:stride].transpose(0, 2, 3, 1)
    return cols.reshape(b, ho, wo, c * k * k)


def conv2d_fwd(x, w, bias, stride):
    """Valid cross-correlation via im2col + matmul; x [B,C,H,W], w [O,C,k,k] -> [B,O,Ho,Wo]."""
    o, c, k, _ = w.shape
    cols = _im2col(x, k, stride)
    y = cols @ w.reshape(o, -1).T + bias
    return y.transpose(0, 3, 1, 2), (x.shape, cols, w, stride)


def conv2d_bwd(dy, cache, need_dx=True):
    xshape, cols, w, stride = cache
    o, c, k, _ = w.shape
    dyc = dy.transpose(0, 2, 3, 1)                        # [B, Ho, Wo, O]
    dw = np.einsum("bijo,bijk->ok", dyc, cols).reshape(w.shape)
    db = dyc.sum(axis=(0, 1, 2))
    dx = None
    if need_dx:
        dcols = (dyc @ w.reshape(o, -1)).reshape(dyc.shape[:3] + (c, k, k))
        dx = np.zeros(xshape)
        ho, wo = dyc.shape[1], dyc.shape[2]
        for ki in range(k):
            for kj in range(k):
                dx[:, :, ki:ki + stride * (ho - 1) + 1:stride, kj:kj + stride * (wo - 1) + 1:stride] += \
                    dcols[:, :, :, :, ki, kj].transpose(0, 3, 1, 2)
    return dw, db, dx


def conv2d_direct(x, w, bias, stride):
    """Nested-loop definition of the same convolution (cross-check on tiny shapes)."""
    b, c, h, wd = x.shape
    o, _, k, _ = w.shape
    ho, wo = (h - k) // stride + 1, (wd - k) // stride + 1
    y = np.zeros((b, o, ho, wo))
    for n in range(b):
        for oc in range(o):
            for i in range(ho):
                for j in range(wo):
                    acc = bias[oc]
                    for ic in range(c):
                        for ki in range(k):
                            for kj in range(k):
                                acc += w[oc, ic, ki, kj] * x[n, ic, stride * i + ki, stride * j + kj]
                    y[n, oc, i, j] = acc
    return y


def encoder_fwd(p, x):
    """h = flatten(ReLU(conv2(ReLU(conv1(x))))) in (c, i, j) order; x already /255."""
    a1, c1 = conv2d_fwd(x, p["enc.conv1.w"], p["enc.conv1.b"], 2)
    y1 = np.maximum(a1, 0.0)
    a2, c2 = conv2d_fwd(y1, p["enc.conv2.w"], p["enc.conv2.b"], 1)
    y2 = np.maximum(a2, 0.0)
    return y2.reshape(y2.shape[0], -1), (c1, a1, c2, a2)


def encoder_bwd(dh, cache):
    """Gradients of psi from dL/dh (ReLU'(0) = 0, Q31).  No gradient w.r.t. the pixels."""
    c1, a1, c2, a2 = cache
    da2 = dh.reshape(a2.shape) * (a2 > 0)
    dw2, db2, dy1 = conv2d_bwd(da2, c2, need_dx=True)
    da1 = dy1 * (a1 > 0)
    dw1, db1, _ = conv2d_bwd(da1, c1, need_dx=False)
    return {"enc.conv1.w": dw1, "enc.conv1.b": db1, "enc.conv2.w": dw2, "enc.conv2.b": db2}


# --------------------------------------------------------------------------------------
# LayerNorm (Q9: biased variance, eps 1e-5, affine) and linear layers.
# --------------------------------------------------------------------------------------
def layernorm_fwd(x, g, b, eps):
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xh = (x - mu) * rstd
    return xh * g + b, (xh, rstd, g)


def layernorm_bwd(dy, cache):
    xh, rstd, g = cache
    dg = (dy * xh).sum(axis=0)
    db = dy.sum(axis=0)
    dxh = dy * g
    dx = rstd * (dxh - dxh.mean(axis=-1, keepdims=True) - xh * (dxh * xh).mean(axis=-1, keepdims=True))
    return dx, dg, db


def linear_fwd(x, w, b):
    """y = x W^T + b, W stored [out, in]."""
    return x @ w.T + b


def projection_fwd(p, prefix, h, eps):
    """z = tanh(LN(W h + b)): the one-layer projection of P:157 (Q8, Q9)."""
    a = linear_fwd(h, p[f"{prefix}.proj.w"], p[f"{prefix}.proj.b"])
    n, lnc = layernorm_fwd(a, p[f"{prefix}.proj.ln.g"], p[f"{prefix}.proj.ln.b"], eps)
    z = np.tanh(n)
    return z, (h, lnc, z)


def projection_bwd(dz, cache, prefix, p, need_dh):
    h, lnc, z = cache
    dn = dz * (1.0 - z * z)
    da, dg, dbeta = layernorm_bwd(dn, lnc)
    grads = {f"{prefix}.proj.w": da.T @ h, f"{prefix}.proj.b": da.sum(axis=0),
             f"{prefix}.proj.ln.g": dg, f"{prefix}.proj.ln.b": dbeta}
    dh = da @ p[f"{prefix}.proj.w"] if need_dh else None
    return grads, dh


def mlp_fwd(p, prefix, x0, eps):
    """Linear -> LN -> ReLU -> Linear -> LN -> ReLU -> Linear (Q9, Q10)."""
    a1 = linear_fwd(x0, p[f"{prefix}.l1.w"], p[f"{prefix}.l1.b"])
    n1, ln1 = layernorm_fwd(a1, p[f"{prefix}.ln1.g"], p[f"{prefix}.ln1.b"], eps)
    h1 = np.maximum(n1, 0.0)
    a2 = linear_fwd(h1, p[f"{prefix}.l2.w"], p[f"{prefix}.l2.b"])
    n2, ln2 = layernorm_fwd(a2, p[f"{prefix}.ln2.g"], p[f"{prefix}.ln2.b"], eps)
    h2 = np.maximum(n2, 0.0)
    out = linear_fwd(h2, p[f"{prefix}.l3.w"], p[f"{prefix}.l3.b"])
    return out, (x0, n1, ln1, h1, n2, ln2, h2)


def mlp_bwd(dout, cache, prefix, p):
    x0, n1, ln1, h1, n2, ln2, h2 = cache
    g = {f"{prefix}.l3.w": dout.T @ h2, f"{prefix}.l3.b": dout.sum(axis=0)}
    dh2 = dout @ p[f"{prefix}.l3.w"]
    da2, g[f"{prefix}.ln2.g"], g[f"{prefix}.ln2.b"] = layernorm_bwd(dh2 * (n2 > 0), ln2)
    g[f"{prefix}.l2.w"] = da2.T @ h1
    g[f"{prefix}.l2.b"] = da2.sum(axis=0)
    dh1 = da2 @ p[f"{prefix}.l2.w"]
    da1, g[f"{prefix}.ln1.g"], g[f"{prefix}.ln1.b"] = layernorm_bwd(dh1 * (n1 > 0), ln1)
    g[f"{prefix}.l1.w"] = da1.T @ x0
    g[f"{prefix}.l1.b"] = da1.sum(axis=0)
    dx0 = da1 @ p[f"{prefix}.l1.w"]
    return g, dx0


# --------------------------------------------------------------------------------------
# a7: tanh-Gaussian policy head (Q13, Q14).
# --------------------------------------------------------------------------------------
def tanh_gaussian_fwd(out, eps, lo, hi):
    """out = [mu | l] (A each); log sigma = lo + (hi-lo)/2 (tanh l + 1); u = mu + sigma eps;
    a = tanh u; log pi = sum_d [-eps^2/2 - log sigma - ln(2 pi)/2 - ln(1 - a^2 + 1e-6)]."""
    A = out.shape[1] // 2
    mu, l = out[:, :A], out[:, A:]
    tl = np.tanh(l)
    log_std = lo + 0.5 * (hi - lo) * (tl + 1.0)
    std = np.exp(log_std)
    u = mu + std * eps
    a = np.tanh(u)
    logp = (-0.5 * eps * eps - log_std - 0.5 * LOG_2PI - np.log(1.0 - a * a + SQUASH_EPS)).sum(axis=1)
    return a, logp, (eps, tl, std, a, lo, hi)


def tanh_gaussian_bwd(da, dlogp, cache):
    """Reparameterised gradient w.r.t. out = [mu | l] given dL/da [B,A] and dL/dlogpi [B]."""
    eps, tl, std, a, lo, hi = cache
    one_m_a2 = 1.0 - a * a
    dlp = dlogp[:, None]
    du = da * one_m_a2 + dlp * (2.0 * a * one_m_a2 / (one_m_a2 + SQUASH_EPS))
    dmu = du
    dlog_std = du * std * eps - dlp
    dl = dlog_std * 0.5 * (hi - lo) * (1.0 - tl * tl)
    return np.concatenate([dmu, dl], axis=1)


# --------------------------------------------------------------------------------------
# a9/a10: C51 machinery (Q20-Q24).
# --------------------------------------------------------------------------------------
def softmax(x):
    e = np.exp(x - x.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def log_softmax(x):
    m = x.max(axis=-1, keepdims=True)
    return x - m - np.log(np.exp(x - m).sum(axis=-1, keepdims=True))


def make_support(v_min, v_max, n_atoms):
    """z_j = v_min + j * dz, dz = (v_max - v_min)/(N - 1) (Q23)."""
    if not (v_min < v_max) or n_atoms < 2:
        raise ValueError("invalid support (S:272)")
    dz = (v_max - v_min) / (n_atoms - 1)
    return v_min + np.arange(n_atoms) * dz, dz


def categorical_project(p, r, not_done, gamma, shift, v_min, v_max):
    """Per-atom scatter (Q21, Q23): g_j = clip(r + nd*gamma*(z_j - shift)); b_j =
    clip((g_j - v_min)/dz, 0, N-1); mass to floor/ceil, all of it on an exact landing.

    p [B, N] probabilities, r [B], not_done [B], shift [B] (= alpha * log pi')."""
    B, N = p.shape
    z, dz = make_support(v_min, v_max, N)
    m = np.zeros((B, N))
    for b in range(B):
        for j in range(N):
            g = r[b] + not_done[b] * gamma * (z[j] - shift[b])
            g = min(max(g, v_min), v_max)
            bj = (g - v_min) / dz
            bj = min(max(bj, 0.0), N - 1.0)
            lo, hi = int(math.floor(bj)), int(math.ceil(bj))
            if lo == hi:
                m[b, lo] += p[b, j]
            else:
                m[b, lo] += p[b, j] * (hi - bj)
                m[b, hi] += p[b, j] * (bj - lo)
    return m


def expected_value(probs, z):
    return probs @ z


def cross_entropy(m, logits):
    """mean_b -sum_k m_bk log softmax(logits)_bk."""
    return float(-(m * log_softmax(logits)).sum(axis=1).mean())


# --------------------------------------------------------------------------------------
# a13/a14: Adam (Q26) and Polyak (Q28).
# --------------------------------------------------------------------------------------
def adam_step(p, g, m, v, t, lr, b1, b2, eps):
    """t is the step AFTER increment (1 on the first step)."""
    m = b1 * m + (1.0 - b1) * g
    v = b2 * v + (1.0 - b2) * g * g
    mhat = m / (1.0 - b1 ** t)
    vhat = v / (1.0 - b2 ** t)
    return p - lr * mhat / (np.sqrt(vhat) + eps), m, v


def polyak(target, online, tau):
    """theta_bar <- rho theta_bar + (1 - rho) theta, rho = 1 - tau (Algorithm 1 L24)."""
    return (1.0 - tau) * target + tau * online


def soft_update(target, online, tau):
    return polyak(np.asarray(target, np.float64), np.asarray(online, np.float64), tau)


# --------------------------------------------------------------------------------------
# One update (Algorithm 1 lines 9-24 with the distributional critic; Q17-Q30).
# --------------------------------------------------------------------------------------
def _head_input(*parts):
    return np.concatenate(parts, axis=1)


def target_probs(p1, p2, z, mode=0):
    """The twin target heads' distributions -> the one that is projected.

    mode 0 (the paper's choice, "the average rather than CDQ", Algorithm 1 line 13, Q20):
    pbar = (p1 + p2) / 2.  mode 1 (CDQ ablation, f3): per sample the head with the
    smaller expected value sum_k p_ik z_k (ties: head 1)."""
    if mode == 0:
        return 0.5 * (p1 + p2)
    q1, q2 = expected_value(p1, z), expected_value(p2, z)
    return np.where((q2 < q1)[:, None], p2, p1)


def target_distribution(d, hp, tgt, actor, hn, sn, r, done, eps_next, alpha0):
    """Lines 11-13: a' ~ pi(.|z', s'), pbar = mean_i softmax(head_bar_i) (or CDQ-min,
    ``hp.target_mode``), m = Proj(...)."""
    zpn, _ = projection_fwd(actor, "actor", hn, hp.ln_eps)
    out_n, _ = mlp_fwd(actor, "actor", _head_input(zpn, sn), hp.ln_eps)
    an, logpn, _ = tanh_gaussian_fwd(out_n, eps_next, hp.log_std_min, hp.log_std_max)
    zqn, _ = projection_fwd(tgt, "critic", hn, hp.ln_eps)
    x0 = _head_input(zqn, sn, an)
    z, _ = make_support(d.v_min, d.v_max, d.n_atoms)
    pbar = target_probs(softmax(mlp_fwd(tgt, "critic.q1", x0, hp.ln_eps)[0]),
                        softmax(mlp_fwd(tgt, "critic.q2", x0, hp.ln_eps)[0]), z, hp.target_mode)  # Q20
    not_done = 1.0 - done.astype(np.float64)                                          # Q22
    m = categorical_project(pbar, r, not_done, hp.gamma, alpha0 * logpn, d.v_min, d.v_max)  # Q21
    return m, logpn


def target_value(d, hp, tgt, actor, hn, sn, r, done, eps_next, alpha0):
    """f3 scalar critic, Algorithm 1 lines 11-13 as printed (Eq. 1):
    a' ~ pi(.|z', s'), y = r + (1-d) gamma/2 sum_i (Qbar_i(z', s', a') - alpha_0 log pi(a'|.))
    (the (1-d) mask is Q22).  CDQ (hp.target_mode 1; "elementwise min of expected
    values (scalar)"): y = r + (1-d) gamma (min_i Qbar_i - alpha_0 log pi)."""
    zpn, _ = projection_fwd(actor, "actor", hn, hp.ln_eps)
    out_n, _ = mlp_fwd(actor, "actor", _head_input(zpn, sn), hp.ln_eps)
    an, logpn, _ = tanh_gaussian_fwd(out_n, eps_next, hp.log_std_min, hp.log_std_max)
    zqn, _ = projection_fwd(tgt, "critic", hn, hp.ln_eps)
    x0 = _head_input(zqn, sn, an)
    q1 = mlp_fwd(tgt, "critic.q1", x0, hp.ln_eps)[0][:, 0]
    q2 = mlp_fwd(tgt, "critic.q2", x0, hp.ln_eps)[0][:, 0]
    not_done = 1.0 - done.astype(np.float64)
    if hp.target_mode == 0:
        y = r + not_done * hp.gamma / 2.0 * ((q1 - alpha0 * logpn) + (q2 - alpha0 * logpn))
    else:
        y = r + not_done * hp.gamma * (np.minimum(q1, q2) - alpha0 * logpn)
    return y, logpn


def critic_loss_and_grads(d, hp, critic, O, s, a, m, scale):
    """Line 15 (distributional, Q24): L_Q = sum_i mean_b CE(m, l_i); grads for psi, theta.
    Scalar critic (d.critic_kind 1, f3): L_Q = sum_i mean_b (Q_i - y)^2 with m = y [B].

    ``scale`` multiplies the per-sample gradient (1/B for the full batch; 1/B_global
    for a data-parallel shard, Q33).  Returns (loss computed with ``scale``, grads, h)."""
    h, enc_cache = encoder_fwd(critic, normalize_pixels(O))
    zq, pc = projection_fwd(critic, "critic", h, hp.ln_eps)
    x0 = _head_input(zq, s, a)
    grads = {}
    loss = 0.0
    dzq = np.zeros_like(zq)
    for i in (1, 2):
        logits, cache = mlp_fwd(critic, f"critic.q{i}", x0, hp.ln_eps)
        if d.critic_kind == 1:
            # f3 scalar critic, line 15 / Eq. 2: (Q_i - y)^2 per sample, m holds y [B]
            q = logits[:, 0]
            loss += float(((q - m) ** 2).sum() * scale)
            dlogits = (2.0 * (q - m) * scale)[:, None]
        else:
            loss += float(-(m * log_softmax(logits)).sum(axis=1).sum() * scale)
            dlogits = (softmax(logits) - m) * scale
        gi, dx0 = mlp_bwd(dlogits, cache, f"critic.q{i}", critic)
        grads.update(gi)
        dzq += dx0[:, :d.latent]
    gp, dh = projection_bwd(dzq, pc, "critic", critic, need_dh=True)
    grads.update(gp)
    grads.update(encoder_bwd(dh, enc_cache))
    return loss, grads, h


def actor_forward(d, hp, actor, h, s, eps_cur):
    """Line 21: a~ ~ pi(.|sg(z), s) with the pre-step phi (Q18, Q19)."""
    zp, pc = projection_fwd(actor, "actor", h, hp.ln_eps)
    out, mc = mlp_fwd(actor, "actor", _head_input(zp, s), hp.ln_eps)
    a, logp, tc = tanh_gaussian_fwd(out, eps_cur, hp.log_std_min, hp.log_std_max)
    return a, logp, (pc, mc, tc)


def alpha_loss_and_grad(hp, log_alpha, mean_logp):
    """Line 17 with the sign of Q17: L_a = -alpha (mean log pi + H_t); d/d log alpha."""
    alpha = math.exp(log_alpha)
    loss = -alpha * (mean_logp + hp.target_entropy)
    return loss, loss  # dL/dlog_alpha = -exp(log_alpha)(...) = L


def actor_loss_and_grads(d, hp, critic_new, actor, h, s, a, logp, caches, alpha1, scale):
    """Lines 19-22 (Q25): L_pi = mean_b [alpha+ log pi - (Q1+Q2)/2] on critic theta+."""
    zq, _ = projection_fwd(critic_new, "critic", h, hp.ln_eps)
    x0 = _head_input(zq, s, a)
    qs = []
    da = np.zeros_like(a)
    for i in (1, 2):
        logits, cache = mlp_fwd(critic_new, f"critic.q{i}", x0, hp.ln_eps)
        if d.critic_kind == 1:  # f3 scalar critic: the head's output is Q_i (line 22)
            q = logits[:, 0]
            dq = -0.5 * scale * np.ones_like(q)
            dlogits = dq[:, None]
        else:
            z, _ = make_support(d.v_min, d.v_max, d.n_atoms)
            pr = softmax(logits)
            q = expected_value(pr, z)
            dq = -0.5 * scale * np.ones_like(q)
            dlogits = pr * (z[None, :] - q[:, None]) * dq[:, None]   # softmax Jacobian times z
        qs.append(q)
        _, dx0 = mlp_bwd(dlogits, cache, f"critic.q{i}", critic_new)
        da += dx0[:, d.latent + d.proprio_dim:]
    qmean = 0.5 * (qs[0] + qs[1])
    loss = float(((alpha1 * logp - qmean) * scale).sum())
    pc, mc, tc = caches
    dout = tanh_gaussian_bwd(da, alpha1 * scale * np.ones_like(logp), tc)
    grads, dx0 = mlp_bwd(dout, mc, "actor", actor)
    gp, _ = projection_bwd(dx0[:, :d.latent], pc, "actor", actor, need_dh=False)
    grads.update(gp)
    return loss, grads, qmean


def _flat_norm(grads):
    return math.sqrt(sum(float((g * g).sum()) for g in grads.values()))


def init_state(specs, values):
    """Build an oracle state from {(group, name): array}."""
    st = {"critic": {}, "target": {}, "actor": {}, "log_alpha": 0.0,
          "m": {"critic": {}, "actor": {}, "alpha": 0.0}, "v": {"critic": {}, "actor": {}, "alpha": 0.0},
          "step": [0, 0, 0]}
    for grp, name, shape, *_ in specs:
        arr = np.asarray(values[(grp, name)], np.float64).reshape(shape)
        if grp == "alpha":
            st["log_alpha"] = float(arr.reshape(-1)[0])
        else:
            st[grp][name] = arr.copy()
    for g in ("critic", "actor"):
        for k, v in st[g].items():
            st["m"][g][k] = np.zeros_like(v)
            st["v"][g][k] = np.zeros_like(v)
    return st


def _adam_group(params, grads, m, v, t, lr, hp):
    for k in params:
        params[k], m[k], v[k] = adam_step(params[k], grads[k], m[k], v[k], t, lr, hp.beta1, hp.beta2, hp.adam_eps)


def update(d: Dims, hp: HParams, replay: dict, idx, shifts, eps, state, utd=None, trace=None):
    """``utd`` sequential updates (Q30).  idx [utd,B] i64, shifts [utd,B,4] u8 =
    (dx, dy) for obs then (dx', dy') for next_obs, eps [utd,2,B,A] (0 = next-state sample,
    1 = current-state sample).  Returns (new state, metrics [utd, 8]) with metrics =
    (L_Q, L_pi, L_alpha, alpha+, mean Q, entropy, |grad critic|, nonfinite).
    If ``trace`` is a list, per-update intermediates (grads, m, ...) are appended to it."""
    import copy
    st = copy.deepcopy(state)
    idx = np.asarray(idx)
    utd = idx.shape[0] if utd is None else utd
    metrics = np.zeros((utd, 8))
    for j in range(utd):
        metrics[j], tr = _update_one(d, hp, replay, idx[j], shifts[j], eps[j], st)
        if trace is not None:
            trace.append(tr)
    return st, metrics


def _update_one(d, hp, R, idx, shift, eps, st):
    B = idx.shape[0]
    p = d.pad
    O = shift_images(R["obs"][idx], shift[:, 0], shift[:, 1], p)
    On = shift_images(R["next_obs"][idx], shift[:, 2], shift[:, 3], p)
    s, sn = R["proprio"][idx].astype(np.float64), R["next_proprio"][idx].astype(np.float64)
    a = R["action"][idx].astype(np.float64)
    r = R["reward"][idx].astype(np.float64)
    done = R["done"][idx]
    alpha0 = math.exp(st["log_alpha"])
    scale = 1.0 / B

    # Line 10: both encodings with the current psi; h' carries no gradient.
    hn, _ = encoder_fwd(st["critic"], normalize_pixels(On))
    # Lines 11-13: target distribution (alpha_0, pre-step phi, theta_bar).
    if d.critic_kind == 1:  # f3 scalar critic: m carries the TD target y [B]
        m, logpn = target_value(d, hp, st["target"], st["actor"], hn, sn, r, done, eps[0], alpha0)
    else:
        m, logpn = target_distribution(d, hp, st["target"], st["actor"], hn, sn, r, done, eps[0], alpha0)
    # Lines 14-15: critic + encoder step.
    LQ, gc, h = critic_loss_and_grads(d, hp, st["critic"], O, s, a, m, scale)
    gnorm = _flat_norm(gc)
    st["step"][0] += 1
    _adam_group(st["critic"], gc, st["m"]["critic"], st["v"]["critic"], st["step"][0], hp.lr_critic, hp)
    # Lines 16-17: temperature step from the current-state sample (Q17, Q18).
    at, logp, caches = actor_forward(d, hp, st["actor"], h, s, eps[1])
    La, ga = alpha_loss_and_grad(hp, st["log_alpha"], float(logp.mean()))
    st["step"][2] += 1
    la, ma, va = adam_step(np.array([st["log_alpha"]]), np.array([ga]), np.array([st["m"]["alpha"]]),
                           np.array([st["v"]["alpha"]]), st["step"][2], hp.lr_alpha, hp.beta1, hp.beta2,
                           hp.adam_eps)
    st["log_alpha"], st["m"]["alpha"], st["v"]["alpha"] = float(la[0]), float(ma[0]), float(va[0])
    alpha1 = math.exp(st["log_alpha"])
    # Lines 18-22: actor step on sg(h) against theta+ (Q19, Q25).
    Lpi, gpi, qmean = actor_loss_and_grads(d, hp, st["critic"], st["actor"], h, s, at, logp, caches, alpha1, scale)
    st["step"][1] += 1
    _adam_group(st["actor"], gpi, st["m"]["actor"], st["v"]["actor"], st["step"][1], hp.lr_actor, hp)
    # Line 24: Polyak on every critic tensor except the encoder (Q28).
    for k in st["target"]:
        st["target"][k] = polyak(st["target"][k], st["critic"][k], hp.tau)
    vals = [LQ, Lpi, La]
    nonfinite = 0.0 if all(math.isfinite(x) for x in vals) else 1.0
    met = np.array([LQ, Lpi, La, alpha1, float(qmean.mean()), float(-logp.mean()), gnorm, nonfinite])
    trace = {"m": m, "logp_next": logpn, "grad_critic": gc, "grad_actor": gpi, "grad_log_alpha": ga,
             "h": h, "hn": hn, "logp": logp, "a_cur": at}
    return met, trace


# --------------------------------------------------------------------------------------
# a16: rollout act (Algorithm 1 lines 4-5): squint -> encoder -> actor -> sample.
# --------------------------------------------------------------------------------------
def act(d: Dims, hp: HParams, critic, actor, frames, proprio, eps=None):
    """frames u8 [n, 3, H, W] (H = W = 16 f).  eps None = mean action tanh(mu) with
    log pi evaluated at eps = 0 (reading R-act)."""
    f = frames.shape[2] // d.img_h
    small = area_downsample(frames, f) if f > 1 else frames
    h, _ = encoder_fwd(critic, normalize_pixels(small))
    zp, _ = projection_fwd(actor, "actor", h, hp.ln_eps)
    out, _ = mlp_fwd(actor, "actor", _head_input(zp, proprio.astype(np.float64)), hp.ln_eps)
    e = np.zeros((frames.shape[0], d.action_dim)) if eps is None else eps.astype(np.float64)
    a, logp, _ = tanh_gaussian_fwd(out, e, hp.log_std_min, hp.log_std_max)
    return a, logp, small
