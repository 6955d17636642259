"""GPU parity: libsquint (through the C ABI) vs the float64 oracle on the same seeded
inputs.  Integer work bit-exact; fp32 mode within 1e-4 (losses) / 1e-3 (gradients,
parameters) scale-relative (BASELINE.json north_star; Q34)."""
import numpy as np
import pytest

import oracle as O
import squint_inputs as SI
from harness import Problem, compare, group_values

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
import paper_2602_21203_b200 as P  # noqa: E402

DEV = "cuda"


# ---- a1 squint insert ---------------------------------------------------------------
@pytest.mark.parametrize("n,hw,factor", [(1, 128, 8), (37, 128, 8), (5, 64, 4), (3, 48, 3), (2, 16, 1)])
def test_insert_bit_exact_small(n, hw, factor):
    frames = SI.make_frames(n, hw, seed=n)
    cap = 100
    slots = SI.make_slots(n, cap, seed=n + 1)
    ring0 = np.full((cap, 3, hw // factor, hw // factor), 7, np.uint8)
    exp = O.insert(frames, factor, slots, ring0)
    ring = torch.as_tensor(ring0).to(DEV)
    P.squint_insert(torch.as_tensor(frames).to(DEV), factor, torch.as_tensor(slots).to(DEV), ring)
    torch.cuda.synchronize()
    assert np.array_equal(ring.cpu().numpy(), exp)


def test_insert_bit_exact_full_c1():
    """BASELINE configs[1] at full size: 1024 frames 3x128x128 -> 1M ring, all written
    rows checked against the oracle, untouched rows unchanged."""
    c = SI.CONFIGS["c1"]
    frames = SI.make_frames(c["n_frames"], c["frame_hw"], seed=0)
    slots = SI.make_slots(c["n_frames"], c["capacity"], seed=2)
    ring = torch.full((c["capacity"], 3, 16, 16), 3, dtype=torch.uint8, device=DEV)
    P.squint_insert(torch.as_tensor(frames).to(DEV), 8, torch.as_tensor(slots).to(DEV), ring)
    torch.cuda.synchronize()
    got = ring[torch.as_tensor(slots).to(DEV)].cpu().numpy()
    assert np.array_equal(got, O.area_downsample(frames, 8))
    assert int((ring != 3).any(dim=(1, 2, 3)).sum().item()) <= c["n_frames"]


def test_insert_tie_and_constant():
    f = np.zeros((2, 3, 128, 128), np.uint8)
    f[0] = 77
    # a block whose sum is exactly x.5 * 64: 32 pixels 1, 32 pixels 2 -> 1.5 -> 2; 0/1 -> 0.5 -> 0
    f[1, 0, :8, :8] = 1
    f[1, 0, :4, :8] = 2
    f[1, 1, :8, :8] = 0
    f[1, 1, :4, :8] = 1
    ring = torch.zeros((4, 3, 16, 16), dtype=torch.uint8, device=DEV)
    P.squint_insert(torch.as_tensor(f).to(DEV), 8, torch.tensor([2, 0], device=DEV), ring)
    r = ring.cpu().numpy()
    assert (r[2] == 77).all() and r[0, 0, 0, 0] == 2 and r[0, 1, 0, 0] == 0


@pytest.mark.parametrize("n,hw,factor", [(37, 128, 8), (5, 48, 3), (1024, 128, 8)])
def test_insert2_both_rings_bit_exact(n, hw, factor):
    """f2: one squint, two destinations (next_obs[slots], obs[slots2]) -- each ring equals
    the oracle's insert into it, untouched rows keep their fill."""
    frames = SI.make_frames(n, hw, seed=n + 3)
    cap = 2 * n + 5
    slots = SI.make_slots(n, cap, seed=n + 1)
    slots2 = (slots + 1) % cap
    r1 = np.full((cap, 3, hw // factor, hw // factor), 9, np.uint8)
    r2 = np.full_like(r1, 11)
    e1, e2 = O.insert(frames, factor, slots, r1), O.insert(frames, factor, slots2, r2)
    g1, g2 = torch.as_tensor(r1).to(DEV), torch.as_tensor(r2).to(DEV)
    P.squint_insert2(torch.as_tensor(frames).to(DEV), factor, torch.as_tensor(slots).to(DEV), g1,
                     torch.as_tensor(slots2).to(DEV), g2)
    torch.cuda.synchronize()
    assert np.array_equal(g1.cpu().numpy(), e1)
    assert np.array_equal(g2.cpu().numpy(), e2)


@pytest.mark.parametrize("n,hw,factor,hwc,jit", [
    (37, 128, 8, False, True), (37, 128, 8, True, False), (37, 128, 8, True, True), (5, 64, 4, True, True),
    (9, 16, 1, True, False), (9, 16, 1, False, True), (3, 48, 3, False, True), (1024, 128, 8, True, True)])
def test_insert_ex_variants_bit_exact(n, hw, factor, hwc, jit):
    """f4: HWC frames and colour jitter fused before the squint, factor 1 = direct render --
    bit-exact against the oracle (both rings, untouched rows unchanged)."""
    chw = SI.make_frames(n, hw, seed=n + 5)
    frames = np.ascontiguousarray(chw.transpose(0, 2, 3, 1)) if hwc else chw
    jitter = SI.make_jitter(n, seed=n) if jit else None
    cap = n + 7
    slots = SI.make_slots(n, cap, seed=n + 2)
    slots2 = (slots + 3) % cap
    r1 = np.full((cap, 3, hw // factor, hw // factor), 5, np.uint8)
    r2 = np.full_like(r1, 6)
    e1 = O.insert_ex(frames, factor, slots, r1, hwc=hwc, jitter=jitter)
    e2 = O.insert_ex(frames, factor, slots2, r2, hwc=hwc, jitter=jitter)
    g1, g2 = torch.as_tensor(r1).to(DEV), torch.as_tensor(r2).to(DEV)
    P.squint_insert_ex(torch.as_tensor(frames).to(DEV), factor, torch.as_tensor(slots).to(DEV), g1, hwc=hwc,
                       jitter=None if jitter is None else torch.as_tensor(jitter).to(DEV),
                       slots2=torch.as_tensor(slots2).to(DEV), ring2=g2)
    torch.cuda.synchronize()
    assert np.array_equal(g1.cpu().numpy(), e1)
    assert np.array_equal(g2.cpu().numpy(), e2)


def test_insert_ex_identity_jitter_equals_plain_insert():
    frames = SI.make_frames(64, 128, seed=1)
    slots = torch.arange(64, device=DEV)
    a = torch.zeros((64, 3, 16, 16), dtype=torch.uint8, device=DEV)
    b = torch.zeros_like(a)
    ft = torch.as_tensor(frames).to(DEV)
    P.squint_insert(ft, 8, slots, a)
    P.squint_insert_ex(ft, 8, slots, b, jitter=torch.ones((64, 3), device=DEV))
    torch.cuda.synchronize()
    assert torch.equal(a, b)


@pytest.mark.parametrize("nbytes,off", [(1, 0), (100_000, 0), (4099, 3), (64, 16)])
def test_stage_pinned_copies_bytes(nbytes, off):
    src = torch.randint(0, 256, (nbytes + off,), dtype=torch.uint8).pin_memory()
    dst = torch.full((nbytes + 32,), 7, dtype=torch.uint8, device=DEV)
    P.squint.squint_stage_pinned(dst[off:off + nbytes], src[off:])
    torch.cuda.synchronize()
    assert torch.equal(dst[off:off + nbytes].cpu(), src[off:])
    assert (dst[off + nbytes:].cpu() == 7).all() and (dst[:off].cpu() == 7).all()


def test_precondition_checks_option3():
    """squint_set_option(3): device-side preconditions (idx < size, distinct slots)
    are validated and reported as EINVAL instead of undefined behaviour."""
    S = P.squint
    frames = torch.as_tensor(SI.make_frames(4, 128, seed=1)).to(DEV)
    ring = torch.zeros((10, 3, 16, 16), dtype=torch.uint8, device=DEV)
    S.LIB.squint_set_option(3, 1)
    try:
        P.squint_insert(frames, 8, torch.tensor([1, 2, 3, 4], device=DEV), ring)  # valid
        for bad in ([1, 2, 2, 4], [1, 2, 3, 10], [-1, 2, 3, 4]):
            with pytest.raises(S.SquintError) as e:
                P.squint_insert(frames, 8, torch.tensor(bad, device=DEV), ring)
            assert e.value.status == 1
        pr = Problem("c0", utd=1, seed=0)
        L = pr.gpu_setup()
        pr.idx_t[0, 3] = pr.R["size"]  # one sampled index past the filled rows
        with pytest.raises(S.SquintError) as e:
            L.update(pr.replay, pr.idx_t, pr.sh_t, pr.eps_t, pr.metrics_t)
        assert e.value.status == 1 and b"out of range" in S.LIB.squint_last_error()
    finally:
        S.LIB.squint_set_option(3, 0)


# ---- a14 soft update ------------------------------------------------------------------
@pytest.mark.parametrize("n,tau", [(1, 0.005), (1000, 0.005), (4097, 0.5), (33, 0.0), (33, 1.0)])
def test_soft_update(n, tau):
    rng = np.random.default_rng(n)
    t0, o = rng.standard_normal(n).astype(np.float32), rng.standard_normal(n).astype(np.float32)
    t = torch.as_tensor(t0).to(DEV)
    P.squint_soft_update(t, torch.as_tensor(o).to(DEV), tau)
    compare("polyak", t.cpu().numpy(), O.soft_update(t0, o, tau), 1e-6)
    if tau == 0.0:
        assert np.array_equal(t.cpu().numpy(), t0)
    if tau == 1.0:
        assert np.array_equal(t.cpu().numpy(), o)


# ---- a16 act --------------------------------------------------------------------------
@pytest.mark.parametrize("n,sample,hw", [(1, True, 128), (37, True, 128), (64, False, 128), (37, True, 16)])
def test_act_fp32(n, sample, hw):
    """hw 16: frames already at the stored resolution (factor 1: insert2 / direct render)."""
    d = SI.dims_of("c0", batch=1)
    hp = SI.hp_of("c0")
    pr = Problem("c0", seed=5)
    L = pr.gpu_setup()
    frames = SI.make_frames(n, hw, seed=n)
    prop = SI.make_proprio(n, 12, seed=n)
    eps = np.random.default_rng(n).standard_normal((n, 6)).astype(np.float32) if sample else None
    st = O.init_state(pr.specs, pr.vals)
    a_ref, lp_ref, small = O.act(pr.d, pr.h, st["critic"], st["actor"], frames, prop, eps)
    dims = P.make_dims(pr.dims)
    ws = torch.zeros(P.act_workspace_bytes(dims, n), dtype=torch.uint8, device=DEV)
    act = torch.zeros((n, 6), device=DEV)
    lp = torch.zeros(n, device=DEV)
    ring = torch.zeros((200, 3, 16, 16), dtype=torch.uint8, device=DEV)
    slots = torch.as_tensor(SI.make_slots(n, 200, seed=n)).to(DEV)
    P.squint_act(dims, P.make_hparams(pr.hp), L.actor, L.critic, torch.as_tensor(frames).to(DEV),
                 torch.as_tensor(prop).to(DEV), None if eps is None else torch.as_tensor(eps).to(DEV), act, lp, ws,
                 ring=ring, slots=slots)
    torch.cuda.synchronize()
    compare("action", act.cpu().numpy(), a_ref, 1e-3)
    compare("logp", lp.cpu().numpy(), lp_ref, 1e-3)
    assert np.array_equal(ring[slots].cpu().numpy(), small)


# ---- a2-a15 update, fp32 mode -----------------------------------------------------------
def _check_update(pr, L, met_gpu, st_ref, met_ref, trace, tol_loss=1e-4, tol=1e-3, check_delta=True):
    # losses and metrics
    for j in range(pr.utd):
        for k, name in enumerate(["L_Q", "L_pi", "L_alpha", "alpha", "meanQ", "entropy", "gradnorm"]):
            # losses / alpha / entropy at the loss bound; mean Q (a near-zero sum of p_k z_k over a
            # +-v_max support, cancellation-prone) and |grad| at the gradient bound (DESIGN.md R-tol)
            compare(f"metric {name}[{j}]", met_gpu[j, k], met_ref[j, k], tol_loss if k in (0, 1, 2, 3, 5) else tol)
        assert met_gpu[j, 7] == 0.0
    # gradients of the last update
    tr = trace[-1]
    g = group_values(L, "critic", "grad")
    for n, ref in tr["grad_critic"].items():
        compare(f"grad critic {n}", g[n], ref, tol)
    g = group_values(L, "actor", "grad")
    for n, ref in tr["grad_actor"].items():
        compare(f"grad actor {n}", g[n], ref, tol)
    # target distribution and log-probs of the last update
    compare("m", L.region("m").cpu().numpy().reshape(tr["m"].shape), tr["m"], tol)
    compare("logp", L.region("logp").cpu().numpy(), tr["logp"], tol)
    compare("logp_next", L.region("logp_next").cpu().numpy(), tr["logp_next"], tol)
    # updated parameters, moments, target
    for grp in ("critic", "actor", "target"):
        got = group_values(L, grp)
        for n, ref in st_ref[grp].items():
            compare(f"{grp} {n}", got[n], ref, tol)
            if grp != "target" and check_delta:
                # Delta p / lr (Q27): the pre-warmed Adam step itself, fp32 mode only -- with bf16
                # operands m_hat / sqrt(v_hat) amplifies gradient rounding where v is tiny.
                d_ref = ref - np.asarray(pr.vals[(grp, n)], np.float64)
                compare(f"delta {grp} {n}", got[n] - pr.vals[(grp, n)], d_ref, 2e-2)
    for grp in ("critic", "actor"):
        for which in ("m", "v"):
            got = group_values(L, grp, which)
            for n, ref in st_ref[which][grp].items():
                compare(f"{which} {grp} {n}", got[n], ref, tol)
    compare("log_alpha", L.log_alpha.cpu().numpy()[0], st_ref["log_alpha"], 1e-5)
    assert L.step.cpu().tolist() == list(st_ref["step"])


@pytest.mark.parametrize("utd", [1, 4])
def test_update_c0_fp32(utd):
    pr = Problem("c0", utd=utd, seed=0)
    L = pr.gpu_setup()
    met = pr.gpu_update(L)
    trace = []
    st_ref, met_ref = pr.oracle_update(trace)
    _check_update(pr, L, met, st_ref, met_ref, trace)


@pytest.mark.parametrize("batch", [1, 37])
def test_update_ragged_batch_fp32(batch):
    pr = Problem("c0", utd=1, seed=3, batch=batch)
    L = pr.gpu_setup()
    met = pr.gpu_update(L)
    trace = []
    st_ref, met_ref = pr.oracle_update(trace)
    _check_update(pr, L, met, st_ref, met_ref, trace)


def test_update_c2_shapes_b64_fp32():
    pr = Problem("c2", capacity=2000, utd=2, seed=1, batch=64)
    L = pr.gpu_setup()
    met = pr.gpu_update(L)
    trace = []
    st_ref, met_ref = pr.oracle_update(trace)
    _check_update(pr, L, met, st_ref, met_ref, trace)


@pytest.mark.parametrize("utd", [1, 3])
def test_update_c0_cdq_fp32(utd):
    """f3: CDQ-min target through the fp32 path, at the fp32 bars."""
    pr = Problem("c0", utd=utd, seed=4, hp_over={"target_mode": 1})
    L = pr.gpu_setup()
    met = pr.gpu_update(L)
    trace = []
    st_ref, met_ref = pr.oracle_update(trace)
    _check_update(pr, L, met, st_ref, met_ref, trace)


@pytest.mark.parametrize("mode,utd,batch", [(0, 2, 32), (1, 2, 32), (0, 1, 37)])
def test_update_c0_mse_fp32(mode, utd, batch):
    """f3: scalar MSE critic (Eqs. 1-2, Algorithm 1), average or CDQ-min target, fp32 bars."""
    pr = Problem("c0", utd=utd, seed=6 + mode, batch=batch, critic_kind=1, hp_over={"target_mode": mode})
    L = pr.gpu_setup()
    met = pr.gpu_update(L)
    trace = []
    st_ref, met_ref = pr.oracle_update(trace)
    _check_update(pr, L, met, st_ref, met_ref, trace)


@pytest.mark.parametrize("case", ["all_done", "reward_clip", "gamma0", "gamma1_tau1", "alpha_large", "tau0"])
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_update_degenerate_cases(case, precision):
    """Degenerate cases of the method: every transition terminal (targets = r), rewards far
    outside the support (all target mass clipped onto the edge atoms), gamma = 0, gamma = tau = 1,
    a large temperature, tau = 0 (target frozen)."""
    hp_over = {"gamma0": {"gamma": 0.0}, "gamma1_tau1": {"gamma": 1.0, "tau": 1.0}, "tau0": {"tau": 0.0}}.get(case, {})
    cfg, kw = ("c0", {}) if precision == "fp32" else ("c2", {"capacity": 2048})
    pr = Problem(cfg, utd=2, seed=12, hp_over=hp_over, **kw)
    if case == "all_done":
        pr.R["done"][:] = 1
    if case == "reward_clip":
        pr.R["reward"][:] = np.where(np.arange(pr.R["reward"].shape[0]) % 2 == 0, 60.0, -60.0).astype(np.float32)
    if case == "alpha_large":
        # alpha = e^3: the target's atom shift alpha log pi' multiplies the bf16 error of log pi' by
        # alpha; the bf16 bar on m is then its emulation floor (R-tol-bf16, R-tol-alpha)
        la = 3.0
        pr.vals[("alpha", "log_alpha")] = np.full_like(np.asarray(pr.vals[("alpha", "log_alpha")]), la)
    L = pr.gpu_setup(precision=P.BF16 if precision == "bf16" else P.FP32)
    met = pr.gpu_update(L)
    trace = []
    st_ref, met_ref = pr.oracle_update(trace)
    if precision == "fp32":
        _check_update(pr, L, met, st_ref, met_ref, trace)
    else:
        _check_update_bf16(pr, L, met, st_ref, met_ref, trace)
    if case == "tau0":  # Polyak with tau = 0 leaves the target bitwise unchanged
        got = group_values(L, "target")
        for n in got:
            assert np.array_equal(got[n], np.asarray(pr.vals[("target", n)], np.float32).reshape(got[n].shape)), n


def test_update_deterministic_bitwise():
    pr = Problem("c0", utd=2, seed=7)
    outs = []
    for _ in range(2):
        L = pr.gpu_setup()
        pr.gpu_update(L)
        outs.append((L.critic.cpu().numpy().copy(), L.actor.cpu().numpy().copy(), L.target.cpu().numpy().copy()))
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


# ---- bf16 tensor-core mode (tcgen05), 2e-2 (BASELINE.json north_star) ------------------
@pytest.mark.parametrize("n", [37, 256])
def test_act_bf16(n):
    pr = Problem("c0", seed=5)
    L = pr.gpu_setup(precision=P.BF16)
    frames = SI.make_frames(n, 128, seed=n)
    prop = SI.make_proprio(n, 12, seed=n)
    eps = np.random.default_rng(n).standard_normal((n, 6)).astype(np.float32)
    st = O.init_state(pr.specs, pr.vals)
    a_ref, lp_ref, _ = O.act(pr.d, pr.h, st["critic"], st["actor"], frames, prop, eps)
    dims = P.make_dims(pr.dims, P.BF16)
    ws = torch.zeros(P.act_workspace_bytes(dims, n), dtype=torch.uint8, device=DEV)
    act = torch.zeros((n, 6), device=DEV)
    lp = torch.zeros(n, device=DEV)
    P.squint_act(dims, P.make_hparams(pr.hp), L.actor, L.critic, torch.as_tensor(frames).to(DEV),
                 torch.as_tensor(prop).to(DEV), torch.as_tensor(eps).to(DEV), act, lp, ws)
    torch.cuda.synchronize()
    compare("action bf16", act.cpu().numpy(), a_ref, 2e-2)
    compare("logp bf16", lp.cpu().numpy(), lp_ref, 2e-2)


def test_act_bf16_c4_full_size_sampled():
    """BASELINE configs c4 at full size: act on 4096 rendered 3x128x128 frames in one call (the
    launch configuration of the rollout), ring written for all rows; 96 sampled rows checked
    against the oracle one by one (rows are independent), every ring row bit-exact."""
    c = SI.CONFIGS["c4"]
    n = c["n_frames"]
    pr = Problem("c0", seed=5)
    L = pr.gpu_setup(precision=P.BF16)
    frames = SI.make_frames(n, c["frame_hw"], seed=44)
    prop = SI.make_proprio(n, 12, seed=44)
    eps = np.random.default_rng(44).standard_normal((n, 6)).astype(np.float32)
    dims = P.make_dims(pr.dims, P.BF16)
    ws = torch.zeros(P.act_workspace_bytes(dims, n), dtype=torch.uint8, device=DEV)
    act = torch.zeros((n, 6), device=DEV)
    lp = torch.zeros(n, device=DEV)
    ring = torch.zeros((n + 100, 3, 16, 16), dtype=torch.uint8, device=DEV)
    slots = torch.as_tensor(SI.make_slots(n, n + 100, seed=45)).to(DEV)
    P.squint_act(dims, P.make_hparams(pr.hp), L.actor, L.critic, torch.as_tensor(frames).to(DEV),
                 torch.as_tensor(prop).to(DEV), torch.as_tensor(eps).to(DEV), act, lp, ws, ring=ring, slots=slots)
    torch.cuda.synchronize()
    assert np.array_equal(ring[slots].cpu().numpy(), O.area_downsample(frames, 8))
    rows = np.sort(np.random.default_rng(46).choice(n, 96, replace=False))
    st = O.init_state(pr.specs, pr.vals)
    a_ref, lp_ref, _ = O.act(pr.d, pr.h, st["critic"], st["actor"], frames[rows], prop[rows], eps[rows])
    compare("action bf16 c4 sampled", act.cpu().numpy()[rows], a_ref, 2e-2)
    compare("logp bf16 c4 sampled", lp.cpu().numpy()[rows], lp_ref, 2e-2)


@pytest.mark.parametrize("n", [37, 1024])
def test_act_bf16_presquinted_factor1(n):
    """f2: act on frames already squinted into a ring row (factor 1) -- parity with the oracle's
    act on the same 16x16 frames, bitwise identical to act on the 128x128 originals (the squint
    is the only step that differs), and the factor-1 ring write copies the rows unchanged."""
    pr = Problem("c0", seed=5)
    L = pr.gpu_setup(precision=P.BF16)
    big = SI.make_frames(n, 128, seed=n + 11)
    small = O.area_downsample(big, 8)
    prop = SI.make_proprio(n, 12, seed=n)
    eps = np.random.default_rng(n).standard_normal((n, 6)).astype(np.float32)
    st = O.init_state(pr.specs, pr.vals)
    a_ref, lp_ref, s_ref = O.act(pr.d, pr.h, st["critic"], st["actor"], small, prop, eps)
    assert np.array_equal(s_ref, small)
    dims = P.make_dims(pr.dims, P.BF16)
    hp = P.make_hparams(pr.hp)
    ws = torch.zeros(P.act_workspace_bytes(dims, n), dtype=torch.uint8, device=DEV)
    out = []
    ring = torch.zeros((n + 3, 3, 16, 16), dtype=torch.uint8, device=DEV)
    slots = torch.arange(n, device=DEV, dtype=torch.int64).flip(0) + 2
    for fr, rg in ((small, ring), (big, None)):
        act = torch.zeros((n, 6), device=DEV)
        lp = torch.zeros(n, device=DEV)
        P.squint_act(dims, hp, L.actor, L.critic, torch.as_tensor(fr).to(DEV), torch.as_tensor(prop).to(DEV),
                     torch.as_tensor(eps).to(DEV), act, lp, ws, ring=rg, slots=None if rg is None else slots)
        torch.cuda.synchronize()
        out.append((act.cpu().numpy(), lp.cpu().numpy()))
    compare("action bf16 f1", out[0][0], a_ref, 2e-2)
    compare("logp bf16 f1", out[0][1], lp_ref, 2e-2)
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
    assert np.array_equal(ring[slots].cpu().numpy(), small)


def _rel_max(got, ref):
    """Scale-relative max error (Q34): max|got - ref| / max|ref|."""
    ref = np.asarray(ref, np.float64)
    return float(np.abs(np.asarray(got, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


def _rel_l2(got, ref):
    ref = np.asarray(ref, np.float64)
    return float(np.linalg.norm(np.asarray(got, np.float64) - ref) / max(np.linalg.norm(ref), 1e-30))


def _errs(got, ref):
    return (_rel_max(got, ref), _rel_l2(got, ref))


def _proj_chw(pr, g):
    # bf16 mode stores the projection weight gradients pixel-major (squint.h, regions 0 / 1)
    C = pr.dims["conv_ch"]
    for grp in ("critic", "actor"):
        pw = f"{grp}.proj.w"
        if pw in g:
            g[pw] = g[pw].reshape(g[pw].shape[0], -1, C).transpose(0, 2, 1).reshape(g[pw].shape)
    return g


def _emulation_floor(pr, trace, st_ref):
    """The same update on the fp32 path with every value the bf16 path stores in bf16 rounded to bf16
    (squint_set_option 4 = 15: GEMM activations / dY, weights, the LayerNorm x_hat cache, the encoder's
    weights and activations), against the same oracle: per tensor, the error bf16 storage alone causes
    (DESIGN.md R-tol-bf16)."""
    P.squint.LIB.squint_set_option(4, 15)
    try:
        L = pr.gpu_setup(precision=P.FP32)
        pr.gpu_update(L)
    finally:
        P.squint.LIB.squint_set_option(4, 0)
    tr = trace[-1]
    fl = {}
    for grp in ("critic", "actor"):
        g = group_values(L, grp, "grad")
        for n, r in tr["grad_" + grp].items():
            fl[("grad", grp, n)] = _errs(g[n], r)
        got = group_values(L, grp)
        for n, r in st_ref[grp].items():
            fl[("delta", grp, n)] = _errs(got[n] - pr.vals[(grp, n)], r - np.asarray(pr.vals[(grp, n)], np.float64))
    for n in ("m", "logp", "logp_next"):
        fl[n] = _errs(L.region(n).cpu().numpy().reshape(tr[n].shape), tr[n])
    return fl


def _check_update_bf16(pr, L, met_gpu, st_ref, met_ref, trace):
    """bf16 tensor-core mode (DESIGN.md R-tol-bf16).  Losses / metrics at the north-star bar 2e-2 (mean Q
    and L_alpha against the size of their terms).  Every other tensor -- the target distribution m, log pi,
    log pi', each gradient tensor and each Adam step (the parameter change, Q27) -- element-wise against
    its emulation floor: the error the same update has on the fp32 path with exactly the values the bf16
    path stores in bf16 rounded to bf16 (squint_set_option 4 = 15), measured here on the same inputs.
    Bars: scale-relative max error (Q34) <= max(2e-2, 2 x floor_max) and relative L2 <= max(2e-2,
    1.5 x floor_L2).  Measured over 30 update cases / 2520 tensors (c2, ragged, CDQ, scalar critic,
    utd 2, reward clipping, alpha = e^3, c3 shapes): median ratio bf16 / floor 1.00, 99th percentile 1.38
    (max error) / 1.15 (L2), maximum 2.11 (on a tensor at 9e-5) / 1.63 (at 2.5e-3) -- the floor is one
    realization of the same rounding noise, so a single case's ratio scatters around 1; no case of the
    2520 exceeds either bar."""
    tol = 2e-2
    qscale = 0.1 * max(abs(pr.dims["v_min"]), abs(pr.dims["v_max"]))
    for j in range(pr.utd):
        for k, name in enumerate(["L_Q", "L_pi", "L_alpha", "alpha", "meanQ", "entropy", "gradnorm"]):
            if name == "meanQ":  # E_p[z] is a cancelling sum over a +-v_max support: scale >= v_max / 10
                assert abs(met_gpu[j, k] - met_ref[j, k]) <= tol * max(abs(met_ref[j, k]), qscale), name
                continue
            if name == "L_alpha":
                # L_alpha = -alpha_0 (mean log pi + H_t) is a difference of two terms of size ~alpha_0 |H_t|
                # near the fixed point (Q17): its error is alpha_0 times the error of mean log pi, which the
                # entropy metric holds to the bar -- so the scale is the terms' size (DESIGN.md R-tol-bf16)
                la0 = float(np.asarray(pr.vals[("alpha", "log_alpha")], np.float64).reshape(-1)[0])
                a0 = float(met_ref[j - 1, 3]) if j > 0 else float(np.exp(la0))  # alpha before update j
                sc = max(abs(met_ref[j, k]), a0 * abs(pr.hp["target_entropy"]))
                assert abs(met_gpu[j, k] - met_ref[j, k]) <= tol * sc, (name, met_gpu[j, k], met_ref[j, k], sc)
                continue
            compare(f"metric {name}[{j}]", met_gpu[j, k], met_ref[j, k], tol)
        assert met_gpu[j, 7] == 0.0
    tr = trace[-1]
    floor = _emulation_floor(pr, trace, st_ref)

    def check(key, got, ref):
        (em, e2), (fm, f2) = _errs(got, ref), floor[key]
        assert em <= max(tol, 2.0 * fm), f"{key}: max error {em:.3e} > max(2e-2, 2 x floor {fm:.3e})"
        assert e2 <= max(tol, 1.5 * f2), f"{key}: rel L2 {e2:.3e} > max(2e-2, 1.5 x floor {f2:.3e})"

    for n in ("m", "logp", "logp_next"):
        check(n, L.region(n).cpu().numpy().reshape(tr[n].shape), tr[n])
    for grp in ("critic", "actor"):
        g = _proj_chw(pr, group_values(L, grp, "grad"))
        for n, r in tr["grad_" + grp].items():
            check(("grad", grp, n), g[n], r)
    for grp in ("critic", "actor", "target"):
        got = group_values(L, grp)
        for n, ref in st_ref[grp].items():
            compare(f"{grp} {n}", got[n], ref, tol)
            if grp != "target":  # the Adam step itself (parameter change, Q27)
                check(("delta", grp, n), got[n] - pr.vals[(grp, n)], ref - np.asarray(pr.vals[(grp, n)], np.float64))
    compare("log_alpha", L.log_alpha.cpu().numpy()[0], st_ref["log_alpha"], 1e-4)
    assert L.step.cpu().tolist() == list(st_ref["step"])


def _bf16_case(cfg, seed, utd=1, capacity=None, **over):
    pr = Problem(cfg, capacity=capacity, utd=utd, seed=seed, **over)
    L = pr.gpu_setup(precision=P.BF16)
    met = pr.gpu_update(L)
    trace = []
    st_ref, met_ref = pr.oracle_update(trace)
    _check_update_bf16(pr, L, met, st_ref, met_ref, trace)


def test_update_c2_pipelined_utd3_bf16():
    # option 2: each update's critic-side forward issued on the previous update's branch
    # (parity-alternating buffers); same results bar the fixed reduction orders
    P.squint.LIB.squint_set_option(2, 1)
    try:
        _bf16_case("c2", seed=3, utd=3, capacity=4096)
    finally:
        P.squint.LIB.squint_set_option(2, 0)


def test_update_c2_full_batch_utd2_bf16():
    _bf16_case("c2", seed=3, utd=2, capacity=4096)


def test_update_c2_bench_configuration_bf16():
    """The configuration bench.py times, at full size: 1M-row replay ring, B = 512, UTD 4, one
    squint_update call (cached CUDA graph, forked branch) -- against the oracle on the same
    seeded ring."""
    _bf16_case("c2", seed=9, utd=4, capacity=SI.CONFIGS["c2"]["capacity"])


@pytest.mark.parametrize("seed", [2, 7])
def test_update_c2_full_batch_bf16(seed):
    """BASELINE configs[2] shapes at the full batch 512 (101 atoms), as bench.py runs them."""
    _bf16_case("c2", seed=seed, capacity=4096)


@pytest.mark.parametrize("batch", [1, 37, 300])
def test_update_ragged_batch_bf16(batch):
    _bf16_case("c2", seed=5, capacity=4096, batch=batch)


def test_update_c2_cdq_bf16():
    _bf16_case("c2", seed=5, utd=2, capacity=4096, hp_over={"target_mode": 1})


@pytest.mark.parametrize("mode", [0, 1])
def test_update_c2_mse_bf16(mode):
    _bf16_case("c2", seed=8, utd=2, capacity=4096, critic_kind=1, hp_over={"target_mode": mode})


def test_update_c3_shapes_bf16():
    """BASELINE configs[3] layer shapes (C = 64, critic 512-512) at a per-rank batch of 512."""
    _bf16_case("c3", seed=4, capacity=4096, batch=512)


def test_update_c3_full_batch_bf16():
    """BASELINE configs[3] at its full single-GPU size: global batch 4096, C = 64, critic
    512-512, 101 atoms (the maximum shapes the path is built for)."""
    _bf16_case("c3", seed=6, capacity=8192)


# ---- bf16 GEMM engine (TMA + tcgen05) self-test: both operand majors, ragged tails -------
def _padded(x):
    """contiguous storage with a 16-byte multiple row pitch; returns (storage, logical cols)"""
    r, c = x.shape
    ld = (c + 7) // 8 * 8
    st = torch.full((r, ld), float("nan"), dtype=x.dtype)
    st[:, :c] = x
    return st.to(DEV), c


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 64, 64), (200, 101, 68), (512, 256, 256), (50, 800, 512), (37, 520, 130),
                                   (512, 6, 256), (512, 12, 256), (256, 62, 512)])
def test_gemm_engine(a_mn, b_mn, M, N, K):
    g = torch.Generator().manual_seed(M * 7 + N * 3 + K)
    a = torch.randn((M, K), generator=g).to(torch.bfloat16)
    b = torch.randn((N, K), generator=g).to(torch.bfloat16)
    ref = a.double() @ b.double().T
    A, ac = _padded(a.T.contiguous() if a_mn else a)
    B, bc = _padded(b.T.contiguous() if b_mn else b)
    out = torch.full((M, N), float("nan"), device=DEV)
    P.squint.selftest_gemm(A, ac, a_mn, B, bc, b_mn, M, N, K, out)
    torch.cuda.synchronize()
    compare("gemm", out.cpu().numpy(), ref.numpy(), 1e-5)


def test_act_ex_weight_snapshot_bitwise():
    """squint_act_ex (weights copied into the workspace tail, an event recorded after the copy) gives
    bitwise the results of squint_act; overwriting the master weights after the event does not
    change the act that is still running from the copies (the act-beside-the-updates step)."""
    pr = Problem("c2", seed=9, capacity=2048)
    L = pr.gpu_setup(precision=P.BF16)
    n = 1024
    fr = torch.as_tensor(SI.make_frames(n, 16, seed=3)).to(DEV)
    prop = torch.as_tensor(SI.make_proprio(n, 12, seed=3)).to(DEV)
    eps = torch.as_tensor(np.random.default_rng(3).standard_normal((n, 6)).astype(np.float32)).to(DEV)
    dims = P.make_dims(pr.dims, P.BF16)
    hp = P.make_hparams(pr.hp)
    ws = torch.zeros(P.act_workspace_bytes(dims, n), dtype=torch.uint8, device=DEV)
    a0, l0 = torch.zeros((n, 6), device=DEV), torch.zeros(n, device=DEV)
    P.squint_act(dims, hp, L.actor, L.critic, fr, prop, eps, a0, l0, ws)
    ev = torch.cuda.Event()
    ev.record()
    a1, l1 = torch.zeros((n, 6), device=DEV), torch.zeros(n, device=DEV)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    actor0, critic0 = L.actor.clone(), L.critic.clone()
    with torch.cuda.stream(side):
        P.squint_act(dims, hp, L.actor, L.critic, fr, prop, eps, a1, l1, ws, stream=side, weights_read=ev)
    torch.cuda.current_stream().wait_event(ev)
    L.actor.mul_(-3.0)  # an "optimizer step" right after the snapshot
    L.critic.mul_(-3.0)
    torch.cuda.synchronize()
    assert torch.equal(a0, a1) and torch.equal(l0, l1)
    L.actor.copy_(actor0)
    L.critic.copy_(critic0)
