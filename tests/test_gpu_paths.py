"""GPU tests of paths round 1 left unexercised (VERDICT r01 "Next round" item 2):

* the data-parallel branch of squint_update (a15 / SURVEY §8(e)) with a real NCCL communicator of
  one rank: no forked graph branch, row sums through k_row_sums, the reduced tails read by the
  alpha step and the metrics, ncclAllReduce on the flat gradient buffers -- against the oracle;
* the a3-a4 integer work (replay gather + random shift) bit-exact: the encoder's gathered,
  shifted u8 obs / next_obs images (workspace regions 8 / 9) memcmp'd against the oracle;
* exact atom placement through k_target_ce (BJ.ns "exact atom placement when r + gamma z lands on
  the grid"): a dyadic support and point-mass target heads, m bit-exact;
* DP semantics (Q33) on one GPU: a 1-rank communicator reproduces the single-GPU update.
"""
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
from test_gpu_parity import _check_update, _check_update_bf16  # noqa: E402

DEV = "cuda"


# ---- a15: the DP branch with a one-rank NCCL communicator ------------------------------------
@pytest.fixture(scope="module")
def comm1():
    h = P.squint.comm_init(P.squint.comm_unique_id(), 0, 1)
    yield h
    P.squint.comm_destroy(h)


@pytest.mark.parametrize("cfg,prec,over", [
    ("c0", "fp32", dict(utd=2)),
    ("c2", "bf16", dict(utd=2, capacity=4096)),
    ("c3", "bf16", dict(utd=1, capacity=4096, batch=512)),
    ("c3", "bf16", dict(utd=1, capacity=8192)),
])
def test_update_one_rank_comm(comm1, cfg, prec, over):
    """squint_update with comm != NULL (Q33 at G = 1: losses scaled by 1/B, SUM all-reduce over one
    rank) against the oracle at the mode's bars, and against the same call without a communicator."""
    over = dict(over)
    utd = over.pop("utd")
    pr = Problem(cfg, utd=utd, seed=21, **over)
    precision = P.BF16 if prec == "bf16" else P.FP32
    L = pr.gpu_setup(precision=precision)
    L.comm = comm1
    met = pr.gpu_update(L)
    trace = []
    st_ref, met_ref = pr.oracle_update(trace)
    (_check_update if prec == "fp32" else _check_update_bf16)(pr, L, met, st_ref, met_ref, trace)
    # the same update without a communicator: the DP branch computes the same sums in another
    # order (k_row_sums + all-reduce vs in-kernel sums), so parameters agree to fp32 rounding
    L2 = pr.gpu_setup(precision=precision)
    pr.gpu_update(L2)
    for grp in ("critic", "actor", "target"):
        a, b = group_values(L, grp), group_values(L2, grp)
        for n in a:
            compare(f"comm vs local {grp} {n}", a[n], b[n], 1e-4)


@pytest.fixture(scope="module")
def comm1_peer():
    h = P.squint.comm_init(P.squint.comm_unique_id(), 0, 1)
    P.squint.comm_set_mode(h, 1)
    yield h
    P.squint.comm_destroy(h)


@pytest.mark.parametrize("cfg,over,oracle", [
    ("c2", dict(utd=2, capacity=4096), True),
    ("c3", dict(utd=1, capacity=4096, batch=512), True),
    ("c2", dict(utd=3, capacity=4096, batch=37), False),
])
def test_update_one_rank_peer_mode(comm1, comm1_peer, cfg, over, oracle):
    """f1 (comm mode 1: peer-memory all-reduce fused with a sharded Adam) at G = 1: the slice is the
    whole group, the barrier passes on the rank's own counters, the tails are copied.  Bit for bit
    against mode 0 (ncclAllReduce + replicated Adam) on the same inputs -- same gradient sums, same
    Adam arithmetic, same per-block sum(g^2) partials -- over several updates (the barrier epochs
    advance in device memory), and against the oracle at the bf16 bars (the a15 cases of
    test_update_one_rank_comm)."""
    over = dict(over)
    utd = over.pop("utd")
    pr = Problem(cfg, utd=utd, seed=21, **over)
    L = pr.gpu_setup(precision=P.BF16)
    L.comm = comm1_peer
    met = pr.gpu_update(L)
    L0 = pr.gpu_setup(precision=P.BF16)
    L0.comm = comm1
    met0 = pr.gpu_update(L0)
    assert np.array_equal(np.asarray(met), np.asarray(met0)), "metrics differ between comm modes"
    for grp in ("critic", "actor", "target"):
        a, b = group_values(L, grp), group_values(L0, grp)
        for n in a:
            assert np.array_equal(a[n], b[n]), f"mode 1 vs mode 0: {grp} {n}"
    if oracle:
        trace = []
        st_ref, met_ref = pr.oracle_update(trace)
        _check_update_bf16(pr, L, met, st_ref, met_ref, trace)


# ---- a3-a4: gather + random shift, bit-exact ----------------------------------------------------
@pytest.mark.parametrize("cfg,utd,batch", [("c2", 2, 512), ("c2", 1, 37), ("c3", 1, 4096)])
def test_gather_shift_bit_exact_bf16(cfg, utd, batch):
    """The u8 images the tensor-core encoder stages (gather of rows idx from the ring, replicate pad
    2, crop at (dx, dy) / (dx', dy'), Q5) equal O.shift_images of the oracle rows, byte for byte."""
    pr = Problem(cfg, utd=utd, seed=13, capacity=100_000, batch=batch)
    L = pr.gpu_setup(precision=P.BF16)
    P.squint.LIB.squint_set_option(5, 1)
    try:
        pr.gpu_update(L)
    finally:
        P.squint.LIB.squint_set_option(5, 0)
    d = pr.dims
    B = d["batch"]
    shape = (B, d["img_c"], d["img_h"], d["img_w"])
    idx, sh = pr.idx[-1], pr.shifts[-1]
    exp_o = O.shift_images(pr.R["obs"][idx], sh[:, 0], sh[:, 1], d["pad"])
    exp_n = O.shift_images(pr.R["next_obs"][idx], sh[:, 2], sh[:, 3], d["pad"])
    got_o = L.region_u8("obs_shifted").cpu().numpy().reshape(shape)
    got_n = L.region_u8("next_obs_shifted").cpu().numpy().reshape(shape)
    assert np.array_equal(got_o, exp_o)
    assert np.array_equal(got_n, exp_n)


def test_gather_shift_bit_exact_fp32():
    pr = Problem("c0", utd=1, seed=14)
    L = pr.gpu_setup()
    pr.gpu_update(L)
    d = pr.dims
    shape = (d["batch"], d["img_c"], d["img_h"], d["img_w"])
    idx, sh = pr.idx[-1], pr.shifts[-1]
    exp_o = O.shift_images(pr.R["obs"][idx], sh[:, 0], sh[:, 1], d["pad"])
    assert np.array_equal(L.region_u8("obs_shifted").cpu().numpy().reshape(shape), exp_o)


# ---- a9: exact atom placement on a dyadic grid ------------------------------------------------
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_target_exact_landing_dyadic(precision):
    """Support [-16, 16] with 33 atoms (dz = 1), gamma = 0.5, r = 1, alpha = 0 (log alpha = -200
    underflows), target heads whose logits are their output bias (h2 = 0: ln2 affine zeroed) with a
    point mass at z = 4: g = 1 + 0.5 * 4 = 3 lands exactly on atom z = 3 (index 19), terminal rows
    on z = r = 1 (index 17).  m is one-hot, bit-exact, through k_target_ce (SURVEY §8(c) pin)."""
    cfg, kw = ("c0", {}) if precision == "fp32" else ("c2", {"capacity": 2048})
    pr = Problem(cfg, utd=1, seed=15, hp_over={"gamma": 0.5}, n_atoms=33, v_min=-16.0, v_max=16.0, **kw)
    for i in (1, 2):
        for t in ("ln2.g", "ln2.b"):
            pr.vals[("target", f"critic.q{i}.{t}")] = np.zeros_like(pr.vals[("target", f"critic.q{i}.{t}")])
        b3 = np.full(33, -1000.0, np.float32)
        b3[20] = 1000.0  # z_20 = 4
        pr.vals[("target", f"critic.q{i}.l3.b")] = b3
    pr.vals[("alpha", "log_alpha")] = np.full_like(np.asarray(pr.vals[("alpha", "log_alpha")]), -200.0)
    cap = pr.R["reward"].shape[0]
    pr.R["reward"][:] = 1.0
    pr.R["done"][:] = (np.arange(cap) % 3 == 0).astype(np.uint8)
    L = pr.gpu_setup(precision=P.BF16 if precision == "bf16" else P.FP32)
    pr.gpu_update(L)
    B = pr.dims["batch"]
    m = L.region("m").cpu().numpy().reshape(B, 33)
    done = pr.R["done"][pr.idx[0]]
    exp = np.zeros((B, 33), np.float32)
    exp[np.arange(B), np.where(done == 1, 17, 19)] = 1.0
    assert np.array_equal(m, exp)
    trace = []
    pr.oracle_update(trace)
    assert np.array_equal(trace[0]["m"], exp.astype(np.float64))


# ---- races: the forked graph branch (encoder backward beside the critic dW / actor pass) --------
@pytest.mark.parametrize("cfg,kw", [("c2", dict(capacity=4096)), ("c3", dict(capacity=4096, batch=512)),
                                    ("c3", dict(capacity=8192))])
def test_update_bf16_bitwise_reproducible(cfg, kw):
    """The bf16 update with its forked branch is bitwise reproducible over repeated calls (fixed-order
    reductions, no float atomics): a branch kernel reading a buffer the main stream rewrites (e.g. a
    weight shadow stepped by Adam) would show up here as run-to-run differences."""
    pr = Problem(cfg, utd=2, seed=6, **kw)
    ref = None
    for rep in range(6):
        L = pr.gpu_setup(precision=P.BF16)
        pr.gpu_update(L)
        out = {g: L.buffer(b).cpu().numpy().copy() for g, b in (("critic", P.squint.GROUP_CRITIC),
                                                                ("actor", P.squint.GROUP_ACTOR),
                                                                ("target", P.squint.GROUP_TARGET))}
        out["grad"] = L.grad(P.squint.GROUP_CRITIC).cpu().numpy().copy()
        if ref is None:
            ref = out
        else:
            for k in ref:
                assert np.array_equal(ref[k], out[k]), (k, rep)
