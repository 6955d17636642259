"""Data-parallel update on CPU: torch.distributed with the gloo backend,
world size 2.  Each rank runs the oracle's update pieces on its shard of the global batch with
the per-sample scale 1/B_global; the exchange follows libsquint's NCCL protocol (update_bf16.cu
/ api.cu): one SUM all-reduce of [critic grads | sum log pi | sum L_Q] before the critic Adam
and the alpha step, one of [actor grads | sum L_pi | sum Q] before the actor Adam; Adam, alpha
and Polyak then run replicated.  Checks: the ranks hold bit-identical state, and the state
equals the single-process oracle update on the rank-major concatenated batch (Q33).
Test infrastructure only (oracle on both sides of the comparison; no GPU)."""
import copy
import math
import os
import socket

import numpy as np
import pytest

import oracle as O
import squint_inputs as SI

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

WORLD = 2


def _flat(g, keys):
    return np.concatenate([np.asarray(g[k], np.float64).reshape(-1) for k in keys])


def _unflat(v, like, keys):
    out, o = {}, 0
    for k in keys:
        n = like[k].size
        out[k] = v[o:o + n].reshape(like[k].shape)
        o += n
    return out


def _adam_group(params, grads, m, v, t, lr, hp):
    for k in params:
        params[k], m[k], v[k] = O.adam_step(params[k], grads[k], m[k], v[k], t, lr, hp.beta1, hp.beta2, hp.adam_eps)


def _shard(n, rank, world):
    """libsquint's slice of a flat group for comm mode 1 (update_bf16.cu dp_adam): float4 units,
    [n4 * rank / G, n4 * (rank + 1) / G), the group size a multiple of 4 there; here the flat
    oracle group may have a ragged tail, which the last rank owns."""
    n4 = n // 4
    lo, hi = 4 * (n4 * rank // world), 4 * (n4 * (rank + 1) // world)
    return lo, (n if rank == world - 1 else hi)


def _sharded_adam_group(params, grads_local, m, v, t, lr, hp):
    """f1 (comm mode 1): this rank's slice of the SUM of every rank's gradient through Adam, the
    stepped slice written into every rank's parameters (here: a SUM all-reduce of a buffer that
    holds only this rank's slice, so each element comes from exactly one owner); m and v are
    touched on the slice only."""
    keys = sorted(params)
    world, rank = dist.get_world_size(), dist.get_rank()
    g = _allreduce(_flat(grads_local, keys))  # the peers' gradients, summed for the slice
    p, mf, vf = _flat(params, keys), _flat(m, keys), _flat(v, keys)
    lo, hi = _shard(p.size, rank, world)
    out = np.zeros_like(p)
    out[lo:hi], mf[lo:hi], vf[lo:hi] = O.adam_step(p[lo:hi], g[lo:hi], mf[lo:hi], vf[lo:hi], t, lr, hp.beta1,
                                                   hp.beta2, hp.adam_eps)
    p = _allreduce(out)
    for k, val in _unflat(p, params, keys).items():
        params[k] = val
    for k, val in _unflat(mf, m, keys).items():
        m[k] = val
    for k, val in _unflat(vf, v, keys).items():
        v[k] = val


def _allreduce(v):
    t = torch.from_numpy(np.ascontiguousarray(v))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.numpy()


def dp_update_one(d, hp, R, idx, shift, eps, st, b_global, sharded=False):
    """One update of this rank's shard (rows idx) with libsquint's DP exchange (sharded: comm
    mode 1, the row-sum tails summed in the barrier, Adam on this rank's slice)."""
    p = d.pad
    Ob = O.shift_images(R["obs"][idx], shift[:, 0], shift[:, 1], p)
    On = O.shift_images(R["next_obs"][idx], shift[:, 2], shift[:, 3], p)
    s, sn = R["proprio"][idx].astype(np.float64), R["next_proprio"][idx].astype(np.float64)
    a = R["action"][idx].astype(np.float64)
    r = R["reward"][idx].astype(np.float64)
    done = R["done"][idx]
    alpha0 = math.exp(st["log_alpha"])
    scale = 1.0 / b_global
    hn, _ = O.encoder_fwd(st["critic"], O.normalize_pixels(On))
    tgt = O.target_value if d.critic_kind == 1 else O.target_distribution  # f3 variants
    m, _ = tgt(d, hp, st["target"], st["actor"], hn, sn, r, done, eps[0], alpha0)
    LQ, gc, h = O.critic_loss_and_grads(d, hp, st["critic"], Ob, s, a, m, scale)
    # pre-step phi on sg(h): the current-state sample does not depend on the critic step (Q18)
    at, logp, caches = O.actor_forward(d, hp, st["actor"], h, s, eps[1])
    ck = sorted(gc)
    if sharded:
        sum_logp = _allreduce(np.array([logp.sum(), LQ]))[0]
        st["step"][0] += 1
        _sharded_adam_group(st["critic"], gc, st["m"]["critic"], st["v"]["critic"], st["step"][0], hp.lr_critic, hp)
    else:
        buf = _allreduce(np.concatenate([_flat(gc, ck), [logp.sum(), LQ]]))
        gc = _unflat(buf, gc, ck)
        sum_logp = buf[-2]
        st["step"][0] += 1
        _adam_group(st["critic"], gc, st["m"]["critic"], st["v"]["critic"], st["step"][0], hp.lr_critic, hp)
    La, ga = O.alpha_loss_and_grad(hp, st["log_alpha"], sum_logp / b_global)
    st["step"][2] += 1
    la, ma, va = O.adam_step(np.array([st["log_alpha"]]), np.array([ga]), np.array([st["m"]["alpha"]]),
                             np.array([st["v"]["alpha"]]), st["step"][2], hp.lr_alpha, hp.beta1, hp.beta2,
                             hp.adam_eps)
    st["log_alpha"], st["m"]["alpha"], st["v"]["alpha"] = float(la[0]), float(ma[0]), float(va[0])
    alpha1 = math.exp(st["log_alpha"])
    Lpi, gpi, qmean = O.actor_loss_and_grads(d, hp, st["critic"], st["actor"], h, s, at, logp, caches, alpha1, scale)
    ak = sorted(gpi)
    st["step"][1] += 1
    if sharded:
        _sharded_adam_group(st["actor"], gpi, st["m"]["actor"], st["v"]["actor"], st["step"][1], hp.lr_actor, hp)
    else:
        buf = _allreduce(np.concatenate([_flat(gpi, ak), [Lpi, qmean.sum()]]))
        gpi = _unflat(buf, gpi, ak)
        _adam_group(st["actor"], gpi, st["m"]["actor"], st["v"]["actor"], st["step"][1], hp.lr_actor, hp)
    for k in st["target"]:
        st["target"][k] = O.polyak(st["target"][k], st["critic"][k], hp.tau)
    return st


def _problem(b_local, utd, kind=0, mode=0):
    dims = SI.dims_of("c0", batch=b_local, critic_kind=kind)
    hp = SI.hp_of("c0", target_mode=mode)
    hp["target_entropy"] = -float(dims["action_dim"])
    d, h = O.Dims(**dims), O.HParams(**hp)
    specs = O.param_specs(d)
    R = SI.make_replay(200, dims, seed=0)
    vals = SI.make_params(specs, seed=1, perturb=True)
    m, v, steps = SI.make_adam_prewarm(specs, seed=4)
    st = O.init_state(specs, vals)
    for (grp, name), arr in m.items():
        if grp == "alpha":
            st["m"]["alpha"] = float(np.asarray(arr).reshape(-1)[0])
            st["v"]["alpha"] = float(np.asarray(v[(grp, name)]).reshape(-1)[0])
        else:
            st["m"][grp][name] = np.asarray(arr, np.float64).copy()
            st["v"][grp][name] = np.asarray(v[(grp, name)], np.float64).copy()
    st["step"] = list(steps)
    # per-rank seeded indices (data seed 2 + 1000 rank), shifts, noise
    idx = [SI.make_indices(utd, b_local, 200, seed=2 + 1000 * k) for k in range(WORLD)]
    sh = [SI.make_shifts(utd, b_local, dims["pad"], seed=2 + 1000 * k) for k in range(WORLD)]
    eps = [SI.make_eps(utd, b_local, dims["action_dim"], seed=3 + 1000 * k) for k in range(WORLD)]
    return d, h, dims, R, st, idx, sh, eps


def _state_vec(st):
    parts = []
    for g in ("critic", "actor", "target"):
        parts += [st[g][k].reshape(-1) for k in sorted(st[g])]
    for g in ("critic", "actor"):
        parts += [st["m"][g][k].reshape(-1) for k in sorted(st["m"][g])]
        parts += [st["v"][g][k].reshape(-1) for k in sorted(st["v"][g])]
    parts.append(np.array([st["log_alpha"], st["m"]["alpha"], st["v"]["alpha"]] + list(st["step"]), np.float64))
    return np.concatenate(parts)


def _worker(rank, port, b_local, utd, out_dir, kind=0, mode=0, sharded=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    d, h, dims, R, st, idx, sh, eps = _problem(b_local, utd, kind, mode)
    for j in range(utd):
        st = dp_update_one(d, h, R, idx[rank][j], sh[rank][j], eps[rank][j], st, b_local * WORLD, sharded)
    if sharded:
        # m, v: every rank holds only its own slice; assemble the owners' slices
        for g in ("critic", "actor"):
            keys = sorted(st["m"][g])
            for mv in ("m", "v"):
                f = _flat(st[mv][g], keys)
                lo, hi = _shard(f.size, rank, WORLD)
                own = np.zeros_like(f)
                own[lo:hi] = f[lo:hi]
                st[mv][g] = _unflat(_allreduce(own), st[mv][g], keys)
    np.save(os.path.join(out_dir, f"state{rank}.npy"), _state_vec(st))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("b_local,utd,kind,mode", [(3, 1, 0, 0), (4, 2, 0, 0), (3, 1, 0, 1), (3, 2, 1, 0), (3, 1, 1, 1)])
def test_dp_gloo_world2_matches_global_batch(tmp_path, b_local, utd, kind, mode):
    """kind 1: scalar MSE critic, mode 1: CDQ-min target (f3) -- the same exchange protocol."""
    mp.spawn(_worker, args=(_free_port(), b_local, utd, str(tmp_path), kind, mode), nprocs=WORLD, join=True)
    s0 = np.load(tmp_path / "state0.npy")
    s1 = np.load(tmp_path / "state1.npy")
    assert np.array_equal(s0, s1), "data-parallel replicas diverged"
    # single process, global batch = rank-major concatenation of the shards (Q33)
    d, h, dims, R, st, idx, sh, eps = _problem(b_local, utd, kind, mode)
    dg = O.Dims(**dict(dims, batch=b_local * WORLD))
    gidx = np.concatenate(idx, axis=1)
    gsh = np.concatenate(sh, axis=1)
    geps = np.concatenate(eps, axis=2)
    ref, _ = O.update(dg, h, R, gidx, gsh, geps, copy.deepcopy(st))
    r = _state_vec(ref)
    err = np.abs(s0 - r).max() / np.abs(r).max()
    assert err < 1e-10, err


@pytest.mark.parametrize("b_local,utd", [(3, 1), (4, 2)])
def test_dp_gloo_world2_sharded_adam_matches_global_batch(tmp_path, b_local, utd):
    """f1 (comm mode 1): all-reduce fused with a sharded Adam -- each rank steps only its slice of
    the summed gradient and writes it to every rank -- leaves the ranks' parameters bit-identical
    and equal (with the owners' m, v slices) to the single-process update on the global batch."""
    mp.spawn(_worker, args=(_free_port(), b_local, utd, str(tmp_path), 0, 0, True), nprocs=WORLD, join=True)
    s0 = np.load(tmp_path / "state0.npy")
    s1 = np.load(tmp_path / "state1.npy")
    assert np.array_equal(s0, s1), "sharded data-parallel replicas diverged"
    d, h, dims, R, st, idx, sh, eps = _problem(b_local, utd)
    dg = O.Dims(**dict(dims, batch=b_local * WORLD))
    ref, _ = O.update(dg, h, R, np.concatenate(idx, axis=1), np.concatenate(sh, axis=1),
                      np.concatenate(eps, axis=2), copy.deepcopy(st))
    r = _state_vec(ref)
    err = np.abs(s0 - r).max() / np.abs(r).max()
    assert err < 1e-10, err


def test_shard_ranges_tile_the_group():
    """The slices of comm mode 1 are disjoint, float4-aligned and cover the group for G = 1..8."""
    for n in (4, 8, 12, 4 * 37, 4 * 1000 + 4, 4 * 148 * 3):
        for world in range(1, 9):
            covered = np.zeros(n, np.int64)
            for rank in range(world):
                lo, hi = _shard(n, rank, world)
                assert lo % 4 == 0 and hi % 4 == 0 and lo <= hi
                covered[lo:hi] += 1
            assert (covered == 1).all(), (n, world)
