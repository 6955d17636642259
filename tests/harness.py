"""Shared test harness: feeds the same seeded inputs (squint_inputs) to the oracle and to
libsquint, and compares.  Test infrastructure only."""
from __future__ import annotations

import copy

import numpy as np

import oracle as O
import squint_inputs as SI


def compare(name, gpu, ref, tol):
    """Scale-relative max error (Q34): max|gpu - ref| <= tol * max|ref|.  Returns the ratio."""
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    assert gpu.shape == ref.shape, (name, gpu.shape, ref.shape)
    scale = max(np.abs(ref).max(), 1e-30)
    err = np.abs(gpu - ref).max()
    assert np.isfinite(gpu).all(), f"{name}: non-finite values"
    assert err <= tol * scale, f"{name}: max err {err:.3e} > {tol} * {scale:.3e} (rel {err / scale:.3e})"
    return err / scale


def oracle_state(specs, vals, m=None, v=None, steps=None):
    st = O.init_state(specs, vals)
    if m is not None:
        for (grp, name), arr in m.items():
            if grp == "alpha":
                st["m"]["alpha"] = float(np.asarray(arr).reshape(-1)[0])
                st["v"]["alpha"] = float(np.asarray(v[(grp, name)]).reshape(-1)[0])
            else:
                st["m"][grp][name] = np.asarray(arr, np.float64).copy()
                st["v"][grp][name] = np.asarray(v[(grp, name)], np.float64).copy()
        st["step"] = list(steps)
    return st


class Problem:
    """One seeded update problem: replay, params, Adam state, idx/shift/eps."""

    def __init__(self, cfg="c0", capacity=None, utd=1, seed=0, prewarm=True, perturb=True, hp_over=None, **dim_over):
        self.dims = SI.dims_of(cfg, **dim_over)
        self.hp = SI.hp_of(cfg, **(hp_over or {}))
        self.hp["target_entropy"] = -float(self.dims["action_dim"])
        self.d = O.Dims(**self.dims)
        self.h = O.HParams(**self.hp)
        self.specs = O.param_specs(self.d)
        cap = capacity or SI.CONFIGS[cfg].get("capacity", 1000)
        self.R = SI.make_replay(cap, self.dims, seed=seed)
        self.vals = SI.make_params(self.specs, seed=seed + 1, perturb=perturb)
        if prewarm:
            self.m, self.v, self.steps = SI.make_adam_prewarm(self.specs, seed=seed + 4)
        else:
            self.m = self.v = self.steps = None
        B = self.dims["batch"]
        self.utd = utd
        self.idx = SI.make_indices(utd, B, cap, seed=seed + 2)
        self.shifts = SI.make_shifts(utd, B, self.dims["pad"], seed=seed + 2)
        self.eps = SI.make_eps(utd, B, self.dims["action_dim"], seed=seed + 3)

    def oracle_update(self, trace=None):
        st = oracle_state(self.specs, self.vals, self.m, self.v, self.steps)
        return O.update(self.d, self.h, self.R, self.idx, self.shifts, self.eps, st, trace=trace)

    # ---- GPU side --------------------------------------------------------------------
    def gpu_setup(self, precision=0, device="cuda"):
        import torch

        import paper_2602_21203_b200 as P
        L = P.Learner(self.dims, self.hp, precision=precision, device=device, utd=self.utd)
        L.load_values(self.vals)
        if self.m is not None:
            L.load_adam(self.m, self.v, self.steps)
        dev = torch.device(device)
        self.Rt = {k: torch.as_tensor(np.ascontiguousarray(v)).to(dev) for k, v in self.R.items()
                   if isinstance(v, np.ndarray)}
        self.Rt["size"] = self.R["size"]
        self.replay = P.replay_from_tensors(self.Rt)
        self.idx_t = torch.as_tensor(self.idx).to(dev)
        self.sh_t = torch.as_tensor(self.shifts).to(dev)
        self.eps_t = torch.as_tensor(self.eps).to(dev)
        self.metrics_t = torch.zeros((self.utd, 8), dtype=torch.float32, device=dev)
        return L

    def gpu_update(self, L):
        import torch
        L.update(self.replay, self.idx_t, self.sh_t, self.eps_t, self.metrics_t)
        torch.cuda.synchronize()
        return self.metrics_t.cpu().numpy()


def group_values(L, group_name, which="param"):
    """Read every tensor of a group from the learner -> {name: np.ndarray}."""
    import paper_2602_21203_b200 as P
    gid = {"critic": P.squint.GROUP_CRITIC, "actor": P.squint.GROUP_ACTOR, "target": P.squint.GROUP_TARGET}[group_name]
    out = {}
    for g, n, off, shape in L.layout:
        if g != gid:
            continue
        numel = int(np.prod(shape))
        if which == "param":
            base = L.buffer(g)
        elif which == "grad":
            base = L.grad(g)
        else:
            base = getattr(L, f"{which}_{group_name}")
        out[n] = base[off:off + numel].detach().cpu().numpy().reshape(shape)
    return out
