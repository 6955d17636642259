"""Distribution of (bf16 error) / (emulation-floor error) per tensor over seeds and configs: the
scale-relative max (Q34) and the relative L2, for gradients and Adam steps."""
import os, sys, json
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
from harness import Problem, group_values
import paper_2602_21203_b200 as P
from test_gpu_parity import _proj_chw

def relmax(g, r):
    r = np.asarray(r, np.float64); return float(np.abs(np.asarray(g, np.float64) - r).max() / max(np.abs(r).max(), 1e-30))
def rel2(g, r):
    r = np.asarray(r, np.float64); return float(np.linalg.norm(np.asarray(g, np.float64) - r) / max(np.linalg.norm(r), 1e-30))

def errs(pr, L, tr, st_ref, bf):
    out = {}
    for grp in ("critic", "actor"):
        g = group_values(L, grp, "grad")
        if bf: g = _proj_chw(pr, g)
        got = group_values(L, grp)
        for n, r in tr["grad_" + grp].items():
            out[("g", n)] = (relmax(g[n], r), rel2(g[n], r))
            d_ref = st_ref[grp][n] - np.asarray(pr.vals[(grp, n)], np.float64)
            d = got[n] - pr.vals[(grp, n)]
            out[("d", n)] = (relmax(d, d_ref), rel2(d, d_ref))
    return out

cases = []
for seed in range(1, 7):
    cases.append(("c2", dict(capacity=4096, seed=seed, utd=1), None))
    cases.append(("c2", dict(capacity=4096, seed=seed + 10, utd=2), None))
for seed in range(1, 4):
    cases.append(("c2", dict(capacity=4096, seed=seed, batch=37, utd=1), None))
    cases.append(("c2", dict(capacity=4096, seed=seed, critic_kind=1, utd=2), None))
    cases.append(("c2", dict(capacity=4096, seed=seed, hp_over={"target_mode": 1}, utd=2), None))
    cases.append(("c3", dict(capacity=4096, seed=seed, batch=512, utd=1), None))
    cases.append(("c2", dict(capacity=2048, seed=seed + 20, utd=2), "reward_clip"))
    cases.append(("c2", dict(capacity=2048, seed=seed + 20, utd=2), "alpha_large"))
rmax, r2, fmax, f2 = [], [], [], []
worst = []
for cfg, kw, case in cases:
    pr = Problem(cfg, **kw)
    if case == "reward_clip":
        pr.R["reward"][:] = np.where(np.arange(pr.R["reward"].shape[0]) % 2 == 0, 60.0, -60.0).astype(np.float32)
    if case == "alpha_large":
        pr.vals[("alpha", "log_alpha")] = np.full_like(np.asarray(pr.vals[("alpha", "log_alpha")]), 3.0)
    tr = []; st_ref, _m = pr.oracle_update(tr)
    L = pr.gpu_setup(precision=P.BF16); pr.gpu_update(L); eb = errs(pr, L, tr[-1], st_ref, True)
    P.squint.LIB.squint_set_option(4, 15)
    L = pr.gpu_setup(precision=P.FP32); pr.gpu_update(L); ee = errs(pr, L, tr[-1], st_ref, False)
    P.squint.LIB.squint_set_option(4, 0)
    for k in eb:
        a, b = eb[k], ee[k]
        rmax.append(a[0] / max(b[0], 1e-30)); r2.append(a[1] / max(b[1], 1e-30))
        fmax.append(b[0]); f2.append(b[1])
        worst.append((a[0] / max(b[0], 1e-30), a[1] / max(b[1], 1e-30), a[0], b[0], a[1], b[1], cfg, str(kw) + str(case), k))
nfail = {f: sum(1 for w in worst if w[2] > max(2e-2, f * w[3])) for f in (1.2, 1.5, 2.0, 2.5)}
print("cases exceeding max(2e-2, f x floor) [max-element]:", nfail)
nfail2 = {f: sum(1 for w in worst if w[4] > max(2e-2, f * w[5])) for f in (1.1, 1.2, 1.3, 1.5)}
print("cases exceeding max(2e-2, f x floor) [rel L2]:", nfail2)
rmax, r2 = np.array(rmax), np.array(r2)
print("cases", len(cases), "tensors", len(rmax))
for nm, r in (("max", rmax), ("L2", r2)):
    print(nm, "ratio quantiles 50/90/99/100:", np.percentile(r, [50, 90, 99, 100]).round(3))
worst.sort(key=lambda x: -x[0])
for w in worst[:12]: print("max-ratio %.2f L2-ratio %.2f  bf16 %.2e floor %.2e | L2 %.2e floor %.2e  %s %s %s" % w)
worst.sort(key=lambda x: -x[1])
for w in worst[:8]: print("L2-ratio %.2f max-ratio %.2f bf16 %.2e floor %.2e | L2 %.2e floor %.2e  %s %s %s" % (w[1], w[0]) + tuple(w[2:]) if False else "L2-ratio %.2f max-ratio %.2f | L2 %.2e floor %.2e  %s %s %s" % (w[1], w[0], w[4], w[5], w[6], w[7], w[8]))
