"""Per-tensor scale-relative max error (Q34) of the gradients: bf16 path vs fp32 path with bf16-rounded
GEMM operands (option 4 = 3), both against the oracle, c2 shapes B = 512."""
import os, sys, json
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
from harness import Problem, group_values
import paper_2602_21203_b200 as P

def errs(pr, L, tr):
    out = {}
    for grp in ("critic", "actor"):
        g = group_values(L, grp, "grad")
        if L.dims.precision == P.BF16:
            pw = f"{grp}.proj.w"; C = pr.dims["conv_ch"]
            g[pw] = g[pw].reshape(g[pw].shape[0], -1, C).transpose(0, 2, 1).reshape(g[pw].shape)
        for n, r in tr["grad_" + grp].items():
            out[f"g {n}"] = float(np.abs(g[n] - r).max() / max(np.abs(r).max(), 1e-30))
    for n in ("m", "logp", "logp_next"):
        got = L.region(n).cpu().numpy().reshape(tr[n].shape)
        out[n] = float(np.abs(got - tr[n]).max() / max(np.abs(tr[n]).max(), 1e-30))
    return out

res = {}
seeds = [int(x) for x in (sys.argv[1:] or ["2", "3", "7", "11"])]
for seed in seeds:
    pr = Problem("c2", capacity=4096, utd=1, seed=seed)
    tr = []
    pr.oracle_update(tr)
    row = {}
    L = pr.gpu_setup(precision=P.BF16); pr.gpu_update(L); row["bf16"] = errs(pr, L, tr[0])
    for em in (0, 3, 7, 15):
        P.squint.LIB.squint_set_option(4, em)
        L = pr.gpu_setup(precision=P.FP32); pr.gpu_update(L); row[f"emul{em}"] = errs(pr, L, tr[0])
    P.squint.LIB.squint_set_option(4, 0)
    res[seed] = row
names = list(res[seeds[0]]["bf16"].keys())
print(f"{'tensor':28s} " + " ".join(f"{k:>8s}" for k in ("bf16", "emul3", "emul7", "emul15", "fp32")) + "   (max over seeds)")
for n in names:
    vals = [max(res[s][k][n] for s in seeds) for k in ("bf16", "emul3", "emul7", "emul15", "emul0")]
    vals.append(vals[0] / max(vals[3], 1e-30))
    print(f"{n:28s} " + " ".join(f"{v:8.2e}" for v in vals[:5]) + f"  ratio {vals[5]:5.2f}")
json.dump(res, open("/root/repo/gpurun_out/bf16_err.json", "w"))
