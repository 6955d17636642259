"""Workloads for ncu captures (one kernel family each, a few warm-up calls first):
  python tools/ncu_work.py c1   squint_insert of 1024 frames into the 1M ring        (k_insert_f8)
  python tools/ncu_work.py c4   squint_act on 4096 rendered frames (fused squint)    (k_enc_fwd_tc, k_chain, ...)
  python tools/ncu_work.py c3   one c3 update on one GPU (B 4096, C 64, 512-512)     (k_enc_fwd_ws, k_enc_bwd_tc, ...)
  python tools/ncu_work.py c2   one c2 update (B 512)                                (k_gemm<bwd_ln_relu>, k_chain, ...)
Launches go straight to the stream (SQUINT_NO_GRAPH=1) so ncu sees every kernel."""
import os
import sys

os.environ.setdefault("SQUINT_NO_GRAPH", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2602_21203_b200 as P  # noqa: E402
import squint_inputs as SI  # noqa: E402
from paper_2602_21203_b200 import squint as S  # noqa: E402

which = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(1)


def learner(cfg):
    d, hp = SI.dims_of(cfg), SI.hp_of(cfg)
    L = P.Learner(d, hp, precision=P.BF16, device=dev, utd=1)
    L.load_values(SI.make_params(SI.specs_from_layout([(S.GROUP_NAMES[k], n, s) for k, n, o, s in L.layout]), seed=1))
    return d, L


if which == "c1":
    fr = torch.randint(0, 256, (1024, 3, 128, 128), generator=g, device=dev, dtype=torch.uint8)
    ring = torch.zeros((1_000_000, 3, 16, 16), dtype=torch.uint8, device=dev)
    sl = torch.randperm(1_000_000, generator=g, device=dev)[:1024].contiguous()
    for _ in range(reps):
        P.squint_insert(fr, 8, sl, ring)
elif which == "c4":
    d, L = learner("c2")
    n = 4096
    fr = torch.randint(0, 256, (n, 3, 128, 128), generator=g, device=dev, dtype=torch.uint8)
    prop = torch.randn((n, 12), generator=g, device=dev)
    eps = torch.randn((n, 6), generator=g, device=dev)
    act, lp = torch.zeros((n, 6), device=dev), torch.zeros((n,), device=dev)
    ws = torch.zeros(P.act_workspace_bytes(L.dims, n), dtype=torch.uint8, device=dev)
    for _ in range(reps):
        P.squint_act(L.dims, L.hp, L.actor, L.critic, fr, prop, eps, act, lp, ws)
else:
    d, L = learner(which)
    cap = 1_000_000
    A, B = d["action_dim"], d["batch"]
    R = {"obs": torch.randint(0, 256, (cap, 3, 16, 16), generator=g, device=dev, dtype=torch.uint8),
         "next_obs": torch.randint(0, 256, (cap, 3, 16, 16), generator=g, device=dev, dtype=torch.uint8),
         "proprio": torch.randn((cap, 12), generator=g, device=dev),
         "next_proprio": torch.randn((cap, 12), generator=g, device=dev),
         "action": torch.rand((cap, A), generator=g, device=dev) * 2 - 1,
         "reward": torch.rand((cap,), generator=g, device=dev),
         "done": (torch.rand((cap,), generator=g, device=dev) < 0.01).to(torch.uint8)}
    rp = P.replay_from_tensors(R)
    idx = torch.randint(0, cap, (1, B), generator=g, device=dev, dtype=torch.int64)
    sh = torch.randint(0, 5, (1, B, 4), generator=g, device=dev, dtype=torch.uint8)
    eps = torch.randn((1, 2, B, A), generator=g, device=dev)
    met = torch.zeros((1, 8), device=dev)
    for _ in range(reps):
        L.update(rp, idx, sh, eps, met)
torch.cuda.synchronize()
print("ncu_work", which, "done")
