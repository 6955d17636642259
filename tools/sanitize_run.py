"""Small workload for compute-sanitizer: one c0 fp32 update, one bf16 update
at c2 shapes (batch 64, the tcgen05 / TMA / cluster kernels), squint insert / insert2 / insert_ex and
act (fp32 and bf16), each checked against the oracle so a run that passes the tool also computed the
right numbers.  Usage:
  compute-sanitizer --tool memcheck python tools/sanitize_run.py [fp32|bf16|rollout|all]
(SQUINT_NO_GRAPH=1 is set: launches go straight to the stream instead of a cached graph.)"""
import os
import sys

os.environ.setdefault("SQUINT_NO_GRAPH", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import squint_inputs as SI  # noqa: E402
from harness import Problem, compare  # noqa: E402

import paper_2602_21203_b200 as P  # noqa: E402


def fp32():
    pr = Problem("c0", utd=1, seed=0)
    L = pr.gpu_setup()
    met = pr.gpu_update(L)
    _, ref = pr.oracle_update()
    compare("L_Q fp32", met[0, 0], ref[0, 0], 1e-4)


def bf16():
    pr = Problem("c2", capacity=1024, utd=1, seed=2, batch=64)
    L = pr.gpu_setup(precision=P.BF16)
    met = pr.gpu_update(L)
    _, ref = pr.oracle_update()
    compare("L_Q bf16", met[0, 0], ref[0, 0], 2e-2)


def rollout():
    dev = "cuda"
    frames = SI.make_frames(16, 128, seed=1)
    slots = SI.make_slots(16, 64, seed=1)
    ring = torch.zeros((64, 3, 16, 16), dtype=torch.uint8, device=dev)
    ring2 = torch.zeros_like(ring)
    ft, st = torch.as_tensor(frames).to(dev), torch.as_tensor(slots).to(dev)
    P.squint_insert(ft, 8, st, ring)
    P.squint_insert2(ft, 8, st, ring, (st + 7) % 64, ring2)
    P.squint_insert_ex(ft.permute(0, 2, 3, 1).contiguous(), 8, st, ring, hwc=True,
                       jitter=torch.as_tensor(SI.make_jitter(16)).to(dev))
    torch.cuda.synchronize()
    assert np.array_equal(ring2[(st + 7) % 64].cpu().numpy(), O.area_downsample(frames, 8))
    for prec in (P.FP32, P.BF16):
        pr = Problem("c0", seed=5)
        L = pr.gpu_setup(precision=prec)
        prop = SI.make_proprio(16, 12, seed=1)
        eps = np.random.default_rng(1).standard_normal((16, 6)).astype(np.float32)
        dims = P.make_dims(pr.dims, prec)
        ws = torch.zeros(P.act_workspace_bytes(dims, 16), dtype=torch.uint8, device=dev)
        act = torch.zeros((16, 6), device=dev)
        lp = torch.zeros(16, device=dev)
        P.squint_act(dims, P.make_hparams(pr.hp), L.actor, L.critic, ft, torch.as_tensor(prop).to(dev),
                     torch.as_tensor(eps).to(dev), act, lp, ws)
        torch.cuda.synchronize()
        st_ = O.init_state(pr.specs, pr.vals)
        a_ref, _, _ = O.act(pr.d, pr.h, st_["critic"], st_["actor"], frames, prop, eps)
        compare("act", act.cpu().numpy(), a_ref, 2e-2)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    for name, fn in (("fp32", fp32), ("bf16", bf16), ("rollout", rollout)):
        if which in (name, "all"):
            fn()
            print(f"sanitize_run {name}: ok", flush=True)
