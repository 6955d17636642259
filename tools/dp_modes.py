"""f1 at G = 1 on one B200: the bf16 update's time per update with no communicator, with a
one-rank communicator in mode 0 (ncclAllReduce, a no-op at one rank, + replicated Adam) and in
mode 1 (peer-memory all-reduce fused with a sharded Adam: two one-block barriers per group and a
separate shadow refresh).  The difference is the fixed cost of mode 1's structure; at G > 1 its
Adam traffic per rank falls by G and the all-reduce disappears.  CUDA graphs,
CUDA events, W warm-up replays, K timed."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_21203_b200 as P  # noqa: E402
import squint_inputs as SI  # noqa: E402
from paper_2602_21203_b200 import squint as S  # noqa: E402


def run(cfg, mode, K=200, W=20, cap=100_000, kernels=None):
    dev = torch.device("cuda")
    d, hp = SI.dims_of(cfg), SI.hp_of(cfg)
    B, A = d["batch"], d["action_dim"]
    L = P.Learner(d, hp, precision=P.BF16, device=dev, utd=1)
    layout3 = [(S.GROUP_NAMES[g], n, s) for g, n, off, s in L.layout]
    L.load_values(SI.make_params(SI.specs_from_layout(layout3), seed=1))
    comm = None
    if mode is not None:
        comm = S.comm_init(S.comm_unique_id(), 0, 1)
        S.comm_set_mode(comm, mode)
        L.comm = comm
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    Rt = {"obs": torch.randint(0, 256, (cap, 3, 16, 16), generator=g, device=dev, dtype=torch.uint8),
          "next_obs": torch.randint(0, 256, (cap, 3, 16, 16), generator=g, device=dev, dtype=torch.uint8),
          "proprio": torch.randn((cap, d["proprio_dim"]), generator=g, device=dev),
          "next_proprio": torch.randn((cap, d["proprio_dim"]), generator=g, device=dev),
          "action": torch.rand((cap, A), generator=g, device=dev) * 2 - 1,
          "reward": torch.randn((cap,), generator=g, device=dev),
          "done": (torch.rand((cap,), generator=g, device=dev) < 0.01).to(torch.uint8)}
    R = P.replay_from_tensors(Rt)
    idx = [torch.randint(0, cap, (1, B), generator=g, device=dev, dtype=torch.int64) for _ in range(2)]
    sh = [torch.randint(0, 2 * d["pad"] + 1, (1, B, 4), generator=g, device=dev, dtype=torch.uint8) for _ in range(2)]
    eps = [torch.randn((1, 2, B, A), generator=g, device=dev) for _ in range(2)]
    met = torch.zeros((1, 8), device=dev)
    ms = bench._time_graph(torch, lambda j: L.update(R, idx[j], sh[j], eps[j], met), K, W)
    if kernels is not None:
        kern, _ = bench.timeline(S, torch, dev, lambda st: L.update(R, idx[0], sh[0], eps[0], met, stream=st), reps=5)
        kernels.update({k: round(v["us"], 2) for k, v in kern.items()})
    if comm is not None:
        torch.cuda.synchronize()
        S.comm_destroy(comm)
    return ms * 1e3


if __name__ == "__main__":
    out = {}
    for cfg in ("c2", "c3"):
        for mode in (None, 0, 1):
            key = f"{cfg}_{'local' if mode is None else f'comm1_mode{mode}'}"
            out[key] = round(run(cfg, mode), 2)
            print(key, out[key], "us/update", flush=True)
    print(json.dumps(out))
    # per-kernel device time per update in each exchange mode (event timeline, serialised)
    for mode in (0, 1):
        kern = {}
        run("c3", mode, K=20, W=5, kernels=kern)
        print(f"c3 mode {mode} timeline:", json.dumps({k: v for k, v in kern.items()
                                                       if any(x in k for x in ("adam", "dp_", "sums", "shadow"))}))
