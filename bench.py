"""bench.py -- Squint hot path on B200: SAC gradient updates/s (BASELINE.json metric).

One step = one Algorithm-1 iteration at BASELINE configs[2]:
  squint_insert2 of the N_env = 1024 new rendered 3x128x128 frames o_{t+1}: squinted once into
               the ring's next_obs rows and into the 16x16 rows the next act encodes (a1, f2),
  squint_act   on the 1024 squinted o_t (encoder + actor + sample, o_t written into the 1M
               replay ring's obs rows: a16 + a1),
  squint_update with UTD 4 at batch 512 (a2-a15), 101 atoms on [-20, 20].
The insert and the act run on side streams beside the updates: the act reads a snapshot of the
weights taken before the step's first optimizer step (squint_act_ex; the updates wait for that copy
only) and the updates sample ring rows outside the step's own slots (the newest transitions become
sampleable one step later).  (--act-full: the act squints a second 128x128 batch itself, the insert
writes next_obs only.)

value = optimizer updates/s of the GLOBAL batch (UTD * K / time).  With N > 1 ranks (torchrun)
the global batch is split: --config c2 (default) keeps the metric's "batch 512" and gives each rank
512 / N samples and 1024 / N environments (SURVEY §8(d) c3'); --config c3 splits BJ configs[3]'s
global batch 4096 into 4096 / N.  Gradients are NCCL all-reduced (Q33); every rank samples its own
seeded indices from its replica of the ring.  Scaling is therefore "strong"; samples/s =
value * global batch is reported beside it.  Inputs live in HBM before the timed region; the
replay ring (1.66 GB per rank) and four rotating 50 MB frame pools exceed the 126 MB L2.

Beside the headline line's step, rank 0 times the other BJ configs (keys of the same JSON line):
c1 (squint insert of 1024 frames into the 1M ring, µs/call, GB/s against HBM), c4 (rollout act on
4096 128x128 frames: latency, frames/s, GB/s) and, at N = 1, c3 (the large-batch update on one GPU:
updates/s and its dominant kernel's tensor roofline).  Launch: python bench.py [--gpus N --steps K
--warmup W] (torchrun for N > 1).  --impl reference times the CPU oracle instead (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import squint_inputs as SI  # noqa: E402

N_ENV = 1024
UTD = 4
CFG = "c2"
METRIC = "SAC gradient updates/sec (batch 512, 1/2/4/8 B200) + % HBM/tensor roofline"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(n) if n else os.cpu_count()
    except Exception:
        return os.cpu_count()


# ---------------------------------------------------------------------------------------
# CPU oracle sample (cpu_baseline leg and --impl reference)
# ---------------------------------------------------------------------------------------
def variant(args):
    """(dims, hparams, label) of the workload: c2, or one of its f3/f4 variants."""
    d = SI.dims_of(args.config, critic_kind=1 if args.critic == "mse" else 0)
    hp = SI.hp_of(args.config, target_mode=1 if args.target == "cdq" else 0)
    parts = ([] if args.critic == "c51" else ["scalar MSE critic"]) + ([] if args.target == "avg" else ["CDQ-min target"]) \
        + ([] if args.insert == "chw" else [{"hwc": "HWC frames", "jitter": "colour jitter",
                                             "hwc-jitter": "HWC frames + colour jitter"}[args.insert]]) \
        + (["replay capacity (P:189)"] if args.capacity else []) \
        + ([f"{args.config} shapes (batch {d['batch']}, C {d['conv_ch']}, critic {d['critic_hidden']})"]
           if args.config != CFG else [])
    return d, hp, ("; variant: " + ", ".join(parts)) if parts else ""


def oracle_sample(args, seed=0, n_frames=N_ENV // UTD):
    """One update's share of a step on the CPU oracle: act + insert on n_frames frames and
    one c2 update (B = 512) on rows gathered from a seeded replay sample."""
    import oracle as O
    d, hp, _ = variant(args)
    D, H = O.Dims(**d), O.HParams(**hp)
    specs = O.param_specs(D)
    vals = SI.make_params(specs, seed=1)
    st = O.init_state(specs, vals)
    B = d["batch"]
    R = SI.make_replay(4 * B, d, seed=seed)  # rows the sample draws from (same distribution as the ring)
    idx = SI.make_indices(1, B, 4 * B, seed=2 + seed)
    sh = SI.make_shifts(1, B, d["pad"], seed=2 + seed)
    eps = SI.make_eps(1, B, d["action_dim"], seed=3 + seed)
    frames = SI.make_frames(n_frames, 128, seed=seed)
    nxt = SI.make_frames(n_frames, 128, seed=seed + 100)
    prop = SI.make_proprio(n_frames, d["proprio_dim"], seed=seed)
    ae = np.random.default_rng(seed).standard_normal((n_frames, d["action_dim"])).astype(np.float32)
    t0 = time.perf_counter()
    O.act(D, H, st["critic"], st["actor"], frames, prop, ae)
    hwc = args.insert.startswith("hwc")
    jit = SI.make_jitter(n_frames, seed=seed) if args.insert.endswith("jitter") else None
    O.insert_ex(np.ascontiguousarray(nxt.transpose(0, 2, 3, 1)) if hwc else nxt, 8, np.arange(n_frames),
                np.zeros((n_frames, 3, 16, 16), np.uint8), hwc=hwc, jitter=jit)
    O.update(D, H, R, idx, sh, eps, st)
    return time.perf_counter() - t0


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    for w in range(args.warmup):
        oracle_sample(args, seed=w)
    ts = [oracle_sample(args, seed=100 + k) for k in range(args.steps)]
    tot = sum(ts)
    value = args.steps / tot  # one update per sample
    cores = blas_threads()
    sample = (f"per step: oracle act+insert on {N_ENV // UTD} frames + 1 update at B={variant(args)[0]['batch']} "
              f"({args.config} shapes), float64 NumPy")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "updates/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "c2 update share of an Algorithm-1 step (CPU oracle)" + variant(args)[2],
                       "global_batch": variant(args)[0]["batch"],
                       "utd": 1, "n_env_frames": N_ENV // UTD},
            "cpu_baseline": {"value": value, "unit": "updates/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in out.strip().splitlines():
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------------
# the GPU arm
# ---------------------------------------------------------------------------------------
def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2602_21203_b200 as P
    from paper_2602_21203_b200 import squint as S

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # NCCL's own log (stderr) names the ranks, the transport and whether NVLS is used
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        dist.init_process_group("nccl", device_id=dev)
    precision = {"fp32": P.FP32, "bf16": P.BF16}[args.precision]
    d, hp, vlabel = variant(args)
    # the global batch (configs[2]: 512, configs[3]: 4096) and the environments are split over ranks
    gbatch = d["batch"]
    if gbatch % world or N_ENV % world:
        raise SystemExit(f"global batch {gbatch} / {N_ENV} envs not divisible by {world} ranks")
    d["batch"] = gbatch // world
    n_env = N_ENV // world
    B, A = d["batch"], d["action_dim"]
    cap = args.capacity or SI.CONFIGS[args.config]["capacity"]
    K, W = args.steps, args.warmup

    L = P.Learner(d, hp, precision=precision, device=dev, utd=UTD)
    layout3 = [(S.GROUP_NAMES[g], n, s) for g, n, off, s in L.layout]
    L.load_values(SI.make_params(SI.specs_from_layout(layout3), seed=1))
    if world > 1:
        uid = bytearray(128)
        if rank == 0:
            uid = bytearray(S.comm_unique_id())
        t = torch.tensor(list(uid), dtype=torch.uint8, device=dev)
        dist.broadcast(t, 0)
        L.comm = S.comm_init(bytes(t.cpu().tolist()), rank, world)
        if args.comm_mode == 1 and precision == P.BF16:
            # f1: peer-memory all-reduce fused with a sharded Adam (the warm step before the graph
            # capture maps the peers' buffers)
            S.comm_set_mode(L.comm, 1)

    # replay ring (replica per rank, data seed 0): device-side seeded fill, same distributions as c0
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    R = {
        "obs": torch.randint(0, 256, (cap, 3, 16, 16), generator=g, device=dev, dtype=torch.uint8),
        "next_obs": torch.randint(0, 256, (cap, 3, 16, 16), generator=g, device=dev, dtype=torch.uint8),
        "proprio": torch.randn((cap, d["proprio_dim"]), generator=g, device=dev),
        "next_proprio": torch.randn((cap, d["proprio_dim"]), generator=g, device=dev),
        "action": torch.rand((cap, A), generator=g, device=dev) * 2 - 1,
        "reward": torch.rand((cap,), generator=g, device=dev),
        "done": (torch.rand((cap,), generator=g, device=dev) < 0.01).to(torch.uint8),
    }
    replay = P.replay_from_tensors(R)
    # per-step inputs for all K + W steps, resident in HBM
    T = K + W
    gi = torch.Generator(device=dev)
    gi.manual_seed(2 + 1000 * rank)
    # step k's updates sample the ring outside the block its own act / insert write (slots of step
    # k = [k n_env, (k + 1) n_env) mod cap): the newest transitions become sampleable one step later,
    # so the act (policy before the step's updates, weights snapshotted by squint_act_ex) and the
    # insert run beside the updates (R-step)
    idx_all = torch.randint(0, cap - n_env, (T, UTD, B), generator=gi, device=dev, dtype=torch.int64)
    idx_all = (idx_all + ((torch.arange(T, device=dev) + 1) * n_env).view(T, 1, 1)) % cap
    sh_all = torch.randint(0, 2 * d["pad"] + 1, (T, UTD, B, 4), generator=gi, device=dev, dtype=torch.uint8)
    eps_all = torch.randn((T, UTD, 2, B, A), generator=gi, device=dev)
    aeps_all = torch.randn((T, n_env, A), generator=gi, device=dev)
    prop_all = torch.randn((T, n_env, d["proprio_dim"]), generator=gi, device=dev)
    slots_all = torch.stack([(torch.arange(n_env, device=dev) + k * n_env) % cap for k in range(T)])
    # rotating pools of rendered frames o_{t+1} (4 x 50 MB > L2).  Algorithm 1 reads each new
    # observation once: squint_insert2 squints o_{t+1} into the finished transition's
    # next_obs row and into a 16x16 staging buffer that the next step's act encodes (factor 1),
    # writing it on into that transition's obs row.  --act-full: the round-1 step instead (act
    # squints a second frame batch itself; the insert writes next_obs only).
    NPOOL = 4
    hwc = args.insert.startswith("hwc")
    pools = [torch.as_tensor(SI.make_frames(n_env, 128, seed=20 + p)).to(dev) for p in range(NPOOL)]
    if hwc:  # what renderers emit (f4)
        pools = [x.permute(0, 2, 3, 1).contiguous() for x in pools]
    jit = torch.as_tensor(SI.make_jitter(n_env)).to(dev) if args.insert.endswith("jitter") else None
    act_pool = [torch.as_tensor(SI.make_frames(n_env, 128, seed=10 + p)).to(dev) for p in range(NPOOL)] \
        if args.act_full else None
    stage = [torch.empty((n_env, 3, 16, 16), dtype=torch.uint8, device=dev) for _ in range(2)]
    stage_slots = torch.arange(n_env, device=dev, dtype=torch.int64)
    NG = NPOOL  # graphs: pool j % NPOOL, staging parity j % 2 (NPOOL even)
    # static per-step buffers that the graphs read
    idx_s, sh_s, eps_s = idx_all[0].clone(), sh_all[0].clone(), eps_all[0].clone()
    aeps_s, prop_s, slots_s = aeps_all[0].clone(), prop_all[0].clone(), slots_all[0].clone()
    metrics = torch.zeros((UTD, 8), device=dev)
    act_out = torch.zeros((n_env, A), device=dev)
    logp_out = torch.zeros((n_env,), device=dev)
    act_ws = torch.zeros(P.act_workspace_bytes(L.dims, n_env), dtype=torch.uint8, device=dev)
    obs_ring = R["obs"]
    next_ring = R["next_obs"]
    def insert_new(frames, slots, stage_dst, stream=None):
        # o_{t+1} -> next_obs[slots] and the next act's rows, one squint (f2; f4 variants)
        if args.insert == "chw":
            P.squint_insert2(frames, 8, slots, next_ring, stage_slots, stage_dst, stream=stream)
        else:
            P.squint_insert_ex(frames, 8, slots, next_ring, hwc=hwc, jitter=jit, slots2=stage_slots, ring2=stage_dst,
                               stream=stream)

    # o_0, squinted
    P.squint_insert_ex(pools[NPOOL - 1], 8, stage_slots, stage[0], hwc=hwc, jitter=jit)

    side = torch.cuda.Stream(device=dev)
    side_act = torch.cuda.Stream(device=dev)
    ins_fork, ins_done, act_done = torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event()
    weights_read = torch.cuda.Event()
    weights_read.record()  # (created lazily by torch: materialise it before any capture)

    def step(j, stream=None, serial=False):
        # The insert of o_{t+1} (HBM-bound) and the act on o_t run on side streams beside the
        # updates: the updates sample rows outside this step's slots (idx_all), and the act reads a
        # snapshot of the weights taken before the first optimizer step (squint_act_ex: the updates
        # wait only for that copy).  Both join at the end of the step.  serial=True (the launch
        # timeline) runs the act on the caller's stream before the updates.
        nx, par = pools[j % NPOOL], j % 2
        cur = stream if stream is not None else torch.cuda.current_stream()
        ins_fork.record(cur)
        side.wait_event(ins_fork)
        with torch.cuda.stream(side):
            if args.act_full:
                P.squint_insert(nx, 8, slots_s, next_ring, stream=side)
            else:
                insert_new(nx, slots_s, stage[1 - par], stream=side)
            ins_done.record(side)
        fr = act_pool[j % NPOOL] if args.act_full else stage[par]
        if serial:
            P.squint_act(L.dims, L.hp, L.actor, L.critic, fr, prop_s, aeps_s, act_out, logp_out, act_ws,
                         ring=obs_ring, slots=slots_s, stream=stream)
        else:
            side_act.wait_event(ins_fork)
            with torch.cuda.stream(side_act):
                P.squint_act(L.dims, L.hp, L.actor, L.critic, fr, prop_s, aeps_s, act_out, logp_out, act_ws,
                             ring=obs_ring, slots=slots_s, stream=side_act, weights_read=weights_read)
                act_done.record(side_act)
            cur.wait_event(weights_read)
        L.update(replay, idx_s, sh_s, eps_s, metrics, stream=stream)
        cur.wait_event(ins_done)
        if not serial:
            cur.wait_event(act_done)

    def load_inputs(k):
        idx_s.copy_(idx_all[k], non_blocking=True)
        sh_s.copy_(sh_all[k], non_blocking=True)
        eps_s.copy_(eps_all[k], non_blocking=True)
        aeps_s.copy_(aeps_all[k], non_blocking=True)
        prop_s.copy_(prop_all[k], non_blocking=True)
        slots_s.copy_(slots_all[k], non_blocking=True)

    # eager warm step: counts launches, checks errors
    c0 = S.launch_count()
    load_inputs(0)
    step(0)
    torch.cuda.synchronize()
    launches_per_step = S.launch_count() - c0

    graphs = []
    use_graph = not args.no_graph
    if use_graph:
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            step(0)  # warm on the capture stream
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        # the updates (the step's critical path) on a high-priority stream; the act and the insert
        # beside them keep the default priority (c2 6145 -> 6190 updates/s, A/B on one box)
        cap_s = torch.cuda.Stream(device=dev, priority=-1)
        for j in range(NG):
            gph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gph, stream=cap_s):
                step(j)
            graphs.append(gph)
        torch.cuda.synchronize()

    def run_one(k):
        load_inputs(k)
        if use_graph:
            graphs[k % NG].replay()
        else:
            step(k % NG)

    for w in range(W):
        run_one(w)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    st.record()
    for k in range(W, W + K):
        run_one(k)
    en.record()
    torch.cuda.synchronize()
    ms = st.elapsed_time(en)
    clocks = clk.stop()
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    met = metrics.cpu().numpy()
    if not np.isfinite(met).all() or met[:, 7].any():
        print(f"rank {rank}: non-finite metrics {met}", file=sys.stderr)
        sys.exit(3)

    # per-kernel device time inside the step: a second capture of the same step with a CUDA event
    # before every libsquint launch (libsquint's launch timeline), replayed after the timed region.
    # The timeline capture runs the update on one stream (no encoder-backward branch); events
    # between kernels add small gaps and stop programmatic-launch overlap, so these durations
    # are pessimistic; shares are taken against their own sum.
    kern, event_overhead_us = {}, None
    if use_graph and not args.no_timeline:
        kern, event_overhead_us = timeline(S, torch, dev, lambda st: step(0, stream=st, serial=True), reps=10,
                                           load=lambda r: load_inputs(W + (r % K)))

    # e2e: the environment loop through the public API from pinned host buffers.  Step t acts on
    # o_t (squinted by step t-1's insert2), reads the actions back, uploads the new observation
    # o_{t+1} (the env's output; each frame batch crosses PCIe once) and the step's small inputs,
    # runs the UTD updates and inserts o_{t+1} once: next_obs of transition t and the staging rows
    # the next act encodes.  The frame upload runs on copy streams beside the act and the updates
    # (which sample the ring as it was before o_{t+1} is inserted); the insert waits for it.
    # Results (actions, log pi, metrics) go back to pinned host memory every step.
    e2e = None
    if not args.no_e2e:
        h_fr = [pools[p].cpu().pin_memory() for p in range(NPOOL)]
        # the step's small inputs packed into one pinned byte row per step (one H2D copy instead of
        # six) and unpacked on the device as views of one staging buffer (256-byte aligned parts)
        srcs = (idx_all, sh_all, eps_all, aeps_all, prop_all, slots_all)
        offs, o = [], 0
        for t in srcs:
            offs.append(o)
            o += (t[0].numel() * t.element_size() + 255) // 256 * 256
        h_pack = torch.zeros((T, o), dtype=torch.uint8).pin_memory()
        for t, off in zip(srcs, offs):
            nb = t[0].numel() * t.element_size()
            h_pack[:, off:off + nb] = t.reshape(T, -1).contiguous().cpu().view(torch.uint8)
        # two device staging sets: step k+1's inputs are staged during step k
        d_pack = [torch.zeros(o, dtype=torch.uint8, device=dev) for _ in range(2)]
        stage_in = [[dp[off:off + t[0].numel() * t.element_size()].view(t.dtype).view(t[0].shape)
                     for t, off in zip(srcs, offs)] for dp in d_pack]
        h_out = [torch.empty(x.shape, dtype=x.dtype).pin_memory() for x in (act_out, logp_out, metrics)]
        dbuf = [pools[0].clone(), pools[1].clone()]
        main = torch.cuda.current_stream()
        # the small inputs travel through the SMs (squint_stage_pinned: a kernel reading pinned
        # host memory), not a copy engine, so they never queue behind a frame upload; the read
        # shares the link with the upload (~0.2 ms for 100 KB), so it runs one step ahead on a
        # stream of its own
        stg = torch.cuda.Stream(device=dev)
        staged = [torch.cuda.Event(), torch.cuda.Event()]  # d_pack[i] holds its step's inputs
        used = [torch.cuda.Event(), torch.cuda.Event()]    # d_pack[i] read by its step

        def stage_inputs(k):
            if k < T:
                stg.wait_event(used[k % 2])
                P.squint_stage_pinned(d_pack[k % 2], h_pack[k], stream=stg)
                staged[k % 2].record(stg)
        # the frame upload in two halves on two copy streams (one DMA stream does not saturate
        # the link: 47 vs 54 GB/s measured)
        cps = [torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)]
        freed = [torch.cuda.Event(), torch.cuda.Event()]  # dbuf[i] read by its last consumer
        copied = [torch.cuda.Event(), torch.cuda.Event()]
        half = h_fr[0].shape[0] // 2

        def e2e_step(k):
            nxt = dbuf[k % 2]
            idx, sh, eps, aeps, prop, slots = stage_in[k % 2]
            stage_inputs(k + 1)
            main.wait_event(staged[k % 2])
            # o_{t+1} -> dbuf[k % 2] once step k-2's insert (or, --act-full, step k-1's act) read it
            for c, sl in enumerate((slice(0, half), slice(half, None))):
                cps[c].wait_event(freed[k % 2])
                with torch.cuda.stream(cps[c]):
                    nxt[sl].copy_(h_fr[k % NPOOL][sl], non_blocking=True)
                    copied[c].record(cps[c])
            fr = dbuf[(k + 1) % 2] if args.act_full else stage[k % 2]
            # the act (and the read-back of its actions) beside the updates, as in the device step
            side_act.wait_event(staged[k % 2])
            side_act.wait_stream(main)
            with torch.cuda.stream(side_act):
                P.squint_act(L.dims, L.hp, L.actor, L.critic, fr, prop, aeps, act_out, logp_out, act_ws,
                             ring=obs_ring, slots=slots, stream=side_act, weights_read=weights_read)
                if args.act_full:
                    freed[(k + 1) % 2].record(side_act)
                for dst, src in zip(h_out[:2], (act_out, logp_out)):
                    dst.copy_(src, non_blocking=True)
                act_done.record(side_act)
            main.wait_event(weights_read)
            L.update(replay, idx, sh, eps, metrics)
            main.wait_event(act_done)
            main.wait_event(copied[0])
            main.wait_event(copied[1])
            if args.act_full:
                P.squint_insert(nxt, 8, slots, next_ring)
            else:
                insert_new(nxt, slots, stage[(k + 1) % 2])
                freed[k % 2].record(main)
            used[k % 2].record(main)
            h_out[2].copy_(metrics, non_blocking=True)

        dbuf[1].copy_(h_fr[NPOOL - 1], non_blocking=True)  # o_0 (--act-full acts on it)
        P.squint_insert_ex(dbuf[1], 8, stage_slots, stage[0], hwc=hwc, jitter=jit)  # o_0, squinted
        for e in freed + used:
            e.record(main)
        stage_inputs(0)
        for w in range(W):
            e2e_step(w)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        h0 = time.perf_counter()
        for k in range(W, W + K):
            e2e_step(k)
        host_ms = (time.perf_counter() - h0) * 1e3 / K  # enqueue time per step (the host's share)
        b.record()
        torch.cuda.synchronize()
        ems = a.elapsed_time(b)
        if world > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        h2d = h_fr[0].numel() + h_pack[0].numel()
        d2h = sum(x.numel() * x.element_size() for x in h_out)
        e2e = {"value": UTD * K / (ems / 1e3), "unit": "updates/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": ems / K, "host_enqueue_ms_per_step": host_ms,
               "loop": ("act(o_t) -> D2H actions -> H2D o_{t+1} (copy streams, beside the act and the updates) -> "
                        + ("insert(o_{t+1}) after the updates" if args.act_full else
                           "insert2(o_{t+1}: next_obs + the next act's squinted rows) after the updates"))}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    traffic_tab = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))) if os.path.exists(
        os.path.join(ROOT, "profiles", "traffic.json")) else {}
    roof = roofline_of(kern, peaks, traffic_tab)
    if roof:
        roof["timeline_event_overhead_us"] = event_overhead_us
    kernels_us = {k: round(v["us"], 2) for k, v in sorted(kern.items(), key=lambda kv: -kv[1]["us"])}
    # the other BASELINE configs on this GPU (rank 0): c1 insert, c4 act, c3 update (N = 1)
    extra = {}
    if not args.no_sub:
        extra["c1_insert"] = bench_c1(P, torch, dev, pools, cap, K, W, peaks)
        extra["c4_act"] = bench_c4(P, torch, dev, L, d, K, W, peaks)
        if world == 1 and args.config == CFG and args.critic == "c51" and args.target == "avg":
            extra["c3_update"] = bench_c3(P, S, torch, dev, replay, cap, K, W, peaks, traffic_tab)
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args, B)
    value = UTD * K / (ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": "updates/s", "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": {P.FP32: "f32", P.BF16: "bf16"}[precision], "data": "synthetic",
            "samples_per_s": value * gbatch,
            "config": {"workload": f"{args.config}: Algorithm-1 step = insert2({n_env} new 128x128 frames) + act({n_env} envs) + "
                                   f"{UTD} updates at global batch {gbatch} ({B} per rank), "
                                   f"{d['n_atoms']} atoms, {cap:,}-row ring"
                                   + (" (act squints its own frames)" if args.act_full else "") + vlabel,
                       "global_batch": gbatch, "batch_per_rank": B, "utd": UTD,
                       "n_env": N_ENV, "parallelism": f"dp{world}", "capacity": cap,
                       "grad_exchange": ("peer-sharded-adam" if args.comm_mode == 1 and args.precision == "bf16"
                                         else "nccl-allreduce") if world > 1 else "none",
                       "l2": f"ring {cap * 1662 / 1e9:.2f} GB + rotating frame pools (4 x {n_env * 49152 / 1e6:.0f} MB) > L2",
                       "graph": use_graph},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": int(launches_per_step * K), "kernels_us_per_step": kernels_us}
    line.update(extra)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def roofline_of(kern, peaks, traffic_tab):
    """Roofline of the dominant kernel (largest device time per step in a launch timeline)."""
    if not kern:
        return None
    tot_us = sum(e["us"] for e in kern.values())
    dom = max(kern, key=lambda k: kern[k]["us"])
    e = kern[dom]
    t_launch = e["us"] / e["n"] * 1e-6  # seconds per launch
    if e["flops"] > 0:
        peak = peaks.get("bf16_tflops_sustained", 1400.0)  # kernel timed inside a long step
        roof = {"bound": "tensor", "achieved": e["flops"] / e["n"] / t_launch / 1e12, "peak": peak,
                "unit": "TFLOP/s", "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (of measured)"}
    else:
        peak = peaks.get("hbm_gbs", 6650.0)
        roof = {"bound": "hbm", "achieved": e["bytes"] / e["n"] / t_launch / 1e9, "peak": peak, "unit": "GB/s",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = traffic_tab.get(dom)
    roof["kernel"] = dom
    roof["launches_per_step"] = round(e["n"], 2)
    roof["us_per_launch"] = e["us"] / e["n"]
    roof["share_of_step"] = e["us"] / tot_us if tot_us > 0 else None
    return roof


def timeline(S, torch, dev, fn, reps=10, load=None):
    """Per-kernel device time of fn(stream): one graph capture with an event before every libsquint
    launch, replayed `reps` times (calibrated event overhead subtracted)."""
    tl = S.LaunchTimeline(4096)
    s2 = torch.cuda.Stream(device=dev)
    s2.wait_stream(torch.cuda.current_stream())
    oh = tl.calibrate(s2)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s2):
        tl.start()
    with torch.cuda.graph(g, stream=s2):
        fn(s2)
        tl.stop(s2)
    torch.cuda.synchronize()
    kern = {}
    for r in range(reps):
        if load:
            load(r)
        g.replay()
        torch.cuda.synchronize()
        for name, fl, by, us in tl.durations():
            e = kern.setdefault(name, {"us": 0.0, "n": 0, "flops": 0.0, "bytes": 0.0})
            e["us"] += us / reps
            e["n"] += 1.0 / reps
            e["flops"] += fl / reps
            e["bytes"] += by / reps
    return kern, oh


def _time_graph(torch, fn, K, W, pre=None):
    """ms per call of fn(j) captured as CUDA graphs (one per rotating input j % 2), CUDA events."""
    graphs = []
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn(0)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    for j in range(2):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn(j)
        graphs.append(g)
    for w in range(W):
        graphs[w % 2].replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(K):
        graphs[k % 2].replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K


def bench_c1(P, torch, dev, pools, cap, K, W, peaks):
    """BJ configs[1]: squint_insert of 1024 frames (50.3 MB, rotating pools > L2) into the 1M ring at
    seeded distinct random slots.  HBM-bound: 49,152 B read + 768 B written per frame."""
    n = pools[0].shape[0]
    ring = torch.zeros((cap, 3, 16, 16), dtype=torch.uint8, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(2)
    slots = [torch.randperm(cap, generator=g, device=dev)[:n].contiguous() for _ in range(2)]
    frames = [pools[0], pools[1]]  # 2 x 50 MB alternate (plus the ring rows written)
    ms = _time_graph(torch, lambda j: P.squint_insert(frames[j], 8, slots[j], ring), 4 * K, W)
    by = n * (49152 + 768)
    gbs = by / (ms * 1e-3) / 1e9
    peak = peaks.get("hbm_gbs", 6650.0)
    del ring
    return {"workload": f"c1: squint_insert of {n} frames 3x128x128 -> {cap:,}-row ring (random distinct slots)",
            "us_per_call": ms * 1e3, "frames_per_s": n / (ms * 1e-3),
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                         "bytes_per_call": by, "floor_us": by / (peak * 1e9) * 1e6,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)"}}


def bench_c4(P, torch, dev, L, d, K, W, peaks):
    """BJ configs[4]: rollout act on 4096 rendered 3x128x128 frames (201 MB per call; two pools > L2):
    squint -> encoder -> actor projection + MLP -> tanh-Gaussian sample with seeded noise."""
    n = 4096
    g = torch.Generator(device=dev)
    g.manual_seed(44)
    frames = [torch.randint(0, 256, (n, 3, 128, 128), generator=g, device=dev, dtype=torch.uint8) for _ in range(2)]
    prop = torch.randn((n, d["proprio_dim"]), generator=g, device=dev)
    eps = torch.randn((n, d["action_dim"]), generator=g, device=dev)
    act = torch.zeros((n, d["action_dim"]), device=dev)
    lp = torch.zeros((n,), device=dev)
    ws = torch.zeros(P.act_workspace_bytes(L.dims, n), dtype=torch.uint8, device=dev)
    ms = _time_graph(torch, lambda j: P.squint_act(L.dims, L.hp, L.actor, L.critic, frames[j], prop, eps, act, lp, ws),
                     2 * K, W)
    by = n * 49152
    gbs = by / (ms * 1e-3) / 1e9
    peak = peaks.get("hbm_gbs", 6650.0)
    del frames, ws
    return {"workload": f"c4: squint_act on {n} frames 3x128x128 (+ proprio, seeded N(0,1) noise) -> actions, log pi",
            "latency_us": ms * 1e3, "frames_per_s": n / (ms * 1e-3),
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                         "bytes_per_call": by, "floor_us": by / (peak * 1e9) * 1e6,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)"}}


def bench_c3(P, S, torch, dev, replay, cap, K, W, peaks, traffic_tab):
    """BJ configs[3] on one GPU (G = 1): the update at global batch 4096, C = 64, critic 512-512, 101
    atoms, on the same 1M-row ring; updates/s and the dominant kernel's tensor roofline."""
    d = SI.dims_of("c3")
    hp = SI.hp_of("c3")
    B, A = d["batch"], d["action_dim"]
    L3 = P.Learner(d, hp, precision=P.BF16, device=dev, utd=1)
    from paper_2602_21203_b200 import squint as S_
    layout3 = [(S_.GROUP_NAMES[g], n, s) for g, n, off, s in L3.layout]
    L3.load_values(SI.make_params(SI.specs_from_layout(layout3), seed=1))
    gi = torch.Generator(device=dev)
    gi.manual_seed(2)
    idx = [torch.randint(0, cap, (1, B), generator=gi, device=dev, dtype=torch.int64) for _ in range(2)]
    sh = [torch.randint(0, 2 * d["pad"] + 1, (1, B, 4), generator=gi, device=dev, dtype=torch.uint8) for _ in range(2)]
    eps = [torch.randn((1, 2, B, A), generator=gi, device=dev) for _ in range(2)]
    met = torch.zeros((1, 8), device=dev)
    fn = lambda j, stream=None: L3.update(replay, idx[j], sh[j], eps[j], met, stream=stream)
    ms = _time_graph(torch, fn, 2 * K, W)
    kern, oh = timeline(S, torch, dev, lambda st: fn(0, st), reps=5)
    roof = roofline_of(kern, peaks, traffic_tab)
    flops = 74.05e9
    return {"workload": f"c3 on one GPU: update at batch {B}, C {d['conv_ch']}, critic {d['critic_hidden']}-"
                        f"{d['critic_hidden']}, {d['n_atoms']} atoms, {cap:,}-row ring",
            "updates_per_s": 1e3 / ms, "ms_per_update": ms,
            "tflops": flops / (ms * 1e-3) / 1e12, "tensor_frac_of_update": flops / (ms * 1e-3) / 1e12 /
            peaks.get("bf16_tflops_sustained", 1400.0),
            "roofline": roof, "kernels_us_per_update": {k: round(v["us"], 2) for k, v in
                                                        sorted(kern.items(), key=lambda kv: -kv[1]["us"])}}


def cpu_baseline(args, B):
    """The oracle as it stands on this host: BLAS threads = all cores and = 1."""
    import platform
    model = platform.processor() or ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    ts = [oracle_sample(args, seed=s) for s in range(args.cpu_samples)]
    out = {"value": len(ts) / sum(ts), "unit": "updates/s", "cores": blas_threads(), "kind": "oracle",
           "sample": f"{len(ts)} x (oracle act+insert on {N_ENV // UTD} frames + 1 update at B={B}), "
                     f"{sum(ts):.1f} s float64 NumPy", "cpu_count": os.cpu_count(), "cpu_model": model}
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1, user_api="blas"):
            t1 = [oracle_sample(args, seed=s) for s in range(args.cpu_samples)]
        out["value_1_thread"] = len(t1) / sum(t1)
    except Exception as e:  # threadpoolctl missing: report why
        out["value_1_thread"] = None
        out["note_1_thread"] = str(e)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="squint", choices=["squint", "reference"])
    ap.add_argument("--precision", default="bf16", choices=["fp32", "bf16"])  # configs[2]: bf16 tensor cores
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-samples", type=int, default=3)
    ap.add_argument("--no-timeline", action="store_true")
    ap.add_argument("--no-sub", action="store_true")  # skip the c1 / c4 / c3 side measurements
    ap.add_argument("--act-full", action="store_true")  # round-1 step: act squints its own frame batch
    # f3 / f4 variants (not the headline workload): critic head, target rule, insert input
    ap.add_argument("--critic", default="c51", choices=["c51", "mse"])
    ap.add_argument("--target", default="avg", choices=["avg", "cdq"])
    ap.add_argument("--insert", default="chw", choices=["chw", "hwc", "jitter", "hwc-jitter"])
    ap.add_argument("--config", default=CFG, choices=["c2", "c3"])  # c3: the DP shapes on one GPU (B 4096)
    # N > 1: 0 = ncclAllReduce + replicated Adam, 1 = peer-memory all-reduce fused with a sharded Adam (f1)
    ap.add_argument("--comm-mode", type=int, default=0, choices=[0, 1])
    ap.add_argument("--capacity", type=int, default=0)  # replay rows (0: configs' 1M; f3: 100K axis)
    args = ap.parse_args()
    if args.act_full and args.insert != "chw":
        ap.error("--act-full acts on CHW frames: use it with --insert chw")
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
