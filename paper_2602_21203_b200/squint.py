"""Thin ctypes binding of libsquint (include/squint.h).  Argument marshalling only: every
step of the hot path runs in the library's sm_100a kernels.  PyTorch provides device
memory, streams and process groups.  There is no CPU fallback: if the shared library is
missing the import fails loudly."""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsquint.so")

FP32, BF16 = 0, 1
GROUP_CRITIC, GROUP_ACTOR, GROUP_ALPHA, GROUP_TARGET = 0, 1, 2, 3
GROUP_NAMES = {GROUP_CRITIC: "critic", GROUP_ACTOR: "actor", GROUP_ALPHA: "alpha", GROUP_TARGET: "target"}
STATUS = {0: "OK", 1: "EINVAL", 2: "ESHAPE", 3: "ECUDA", 4: "ENCCL", 5: "EUNSUPPORTED"}
REGION = {"grad_critic": 0, "grad_actor": 1, "m": 2, "h": 3, "logp": 4, "logp_next": 5, "a_cur": 6, "scal": 7,
          "obs_shifted": 8, "next_obs_shifted": 9, "y1": 10}


class SquintError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Dims(C.Structure):
    _fields_ = [("img_c", C.c_int), ("img_h", C.c_int), ("img_w", C.c_int), ("pad", C.c_int), ("conv_ch", C.c_int),
                ("latent", C.c_int), ("proprio_dim", C.c_int), ("action_dim", C.c_int),
                ("critic_hidden", C.c_int), ("actor_hidden", C.c_int), ("n_atoms", C.c_int),
                ("v_min", C.c_float), ("v_max", C.c_float), ("batch", C.c_int), ("precision", C.c_int),
                ("critic_kind", C.c_int)]


CRITIC_C51, CRITIC_MSE = 0, 1


class HParams(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("gamma", "tau", "lr_critic", "lr_actor", "lr_alpha", "beta1", "beta2",
                                         "adam_eps", "target_entropy", "ln_eps", "log_std_min", "log_std_max")] + [
        ("target_mode", C.c_int)]


TARGET_AVG, TARGET_CDQ = 0, 1


class Replay(C.Structure):
    _fields_ = [("obs", C.c_void_p), ("next_obs", C.c_void_p), ("proprio", C.c_void_p), ("next_proprio", C.c_void_p),
                ("action", C.c_void_p), ("reward", C.c_void_p), ("done", C.c_void_p), ("capacity", C.c_int64),
                ("size", C.c_int64)]


class State(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("critic", "critic_target", "actor", "log_alpha", "m_critic", "v_critic",
                                          "m_actor", "v_actor", "m_alpha", "v_alpha", "step")]


class TensorDesc(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("group", C.c_int), ("offset", C.c_int64), ("numel", C.c_int64),
                ("ndim", C.c_int), ("shape", C.c_int * 4)]


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: build it with `python paper_2602_21203_b200/build.py` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(_LIB_PATH)
    st, vp, i64, i32, f32, sz = C.c_int, C.c_void_p, C.c_int64, C.c_int, C.c_float, C.c_size_t
    sig = {
        "squint_last_error": (C.c_char_p, []),
        "squint_version": (C.c_char_p, []),
        "squint_param_layout": (st, [C.POINTER(Dims), C.POINTER(TensorDesc), i32, C.POINTER(i32), C.POINTER(i64)]),
        "squint_workspace_bytes": (st, [C.POINTER(Dims), i32, C.POINTER(sz)]),
        "squint_workspace_region": (st, [C.POINTER(Dims), i32, C.POINTER(sz), C.POINTER(sz)]),
        "squint_act_workspace_bytes": (st, [C.POINTER(Dims), i64, C.POINTER(sz)]),
        "squint_comm_unique_id": (st, [vp]),
        "squint_comm_init": (st, [C.POINTER(vp), vp, i32, i32]),
        "squint_comm_destroy": (st, [vp]),
        "squint_comm_set_mode": (st, [vp, i32]),
        "squint_insert": (st, [vp, i64, i32, i32, i32, i32, vp, vp, i64, vp]),
        "squint_insert2": (st, [vp, i64, i32, i32, i32, i32, vp, vp, vp, vp, i64, vp]),
        "squint_insert_ex": (st, [vp, i64, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, i64, vp]),
        "squint_act": (st, [C.POINTER(Dims), C.POINTER(HParams), vp, vp, vp, i64, i32, i32, vp, vp, vp, vp, vp, vp,
                            i64, vp, vp]),
        "squint_act_ex": (st, [C.POINTER(Dims), C.POINTER(HParams), vp, vp, vp, i64, i32, i32, vp, vp, vp, vp, vp, vp,
                            i64, vp, vp, vp]),
        "squint_update": (st, [C.POINTER(Dims), C.POINTER(HParams), C.POINTER(Replay), vp, vp, vp, i32,
                               C.POINTER(State), vp, vp, sz, vp, vp]),
        "squint_soft_update": (st, [vp, vp, i64, f32, vp]),
        "squint_stage_pinned": (st, [vp, vp, sz, vp]),
        "squint_selftest_gemm": (st, [vp, i32, i32, i32, i32, vp, i32, i32, i32, i32, i32, i32, i32, vp, vp]),
        "squint_launch_count": (C.c_long, []),
        "squint_set_phase_events": (st, [C.POINTER(vp), i32, i32]),
        "squint_phase_name": (C.c_char_p, [i32]),
        "squint_set_launch_events": (i32, [C.POINTER(vp), i32]),
        "squint_record_launch_event": (st, [vp]),
        "squint_set_option": (st, [i32, i32]),
        "squint_launch_info": (st, [i32, C.POINTER(C.c_char_p), C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()
EXPORTED = ["squint_last_error", "squint_version", "squint_param_layout", "squint_workspace_bytes",
            "squint_workspace_region", "squint_act_workspace_bytes", "squint_comm_unique_id", "squint_comm_init",
            "squint_comm_destroy", "squint_comm_set_mode", "squint_insert", "squint_insert2", "squint_insert_ex", "squint_act", "squint_act_ex", "squint_update", "squint_soft_update", "squint_stage_pinned",
            "squint_launch_count", "squint_set_phase_events", "squint_phase_name", "squint_selftest_gemm",
            "squint_set_launch_events", "squint_record_launch_event", "squint_launch_info",
            "squint_set_option"]
N_PHASES = 16


def launch_count() -> int:
    return int(LIB.squint_launch_count())


def phase_name(k: int) -> str:
    return LIB.squint_phase_name(k).decode()


class PhaseTimer:
    """CUDA-event instrumentation of libsquint's phases (squint_set_phase_events)."""

    def __init__(self, reps):
        self.reps = reps
        self.events = [torch.cuda.Event(enable_timing=True) for _ in range(N_PHASES * reps * 2)]
        for e in self.events:  # torch creates the cudaEvent lazily, on first record
            e.record()
        torch.cuda.synchronize()
        self._arr = (C.c_void_p * len(self.events))(*[e.cuda_event for e in self.events])

    def enable(self):
        _check(LIB.squint_set_phase_events(self._arr, N_PHASES, self.reps))

    @staticmethod
    def disable():
        _check(LIB.squint_set_phase_events(None, 0, 0))

    def times_ms(self):
        """{phase name: summed ms over reps} for phases that recorded."""
        out = {}
        for k in range(N_PHASES):
            tot, hit = 0.0, False
            for r in range(self.reps):
                a, b = self.events[(k * self.reps + r) * 2], self.events[(k * self.reps + r) * 2 + 1]
                try:
                    tot += a.elapsed_time(b)
                    hit = True
                except RuntimeError:
                    pass
            if hit:
                out[phase_name(k)] = tot
        return out


class LaunchTimeline:
    """CUDA events around every libsquint launch (squint_set_launch_events), for per-kernel
    device durations inside a captured graph.  Capture the work between start() and stop(stream)."""

    def __init__(self, n=4096):
        self.n = n
        self.events = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
        for e in self.events:
            e.record()
        torch.cuda.synchronize()
        self._arr = (C.c_void_p * n)(*[e.cuda_event for e in self.events])
        self.used = 0

    def start(self):
        LIB.squint_set_option(1, 0)  # single-stream update while the timeline is captured
        LIB.squint_set_launch_events(self._arr, self.n)

    def stop(self, stream=None):
        LIB.squint_record_launch_event(_stream(stream))
        self.used = LIB.squint_set_launch_events(None, 0)
        LIB.squint_set_option(1, 1)
        return self.used

    def calibrate(self, stream, n=64, reps=10):
        """Device time of an interval between two consecutive timeline events with no kernel
        (graph-captured like the real timeline): subtracted from every launch interval."""
        g = torch.cuda.CUDAGraph()
        LIB.squint_set_launch_events(self._arr, n)
        with torch.cuda.graph(g, stream=stream):
            for _ in range(n):
                LIB.squint_record_launch_event(_stream(stream))
        LIB.squint_set_launch_events(None, 0)
        tot = 0.0
        for _ in range(reps):
            g.replay()
            torch.cuda.synchronize()
            tot += self.events[0].elapsed_time(self.events[n - 1]) * 1e3 / (n - 1)
        self.overhead_us = tot / reps
        return self.overhead_us

    def durations(self):
        """[(name, flops, bytes, us)] for each recorded launch (after the events completed); the
        calibrated per-event overhead (calibrate()) is subtracted."""
        out = []
        oh = getattr(self, "overhead_us", 0.0)
        for i in range(self.used - 1):
            nm, fl, by = C.c_char_p(), C.c_double(), C.c_double()
            _check(LIB.squint_launch_info(i, C.byref(nm), C.byref(fl), C.byref(by)))
            us = self.events[i].elapsed_time(self.events[i + 1]) * 1e3
            out.append((nm.value.decode(), fl.value, by.value, max(us - oh, 0.0)))
        return out


def _check(status):
    if status != 0:
        raise SquintError(status, LIB.squint_last_error().decode())


def _ptr(t):
    if t is None:
        return None
    if not t.is_contiguous():
        raise ValueError("libsquint takes contiguous tensors only (row-major layouts of squint.h)")
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def make_dims(d: dict, precision=FP32) -> Dims:
    return Dims(d["img_c"], d["img_h"], d["img_w"], d["pad"], d["conv_ch"], d["latent"], d["proprio_dim"],
                d["action_dim"], d["critic_hidden"], d["actor_hidden"], d["n_atoms"], d["v_min"], d["v_max"],
                d["batch"], precision, d.get("critic_kind", CRITIC_C51))


def make_hparams(h: dict) -> HParams:
    return HParams(*[h.get(n, 0) if n == "target_mode" else h[n] for n, _ in HParams._fields_])


def param_layout(dims: Dims):
    """[(group, name, offset, shape)], group_sizes[4]."""
    n = C.c_int(0)
    gs = (C.c_int64 * 4)()
    _check(LIB.squint_param_layout(C.byref(dims), None, 0, C.byref(n), gs))
    arr = (TensorDesc * n.value)()
    _check(LIB.squint_param_layout(C.byref(dims), arr, n.value, C.byref(n), gs))
    out = [(t.group, t.name.decode(), t.offset, tuple(t.shape[:t.ndim])) for t in arr]
    return out, [gs[i] for i in range(4)]


def workspace_bytes(dims: Dims, utd=1):
    b = C.c_size_t(0)
    _check(LIB.squint_workspace_bytes(C.byref(dims), utd, C.byref(b)))
    return b.value


def workspace_region(dims: Dims, name):
    o, b = C.c_size_t(0), C.c_size_t(0)
    _check(LIB.squint_workspace_region(C.byref(dims), REGION[name], C.byref(o), C.byref(b)))
    return o.value, b.value


def act_workspace_bytes(dims: Dims, n):
    b = C.c_size_t(0)
    _check(LIB.squint_act_workspace_bytes(C.byref(dims), n, C.byref(b)))
    return b.value


# ---- the four entry points, same names as the C ABI -----------------------------------
def squint_insert(frames: torch.Tensor, factor: int, slots: torch.Tensor, ring: torch.Tensor, stream=None):
    n, c, h, w = frames.shape
    _check(LIB.squint_insert(_ptr(frames), n, c, h, w, factor, _ptr(slots), _ptr(ring), ring.shape[0],
                             _stream(stream)))


def squint_insert2(frames: torch.Tensor, factor: int, slots: torch.Tensor, ring: torch.Tensor, slots2: torch.Tensor,
                   ring2: torch.Tensor, stream=None):
    n, c, h, w = frames.shape
    _check(LIB.squint_insert2(_ptr(frames), n, c, h, w, factor, _ptr(slots), _ptr(ring), _ptr(slots2), _ptr(ring2),
                              min(ring.shape[0], ring2.shape[0]), _stream(stream)))


LAYOUT_CHW, LAYOUT_HWC = 0, 1


def squint_insert_ex(frames: torch.Tensor, factor: int, slots: torch.Tensor, ring: torch.Tensor, hwc: bool = False,
                     jitter=None, slots2=None, ring2=None, stream=None):
    """frames [n, c, h, w] (or [n, h, w, c] with hwc=True); jitter None or f32 [n, 3]."""
    if hwc:
        n, h, w, c = frames.shape
    else:
        n, c, h, w = frames.shape
    cap = ring.shape[0] if ring2 is None else min(ring.shape[0], ring2.shape[0])
    _check(LIB.squint_insert_ex(_ptr(frames), n, c, h, w, factor, LAYOUT_HWC if hwc else LAYOUT_CHW, _ptr(jitter),
                                _ptr(slots), _ptr(ring), _ptr(slots2), _ptr(ring2), cap, _stream(stream)))


def squint_stage_pinned(dst: torch.Tensor, src: torch.Tensor, stream=None):
    """dst (device) <- src (pinned host), read by a kernel (squint.h)."""
    if not src.is_pinned():
        raise ValueError("squint_stage_pinned: src must be pinned host memory")
    nb = src.numel() * src.element_size()
    assert dst.numel() * dst.element_size() >= nb
    _check(LIB.squint_stage_pinned(_ptr(dst), _ptr(src), nb, _stream(stream)))


def squint_soft_update(target: torch.Tensor, online: torch.Tensor, tau: float, stream=None):
    assert target.numel() == online.numel()
    _check(LIB.squint_soft_update(_ptr(target), _ptr(online), target.numel(), tau, _stream(stream)))


def selftest_gemm(A: torch.Tensor, a_cols: int, a_mn: int, B: torch.Tensor, b_cols: int, b_mn: int, M: int, N: int,
                  K: int, out: torch.Tensor, stream=None):
    """out[m][n] = sum_k A(m, k) B(n, k) on the bf16 tcgen05 GEMM engine (see squint.h).  A, B are
    contiguous row-major storage whose first a_cols / b_cols columns are the matrix."""
    assert A.dtype == torch.bfloat16 and B.dtype == torch.bfloat16 and out.dtype == torch.float32
    _check(LIB.squint_selftest_gemm(_ptr(A), A.shape[0], a_cols, A.shape[1], a_mn, _ptr(B), B.shape[0], b_cols,
                                    B.shape[1], b_mn, M, N, K, _ptr(out), _stream(stream)))


def squint_act(dims: Dims, hp: HParams, actor: torch.Tensor, critic: torch.Tensor, frames: torch.Tensor,
               proprio: torch.Tensor, eps, action_out: torch.Tensor, logp_out, workspace: torch.Tensor,
               ring=None, slots=None, stream=None, weights_read=None):
    """weights_read: optional torch.cuda.Event recorded once the act has copied the weights it reads
    (squint_act_ex): optimizer steps may start after it."""
    n, _, fh, fw = frames.shape
    args = (C.byref(dims), C.byref(hp), _ptr(actor), _ptr(critic), _ptr(frames), n, fh, fw,
            _ptr(proprio), _ptr(eps), _ptr(action_out), _ptr(logp_out), _ptr(ring), _ptr(slots),
            0 if ring is None else ring.shape[0], _ptr(workspace), _stream(stream))
    if weights_read is None:
        _check(LIB.squint_act(*args))
    else:
        if not weights_read.cuda_event:
            raise ValueError("weights_read: record the torch.cuda.Event once before use (it is created lazily)")
        _check(LIB.squint_act_ex(*args, C.c_void_p(weights_read.cuda_event)))


def squint_update(dims: Dims, hp: HParams, replay: Replay, idx, shifts, eps, state: State, metrics,
                  workspace: torch.Tensor, comm=None, stream=None):
    utd = idx.shape[0]
    _check(LIB.squint_update(C.byref(dims), C.byref(hp), C.byref(replay), _ptr(idx), _ptr(shifts), _ptr(eps), utd,
                             C.byref(state), _ptr(metrics), _ptr(workspace), workspace.numel(), comm,
                             _stream(stream)))


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(LIB.squint_comm_unique_id(buf))
    return buf.raw


def comm_init(uid: bytes, rank: int, nranks: int):
    h = C.c_void_p()
    buf = C.create_string_buffer(uid, 128)
    _check(LIB.squint_comm_init(C.byref(h), buf, rank, nranks))
    return h


def comm_set_mode(h, mode: int):
    """0: ncclAllReduce + replicated Adam; 1: peer-memory all-reduce fused with a sharded Adam (f1)."""
    _check(LIB.squint_comm_set_mode(h, int(mode)))


def comm_destroy(h):
    _check(LIB.squint_comm_destroy(h))


# ---- convenience: torch-owned learner state ----------------------------------------
class Learner:
    """Owns the flat fp32 state, optimizer moments, workspace and ring views for one
    rank.  All memory is torch-allocated on `device`; all math runs in libsquint."""

    def __init__(self, dims: dict, hp: dict, precision=FP32, device="cuda", utd=1):
        self.dims_d, self.hp_d = dict(dims), dict(hp)
        self.dims = make_dims(dims, precision)
        self.hp = make_hparams(hp)
        self.layout, self.gsizes = param_layout(self.dims)
        dev = torch.device(device)
        z = lambda n: torch.zeros(max(n, 1), dtype=torch.float32, device=dev)
        gc, ga, gal, gt = self.gsizes
        self.critic, self.target, self.actor = z(gc), z(gt), z(ga)
        self.log_alpha = z(1)
        self.m_critic, self.v_critic, self.m_actor, self.v_actor = z(gc), z(gc), z(ga), z(ga)
        self.m_alpha, self.v_alpha = z(1), z(1)
        self.step = torch.zeros(3, dtype=torch.int64, device=dev)
        self.workspace = torch.zeros(workspace_bytes(self.dims, utd), dtype=torch.uint8, device=dev)
        self.state = State(*[t.data_ptr() for t in (self.critic, self.target, self.actor, self.log_alpha,
                                                      self.m_critic, self.v_critic, self.m_actor, self.v_actor,
                                                      self.m_alpha, self.v_alpha, self.step)])
        self.comm = None

    def buffer(self, group):
        return {GROUP_CRITIC: self.critic, GROUP_ACTOR: self.actor, GROUP_TARGET: self.target,
                GROUP_ALPHA: self.log_alpha}[group]

    def view(self, group, name, which="param"):
        for g, n, off, shape in self.layout:
            if g == group and n == name:
                base = self.buffer(group) if which == "param" else getattr(self, f"{which}_{GROUP_NAMES[group]}")
                numel = 1
                for s in shape:
                    numel *= s
                return base[off:off + numel].view(*shape)
        raise KeyError((group, name))

    def load_values(self, values: dict):
        """values {(group_name, name): array} -> flat buffers (host->device copies)."""
        for g, n, off, shape in self.layout:
            key = (GROUP_NAMES[g], n)
            if key in values:
                t = torch.as_tensor(values[key], dtype=torch.float32).reshape(-1)
                self.buffer(g)[off:off + t.numel()].copy_(t)

    def load_adam(self, m: dict, v: dict, steps):
        for g, n, off, shape in self.layout:
            key = (GROUP_NAMES[g], n)
            if g in (GROUP_CRITIC, GROUP_ACTOR) and key in m:
                gname = GROUP_NAMES[g]
                getattr(self, f"m_{gname}")[off:off + int(torch.tensor(shape).prod())].copy_(
                    torch.as_tensor(m[key], dtype=torch.float32).reshape(-1))
                getattr(self, f"v_{gname}")[off:off + int(torch.tensor(shape).prod())].copy_(
                    torch.as_tensor(v[key], dtype=torch.float32).reshape(-1))
            if g == GROUP_ALPHA and key in m:
                self.m_alpha.copy_(torch.as_tensor(m[key], dtype=torch.float32).reshape(-1))
                self.v_alpha.copy_(torch.as_tensor(v[key], dtype=torch.float32).reshape(-1))
        self.step.copy_(torch.as_tensor(steps, dtype=torch.int64))

    def grad(self, group):
        off, nb = workspace_region(self.dims, "grad_critic" if group == GROUP_CRITIC else "grad_actor")
        return self.workspace[off:off + nb].view(torch.float32)

    def region(self, name):
        off, nb = workspace_region(self.dims, name)
        return self.workspace[off:off + nb].view(torch.float32)

    def region_u8(self, name):
        off, nb = workspace_region(self.dims, name)
        return self.workspace[off:off + nb]

    def update(self, replay: Replay, idx, shifts, eps, metrics, stream=None):
        squint_update(self.dims, self.hp, replay, idx, shifts, eps, self.state, metrics, self.workspace,
                      comm=self.comm, stream=stream)


def replay_from_tensors(R: dict) -> Replay:
    """R: dict of device tensors obs, next_obs, proprio, next_proprio, action, reward, done (+ size)."""
    return Replay(R["obs"].data_ptr(), R["next_obs"].data_ptr(), R["proprio"].data_ptr(),
                  R["next_proprio"].data_ptr(), R["action"].data_ptr(), R["reward"].data_ptr(),
                  R["done"].data_ptr(), R["obs"].shape[0], int(R.get("size", R["obs"].shape[0])))
