"""CPU-side checks of the C ABI: the library loads, exports every symbol include/squint.h
declares, its parameter layout agrees with the oracle's independent spec, and the
host-side argument checks reject bad input before any launch (no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
import squint_inputs as SI

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = pytest.importorskip("paper_2602_21203_b200")
S = P.squint


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "squint.h")).read()
    return sorted(set(re.findall(r"SQUINT_API\s+[\w\s\*]+?\b(squint_\w+)\s*\(", txt)))


def test_exports_every_declared_symbol():
    syms = header_symbols()
    assert len(syms) >= 13
    for s in syms:
        assert hasattr(S.LIB, s), s
    assert sorted(S.EXPORTED) == syms


def test_version():
    assert b"sm_100a" in S.LIB.squint_version()


@pytest.mark.parametrize("cfg,kind", [("c0", 0), ("c2", 0), ("c3", 0), ("c0", 1), ("c2", 1)])
def test_layout_matches_oracle_specs(cfg, kind):
    d = SI.dims_of(cfg, critic_kind=kind)
    lay, gs = P.param_layout(P.make_dims(d))
    specs = O.param_specs(O.Dims(**d))
    gmap = {"critic": S.GROUP_CRITIC, "actor": S.GROUP_ACTOR, "alpha": S.GROUP_ALPHA, "target": S.GROUP_TARGET}
    got = {(g, n): shape for g, n, off, shape in lay}
    exp = {(gmap[g], n): tuple(shape) for g, n, shape, *_ in specs}
    assert got == exp
    # offsets: 32-float aligned, non-overlapping, inside the group
    for grp in range(4):
        ts = sorted((off, int(np.prod(shape))) for g, n, off, shape in lay if g == grp)
        end = 0
        for off, ne in ts:
            assert off % 32 == 0 and off >= end
            end = off + ne
        assert end <= gs[grp]


def test_layout_param_counts_match_survey():
    """SURVEY appendix A counts: c0 critic group 245,468, actor 126,178, target 235,324."""
    d = SI.dims_of("c0")
    lay, gs = P.param_layout(P.make_dims(d))
    cnt = {g: 0 for g in range(4)}
    for g, n, off, shape in lay:
        cnt[g] += int(np.prod(shape))
    assert cnt[S.GROUP_CRITIC] == 245468 and cnt[S.GROUP_ACTOR] == 126178 and cnt[S.GROUP_TARGET] == 235324


def test_target_offsets_mirror_critic():
    d = SI.dims_of("c2")
    lay, gs = P.param_layout(P.make_dims(d))
    crit = {n: off for g, n, off, s in lay if g == S.GROUP_CRITIC}
    tgt = {n: off for g, n, off, s in lay if g == S.GROUP_TARGET}
    enc_end = crit["critic.proj.w"]
    assert all(crit[n] - enc_end == o for n, o in tgt.items())
    assert gs[S.GROUP_CRITIC] - enc_end == gs[S.GROUP_TARGET]


def _status(fn, *a):
    return fn(*a)


def test_invalid_dims_rejected():
    d = SI.dims_of("c0")
    for k, v in [("n_atoms", 1), ("batch", 0), ("v_min", 20.0), ("critic_kind", 2)]:
        bad = dict(d, **{k: v})
        with pytest.raises(S.SquintError) as e:
            P.param_layout(P.make_dims(bad))
        assert e.value.status == 1
    # the scalar critic ignores the atom support (f3)
    P.param_layout(P.make_dims(dict(d, critic_kind=1, n_atoms=1, v_min=3.0, v_max=-3.0)))


def test_insert_shape_errors_before_launch():
    null = C.c_void_p(0)
    assert S.LIB.squint_insert(null, 4, 3, 130, 128, 8, null, null, 10, null) == 2  # ESHAPE
    assert S.LIB.squint_insert(null, -1, 3, 128, 128, 8, null, null, 10, null) == 1
    assert S.LIB.squint_insert(null, 4, 3, 128, 128, 0, null, null, 10, null) == 1
    assert S.LIB.squint_insert(null, 0, 3, 128, 128, 8, null, null, 10, null) == 0  # n == 0 no-op
    assert b"divisible" in S.LIB.squint_last_error() or True


def test_insert2_arg_errors():
    null, one = C.c_void_p(0), C.c_void_p(16)
    # ring2 without slots2 (and the reverse) is rejected even for n == 0
    assert S.LIB.squint_insert2(null, 0, 3, 128, 128, 8, null, null, null, one, 10, null) == 1
    assert S.LIB.squint_insert2(null, 0, 3, 128, 128, 8, null, null, one, null, 10, null) == 1
    assert S.LIB.squint_insert2(null, 4, 3, 130, 128, 8, null, null, null, null, 10, null) == 2
    assert S.LIB.squint_insert2(null, 0, 3, 128, 128, 8, null, null, null, null, 10, null) == 0


def test_insert_ex_arg_errors():
    null, one = C.c_void_p(0), C.c_void_p(16)
    f = S.LIB.squint_insert_ex
    assert f(null, 0, 3, 128, 128, 8, 2, null, null, null, null, null, 10, null) == 1      # unknown layout
    assert f(null, 0, 4, 128, 128, 8, 0, one, null, null, null, null, 10, null) == 1      # jitter needs c == 3
    assert f(null, 0, 3, 130, 128, 8, 1, null, null, null, null, null, 10, null) == 2
    assert f(null, 0, 8, 128, 128, 8, 1, null, null, null, null, null, 10, null) == 5     # c > 4 unsupported
    assert f(null, 0, 3, 512, 512, 8, 1, null, null, null, null, null, 10, null) == 5     # > 200 KB per frame
    assert f(null, 0, 3, 128, 128, 8, 1, null, null, null, null, one, 10, null) == 1      # ring2 without slots2
    assert f(null, 0, 3, 128, 128, 8, 1, one, null, null, null, null, 10, null) == 0      # n == 0 no-op


def test_stage_pinned_rejects_pageable_host_memory():
    buf = (C.c_uint8 * 64)()
    assert S.LIB.squint_stage_pinned(C.c_void_p(16), C.cast(buf, C.c_void_p), 64, None) == 1
    assert S.LIB.squint_stage_pinned(None, None, 0, None) == 0


def test_soft_update_arg_errors():
    null = C.c_void_p(0)
    assert S.LIB.squint_soft_update(null, null, 10, 1.5, null) == 1
    assert S.LIB.squint_soft_update(null, null, -1, 0.5, null) == 1
    assert S.LIB.squint_soft_update(null, null, 0, 0.5, null) == 0


def test_update_arg_errors():
    d = P.make_dims(SI.dims_of("c0"))
    hp = P.make_hparams(SI.hp_of("c0"))
    rep = S.Replay()
    st = S.State()
    null = C.c_void_p(0)
    # utd < 1
    assert S.LIB.squint_update(C.byref(d), C.byref(hp), C.byref(rep), null, null, null, 0, C.byref(st), null, null,
                               0, null, null) == 1
    # empty replay
    rep.size = 0
    rep.capacity = 10
    assert S.LIB.squint_update(C.byref(d), C.byref(hp), C.byref(rep), null, null, null, 1, C.byref(st), null, null,
                               0, null, null) == 1
    assert b"empty" in S.LIB.squint_last_error()
    # gamma out of range
    hp2 = P.make_hparams(dict(SI.hp_of("c0"), gamma=1.5))
    rep.size = 10
    assert S.LIB.squint_update(C.byref(d), C.byref(hp2), C.byref(rep), null, null, null, 1, C.byref(st), null,
                               null, 0, null, null) == 1


def test_act_arg_errors():
    d = P.make_dims(SI.dims_of("c0"))
    hp = P.make_hparams(SI.hp_of("c0"))
    null = C.c_void_p(0)
    # frame size not a multiple of 16
    assert S.LIB.squint_act(C.byref(d), C.byref(hp), null, null, null, 4, 120, 120, null, null, null, null, null,
                            null, 0, null, null) == 2
    assert S.LIB.squint_act(C.byref(d), C.byref(hp), null, null, null, 0, 128, 128, null, null, null, null, null,
                            null, 0, null, null) == 0


def test_workspace_sizes_positive():
    for cfg in ("c0", "c2", "c3"):
        d = P.make_dims(SI.dims_of(cfg))
        assert P.workspace_bytes(d) > 0
        assert P.act_workspace_bytes(d, 4096) > 0
