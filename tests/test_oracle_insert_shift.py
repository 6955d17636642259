"""Pins for the oracle's integer steps: squint (a1), shift (a4).  CPU only."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import squint_inputs as SI

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


def test_downsample_tie_spec43():
    g = GOLD["downsample_tie"]
    img = np.array(g["block"], np.uint8)[None, None]
    assert O.area_downsample(img, g["factor"])[0, 0, 0, 0] == g["expected"]


@pytest.mark.parametrize("block,exp", [([[0, 1], [0, 1]], 0),      # 0.5 -> 0 (even)
                                       ([[1, 2], [1, 2]], 2),      # 1.5 -> 2
                                       ([[2, 3], [2, 3]], 2),      # 2.5 -> 2
                                       ([[254, 255], [254, 255]], 254),  # 254.5 -> 254
                                       ([[0, 0], [0, 3]], 1)])     # 0.75 -> 1
def test_downsample_rhe_small(block, exp):
    img = np.array(block, np.uint8)[None, None]
    assert O.area_downsample(img, 2)[0, 0, 0, 0] == exp


@pytest.mark.parametrize("factor", [1, 2, 4, 8])
def test_downsample_constant_spec44(factor):
    for val in (0, GOLD["downsample_constant"]["value"], 128, 255):
        img = np.full((2, 3, 16 * factor, 16 * factor), val, np.uint8)
        out = O.area_downsample(img, factor)
        assert out.shape == (2, 3, 16, 16) and (out == val).all()


def test_downsample_rhe_exhaustive():
    """Every block sum of an 8x8 u8 block (0..16320): oracle == exact rational RHE
    (Python's round() on a Fraction is round-half-to-even)."""
    s = np.arange(0, 64 * 255 + 1)
    # build one 8x8 block per sum: spread s over 64 cells
    base = s // 64
    rem = s % 64
    blocks = np.repeat(base[:, None], 64, axis=1)
    blocks[np.arange(64)[None, :] < rem[:, None]] += 1
    img = blocks.reshape(-1, 1, 8, 8).astype(np.uint8)
    out = O.area_downsample(img, 8).reshape(-1)
    exp = np.array([round(Fraction(int(v), 64)) for v in s])
    assert (out == exp).all()


def test_downsample_vs_loops_spec45():
    frames = SI.make_frames(2, 128, seed=11)
    vec = O.area_downsample(frames, 8)
    for f in range(2):
        assert (vec[f] == O.area_downsample_loops(frames[f], 8)).all()
    odd = np.random.default_rng(5).integers(0, 256, (1, 3, 12, 12), dtype=np.uint8)
    assert (O.area_downsample(odd, 3)[0] == O.area_downsample_loops(odd[0], 3)).all()


def test_downsample_mean_preserving_spec75():
    frames = SI.make_frames(8, 128, seed=3)
    out = O.area_downsample(frames, 8)
    assert abs(out.astype(np.float64).mean() - frames.astype(np.float64).mean()) <= 0.5
    for f in range(8):
        assert abs(out[f].astype(float).mean() - frames[f].astype(float).mean()) <= 0.5


def test_downsample_composition_spec77():
    rng = np.random.default_rng(7)
    imgs = rng.integers(0, 256, (100, 3, 128, 128), dtype=np.uint8)
    a = O.area_downsample(imgs, 8).astype(int)
    b = O.area_downsample(O.area_downsample(imgs, 2), 4).astype(int)
    assert np.abs(a - b).max() <= 1


def test_downsample_shape_error_spec41():
    with pytest.raises(ValueError):
        O.area_downsample(np.zeros((1, 3, 130, 128), np.uint8), 8)


def test_insert_writes_only_slots():
    frames = SI.make_frames(16, 128, seed=1)
    ring = np.full((100, 3, 16, 16), 7, np.uint8)
    slots = SI.make_slots(16, 100, seed=9)
    out = O.insert(frames, 8, slots, ring)
    assert (out[slots] == O.area_downsample(frames, 8)).all()
    mask = np.ones(100, bool)
    mask[slots] = False
    assert (out[mask] == 7).all()


def test_normalize_spec52():
    g = GOLD["normalize"]
    got = O.normalize_pixels(np.array(g["in"], np.uint8))
    assert np.allclose(got, g["expected"], atol=g["tol"])


# ---- shift (a4) ---------------------------------------------------------------------
def test_shift_identity_at_pad():
    imgs = np.random.default_rng(0).integers(0, 256, (5, 3, 16, 16), dtype=np.uint8)
    p = 2
    out = O.shift_images(imgs, np.full(5, p), np.full(5, p), p)
    assert (out == imgs).all()


def test_shift_origin_replicates_edge():
    imgs = np.random.default_rng(1).integers(0, 256, (2, 3, 16, 16), dtype=np.uint8)
    out = O.shift_images(imgs, np.zeros(2, int), np.zeros(2, int), 2)
    # rows 0..2 all equal the top row of the source cropped/replicated the same way
    for y in range(3):
        assert (out[:, :, y, 2:] == imgs[:, :, 0, :14]).all()
    assert (out[:, :, 3:, 3:] == imgs[:, :, 1:14, 1:14]).all()


def test_shift_vs_edge_pad_crop():
    """Independent formulation: np.pad(mode='edge') then crop at (dy, dx)."""
    rng = np.random.default_rng(2)
    imgs = rng.integers(0, 256, (64, 3, 16, 16), dtype=np.uint8)
    dx, dy = rng.integers(0, 5, 64), rng.integers(0, 5, 64)
    out = O.shift_images(imgs, dx, dy, 2)
    padded = np.pad(imgs, ((0, 0), (0, 0), (2, 2), (2, 2)), mode="edge")
    for k in range(64):
        assert (out[k] == padded[k, :, dy[k]:dy[k] + 16, dx[k]:dx[k] + 16]).all()
