"""Pins for the oracle's f4 insert variants: colour jitter before the squint
(reading R-jit in DESIGN.md §3) and HWC frames.  Every
expected value below is a closed form or a special case, not a re-run of the oracle."""
import numpy as np
import pytest

import oracle as O
import squint_inputs as SI


def _one(img, b, c, s):
    return O.color_jitter(img[None], np.array([[b, c, s]], np.float32))[0]


def _grey_image(levels):
    """u8 [3, H, W] with R = G = B = levels."""
    return np.repeat(np.asarray(levels, np.uint8)[None], 3, axis=0)


def test_identity_is_bitwise_noop_spec61_spec78():
    f = SI.make_frames(4, 64, seed=3)
    assert np.array_equal(O.color_jitter(f, np.ones((4, 3), np.float32)), f)


@pytest.mark.parametrize("b", [0.5, 1.7, 3.0])
def test_zero_image_stays_zero_spec62(b):
    z = np.zeros((3, 32, 32), np.uint8)
    assert not _one(z, b, 1.0, 1.0).any()


def test_brightness_closed_forms():
    x = np.arange(256, dtype=np.uint8).reshape(1, 16, 16).repeat(3, axis=0)
    assert np.array_equal(_one(x, 0.5, 1, 1), x // 2)                            # floor(x / 2)
    assert np.array_equal(_one(x, 2.0, 1, 1), np.minimum(2 * x.astype(int), 255))  # clamp at 255
    assert np.array_equal(_one(x, 0.25, 1, 1), x // 4)


def test_contrast_zero_gives_mean_grey():
    # grey image levels v: grey(v) = floor(0.9999 v) = v - 1 for 1 <= v <= 255, 0 for v = 0;
    # c = 0 replaces every value by u8(m), m = mean grey (256 pixels: exact division)
    rng = np.random.default_rng(0)
    v = rng.integers(0, 256, (16, 16))
    img = _grey_image(v)
    m_num = int(np.maximum(v - 1, 0).sum())
    out = _one(img, 1.0, 0.0, 1.0)
    assert (out == m_num // 256).all()


def test_contrast_two_closed_form():
    # half the pixels at 101, half at 201 (greys 100 and 200, m = 150): x2 = 2 x - 150
    v = np.full((16, 16), 101)
    v[8:] = 201
    out = _one(_grey_image(v), 1.0, 2.0, 1.0)
    assert (out[:, :8] == 52).all() and (out[:, 8:] == 252).all()


def test_saturation_zero_gives_truncated_luma():
    img = np.zeros((3, 4, 4), np.uint8)
    img[0, 0, 0] = 100  # red 100   -> floor(29.89) = 29
    img[1, 0, 1] = 100  # green 100 -> floor(58.7)  = 58
    img[2, 0, 2] = 100  # blue 100  -> floor(11.4)  = 11
    out = _one(img, 1.0, 1.0, 0.0)
    for k, g in ((0, 29), (1, 58), (2, 11)):
        assert (out[:, 0, k] == g).all()
    assert not out[:, 1:].any()


def test_saturation_two_closed_form():
    img = np.zeros((3, 2, 2), np.uint8)
    img[:, :, :] = np.array([100, 50, 50], np.uint8)[:, None, None]
    # grey = floor(29.89 + 29.35 + 5.7) = 64; x3 = u8(2 x - 64)
    out = _one(img, 1.0, 1.0, 2.0)
    assert (out[0] == 136).all() and (out[1] == 36).all() and (out[2] == 36).all()


def test_order_brightness_before_contrast():
    # b = 0.5 then c = 0: mean grey of the halved image, not half the mean grey
    v = np.full((16, 16), 3)  # halved: 1 -> grey 0; the other order would give floor(2/2) = 1
    out = _one(_grey_image(v), 0.5, 0.0, 1.0)
    assert (out == 0).all()


def test_hwc_insert_matches_loops_on_chw():
    f = SI.make_frames(3, 32, seed=9)                       # CHW
    hwc = np.zeros((3, 32, 32, 3), np.uint8)
    for k in range(3):
        for y in range(32):
            for x in range(32):
                for ch in range(3):
                    hwc[k, y, x, ch] = f[k, ch, y, x]
    ring = np.zeros((5, 3, 4, 4), np.uint8)
    got = O.insert_ex(hwc, 8, [4, 0, 2], ring, hwc=True)
    for k, slot in enumerate([4, 0, 2]):
        assert np.array_equal(got[slot], O.area_downsample_loops(f[k], 8))
    assert not got[[1, 3]].any()


def test_jittered_insert_is_squint_of_jitter():
    f = SI.make_frames(2, 64, seed=4)
    jit = np.array([[1.0, 1.0, 1.0], [0.5, 1.0, 1.0]], np.float32)
    got = O.insert_ex(f, 8, [1, 0], np.zeros((2, 3, 8, 8), np.uint8), jitter=jit)
    assert np.array_equal(got[1], O.area_downsample_loops(f[0], 8))          # identity jitter
    assert np.array_equal(got[0], O.area_downsample_loops(f[1] // 2, 8))     # b = 0.5: floor(x/2)
