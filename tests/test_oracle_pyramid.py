"""Pins for the oracle's pyramid (SPEC pyramid S:225-246).

Checked against the SPEC worked example, the unit-scale special cases
(S:232-233), a closed-form level count, and scipy's double-precision
bilinear interpolation (map_coordinates, order 1).
"""
import math

import numpy as np
import pytest
import scipy.ndimage

import oracle

RNG = np.random.default_rng(77)


def test_spec_example(golden):
    ex = golden["pyramid_example"]
    lv = oracle.level_table(ex["W"], ex["H"], ex["min_face"], ex["scale_step"])
    assert len(lv) == ex["levels"]
    assert abs(lv[0][0] - ex["sigma0"]) < 1e-15
    assert abs(lv[-1][0] - ex["sigma_last_approx"]) / ex["sigma_last_approx"] < 2e-3
    assert (lv[-1][1], lv[-1][2]) == (48, 36)


def test_unit_scale_cases():
    lv = oracle.level_table(200, 150, 27, 1.2)
    assert lv[0] == (1.0, 200, 150)
    assert len(oracle.level_table(27, 31, 27, 1.1)) == 1
    assert len(oracle.level_table(26, 31, 27, 1.1)) == 0            # empty pyramid, not an error
    frame = RNG.integers(0, 256, size=(150, 200), dtype=np.uint8)
    assert np.array_equal(oracle.resample(frame, 1.0, 200, 150), frame)
    with pytest.raises(ValueError):
        oracle.level_table(100, 100, 0, 1.2)
    with pytest.raises(ValueError):
        oracle.level_table(100, 100, 20, 1.0)


def test_level_rules_and_closed_form():
    for _ in range(200):
        W, H = int(RNG.integers(27, 4000)), int(RNG.integers(31, 2500))
        mf = int(RNG.integers(10, 200))
        sf = float(np.float32(RNG.uniform(1.03, 1.6)))
        lv = oracle.level_table(W, H, mf, sf)
        s0 = 27.0 / mf
        # closed form (S:228 stop rule), skipped when the log lands within 1e-9 of an integer
        r = min(W * s0 / 27.0, H * s0 / 31.0)
        if r < 1:
            assert lv == []
            continue
        q = math.log(r) / math.log(sf)
        if abs(q - round(q)) > 1e-9:
            assert len(lv) == math.floor(q) + 1
        for k, (s, lw, lh) in enumerate(lv):
            assert lw == math.floor(W * s) and lh == math.floor(H * s)
            assert lw >= 27 and lh >= 31
            if k:
                assert abs(lv[k - 1][0] / s - sf) < 1e-12          # S:206 ratio
        # face-size coverage: every face width F in [minSize, largest window that fits]
        # is mapped by some level to within one scaleFactor ratio of the 27-px window
        sig = np.array([s for s, _, _ in lv])
        for F in np.linspace(mf, min(W, H * 27.0 / 31.0), 25):
            assert np.any((F * sig >= 27.0 / sf * (1 - 1e-12)) & (F * sig <= 27.0 * sf))


def test_resample_vs_scipy_bilinear():
    for _ in range(8):
        H, W = int(RNG.integers(20, 90)), int(RNG.integers(20, 90))
        frame = RNG.integers(0, 256, size=(H, W), dtype=np.uint8)
        sigma = float(RNG.uniform(0.3, 2.5))
        lw, lh = max(1, int(W * sigma)), max(1, int(H * sigma))
        got = oracle.resample(frame, sigma, lw, lh).astype(np.int32)
        xs = np.clip((np.arange(lw) + 0.5) / sigma - 0.5, 0, W - 1)
        ys = np.clip((np.arange(lh) + 0.5) / sigma - 0.5, 0, H - 1)
        yy, xx = np.meshgrid(ys, xs, indexing="ij")
        ref = scipy.ndimage.map_coordinates(frame.astype(np.float64), [yy, xx], order=1,
                                            mode="nearest")
        # O2 with round-half-up output and weights rounded to 1/2048: |error| <= 0.5 (final
        # rounding) + 2 axes x 255 x 2^-12 (a weight off by <= 1/4096 times a pixel step <= 255)
        assert np.max(np.abs(got - ref)) <= 0.5 + 2 * 255 * 2.0 ** -12


def test_resample_constant_and_range():
    frame = np.full((40, 50), 173, np.uint8)
    assert np.all(oracle.resample(frame, 0.7, 35, 28) == 173)
    assert np.all(oracle.resample(frame, 1.6, 80, 64) == 173)


def test_window_grid(golden):
    for lw, lh in [(27, 31), (30, 34), (31, 35), (1728, 972), (64, 36)]:
        nx, ny = oracle.window_grid(lw, lh)
        assert nx == (lw - 27) // 4 + 1 and ny == (lh - 31) // 4 + 1
    assert oracle.window_grid(26, 40) == (0, 0)


def test_to_gray_pins():
    """Reading I1: gray passthrough, SPEC's examples, and exact rational
    round-half-up of the Rec.601 luma on every tie and a random sample."""
    from fractions import Fraction
    g = np.arange(256, dtype=np.uint8).reshape(16, 16)
    assert np.array_equal(oracle.to_gray(g), g)
    px = np.array([[[255, 255, 255], [255, 0, 0], [0, 255, 0], [0, 0, 255], [0, 0, 0]]], np.uint8)
    assert oracle.to_gray(px).tolist() == [[255, 76, 150, 29, 0]]          # round(76.245) = 76
    # exact rational reference: floor(luma + 1/2)
    def ref(r, gg, b):
        v = Fraction(299, 1000) * r + Fraction(587, 1000) * gg + Fraction(114, 1000) * b
        return int(v + Fraction(1, 2))
    rng = np.random.default_rng(5)
    rgb = rng.integers(0, 256, (40, 50, 3)).astype(np.uint8)
    got = oracle.to_gray(rgb)
    for y in range(0, 40, 3):
        for x in range(50):
            assert got[y, x] == ref(*map(int, rgb[y, x]))
    # ties (luma exactly k + 1/2) round up
    ties = [(r, gg, b) for r in range(0, 256, 5) for gg in range(0, 256, 7) for b in range(0, 256, 11)
            if (299 * r + 587 * gg + 114 * b) % 1000 == 500][:200]
    assert ties
    a = np.array([ties], np.uint8)
    assert oracle.to_gray(a)[0].tolist() == [ref(*t) for t in ties]
