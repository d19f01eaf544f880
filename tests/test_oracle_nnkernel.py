"""Pins for the oracle's nnkernel (§3.1, Eq. 1; SPEC nnkernel S:41-101).

Each test checks the oracle against something other than itself: libm tanh, scipy's
correlate2d, torch's conv2d / max_pool2d, numpy reductions, or numbers the paper
prints (tests/golden/paper_fixtures.json).
"""
import numpy as np
import pytest
import scipy.signal

import oracle
from synth import arch

RNG = np.random.default_rng(1234)


def test_activation_bound_vs_libm_tanh(golden):
    # relative error of the approximation <= 1.8%; S:49 protocol.
    x = np.arange(-20000, 20001) * 1e-3
    x = x[x != 0]
    f = oracle.activation(x)
    exact = 1.7159 * np.tanh(2.0 * x / 3.0)
    rel = np.abs(f - exact) / np.abs(exact)
    assert rel.max() <= golden["activation_max_rel_error"]["value"]
    # and the bound is nearly attained (a dropped y^4 or y^2 term would break one side)
    assert rel.max() > 0.015


def test_activation_special_values(golden):
    a = golden["activation_scale"]["value"]
    assert oracle.activation(0.0) == 0.0
    assert abs(oracle.activation(1e6) - a) < 1e-12             # S:48 asymptotes
    assert abs(oracle.activation(-1e6) + a) < 1e-12
    x = RNG.normal(size=2000) * 3
    assert np.array_equal(oracle.activation(-x), -oracle.activation(x))   # S:99 odd
    xs = np.linspace(-10, 10, 20001)
    assert np.all(np.diff(oracle.activation(xs)) > 0)          # monotone
    # small-x slope: f'(0) = 1.7159 * 2/3 (tanh'(0) = 1 and the approx has slope 1 at 0)
    h = 1e-7
    assert abs(oracle.activation(h) / h - 1.7159 * 2 / 3) < 1e-5


def test_conv_fixtures():
    # S:65 all-ones 3x3 with 2x2 ones kernel -> 2x2 of 4s
    out = oracle.conv2d_valid(np.ones((1, 3, 3)), np.ones((1, 1, 2, 2)), np.zeros(1))
    assert out.shape == (1, 2, 2) and np.all(out == 4.0)
    # S:66 identity 1x1 kernel
    x = RNG.normal(size=(1, 7, 5))
    out = oracle.conv2d_valid(x, np.ones((1, 1, 1, 1)), np.zeros(1))
    assert np.array_equal(out, x)
    with pytest.raises(ValueError):
        oracle.conv2d_valid(np.ones((1, 2, 2)), np.ones((1, 1, 3, 3)), np.zeros(1))


def test_conv_vs_scipy_correlate2d():
    # multi-map random input vs a library cross-correlation (no kernel flip).
    for (ni, no, h, w, kh, kw) in [(2, 3, 6, 7, 4, 3), (6, 2, 12, 10, 6, 5), (1, 6, 31, 27, 4, 4)]:
        x = RNG.normal(size=(ni, h, w))
        k = RNG.normal(size=(no, ni, kh, kw)).astype(np.float32)
        b = RNG.normal(size=no).astype(np.float32)
        got = oracle.conv2d_valid(x, k, b)
        ref = np.stack([sum(scipy.signal.correlate2d(x[i], k[o, i].astype(np.float64), "valid")
                            for i in range(ni)) + np.float64(b[o]) for o in range(no)])
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


def test_pool_fixtures():
    c = np.full((2, 4, 4), 3.25)
    assert np.array_equal(oracle.pool2(c), np.full((2, 2, 2), 3.25))
    assert oracle.pool2(RNG.normal(size=(1, 5, 5))).shape == (1, 2, 2)  # S:75 floor
    x = RNG.normal(size=(3, 6, 8))                                       # S:76 vs numpy
    ref = x.reshape(3, 3, 2, 4, 2).max(axis=(2, 4))
    assert np.array_equal(oracle.pool2(x), ref)
    x = RNG.normal(size=(3, 7, 9))
    ref = x[:, :6, :8].reshape(3, 3, 2, 4, 2).max(axis=(2, 4))
    assert np.array_equal(oracle.pool2(x), ref)


def _torch_forward(layers, w, plane):
    """Library forward: torch conv2d / max_pool2d in float64, weights in S:186 layout.
    The activation is applied through oracle.activation (pinned separately above)."""
    import torch
    import torch.nn.functional as F
    x = torch.from_numpy(np.asarray(plane, np.float64))[None, None]
    pos = 0
    for kind, i, o, kw, kh in layers:
        if kind == arch.CONV:
            n = o * i * kh * kw
            k = torch.from_numpy(w[pos:pos + n].astype(np.float64).reshape(o, i, kh, kw))
            b = torch.from_numpy(w[pos + n:pos + n + o].astype(np.float64))
            pos += n + o
            x = F.conv2d(x, k, b)
            x = torch.from_numpy(oracle.activation(x.numpy()))
        else:
            x = F.max_pool2d(x, 2, 2)
    return x[0].numpy()


@pytest.mark.parametrize("net_idx,shape", [(0, (31, 27)), (0, (47, 39)), (1, (55, 51)),
                                           (2, (55, 51)), (1, (63, 60))])
def test_forward_vs_torch(cascade, net_idx, shape):
    layers = arch.NETS[net_idx]
    w = cascade.nets[net_idx].w
    plane = RNG.uniform(-1, 1, size=shape)
    got = oracle.forward(cascade.nets[net_idx], plane)
    ref = _torch_forward(layers, w, plane)
    assert got.shape == ref.shape
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


def test_geometry_and_param_counts(cascade, golden):
    pc = golden["param_counts"]["value"]
    assert [oracle.param_count(n) for n in cascade.nets] == pc
    assert oracle.receptive_field(cascade.nets[0]) == tuple(golden["stage1_window"]["value"])
    assert oracle.output_stride(cascade.nets[0]) == golden["stage1_step"]["value"]
    pw, ph = golden["selective_patch"]["value"]
    mw, mh = golden["selective_map"]["value"]
    for n in cascade.nets[1:]:
        out = oracle.forward(n, np.zeros((ph, pw)))
        assert out.shape == (1, mh, mw)
    out = oracle.forward(cascade.nets[0], np.zeros((31, 27)))
    assert out.shape == (1, 1, 1)
    for kx, ky in [(0, 0), (1, 0), (0, 3), (5, 2)]:
        out = oracle.forward(cascade.nets[0], np.zeros((31 + 4 * ky, 27 + 4 * kx)))
        assert out.shape == (1, ky + 1, kx + 1)
    with pytest.raises(ValueError):
        oracle.forward(cascade.nets[0], np.zeros((30, 27)))


def test_conv_linearity():
    # conv(aX + bY) = a conv(X) + b conv(Y) with zero bias
    k = RNG.normal(size=(3, 2, 3, 4)).astype(np.float32)
    X, Y = RNG.normal(size=(2, 9, 8)), RNG.normal(size=(2, 9, 8))
    z = np.zeros(3, np.float32)
    lhs = oracle.conv2d_valid(2.5 * X - 0.75 * Y, k, z)
    rhs = 2.5 * oracle.conv2d_valid(X, k, z) - 0.75 * oracle.conv2d_valid(Y, k, z)
    np.testing.assert_allclose(lhs, rhs, rtol=1e-10, atol=1e-10)


def test_dense_equals_per_window(cascade):
    # S:97 / AC2: the dense scan at (i, j) equals the per-window forward at (4j, 4i).
    for trial in range(6):
        lh, lw = int(RNG.integers(31, 80)), int(RNG.integers(27, 80))
        level = RNG.integers(0, 256, size=(lh, lw), dtype=np.uint8)
        dense = oracle.stage1_dense(cascade.nets[0], level)
        nx, ny = oracle.window_grid(lw, lh)
        assert dense.shape == (ny, nx)
        for i in range(ny):
            for j in range(nx):
                assert dense[i, j] == oracle.stage1_window(cascade.nets[0], level, i, j)


def test_normalise_range():
    v = np.arange(256)
    x = oracle.normalise(v)
    assert x[0] == -1.0 and x[255] == 1.0 and np.all(np.diff(x) > 0)
