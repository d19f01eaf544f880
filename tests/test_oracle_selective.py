"""Pins for the oracle's selective unit (Eq. 2, Eq. 3).

Patch geometry is pinned with linear-ramp frames (bilinear sampling of a linear
function is exact up to the 11-bit weight rounding) against an independent
parameterisation of reading O5; equalisation, mirror and the decision rule against
the SPEC worked examples and properties; classify against its definition through
the torch-pinned forward pass.
"""
import numpy as np

import oracle

RNG = np.random.default_rng(99)


def _ramp_frames(W=230, H=240):
    fx = np.tile(np.arange(W, dtype=np.uint8), (H, 1))
    fy = np.tile(np.arange(H, dtype=np.uint8)[:, None], (1, W))
    return fx, fy


def test_patch_geometry_on_ramps():
    fx, fy = _ramp_frames()
    H, W = fx.shape
    for sigma, i, j in [(1.0, 20, 18), (0.8, 10, 12), (1.7, 40, 40), (0.55, 5, 6)]:
        px = oracle.extract_patch(fx, sigma, i, j).astype(np.float64)
        py = oracle.extract_patch(fy, sigma, i, j).astype(np.float64)
        assert px.shape == (55, 51)
        u = np.arange(51)
        v = np.arange(55)
        # the 27x31 window occupies the central 35x39 patch pixels (CNN2's receptive
        # field, P:91 5x5 map), i.e. patch pixel u spans window x = (u - 8) * 27/35
        X = (4 * j + (u - 8 + 0.5) * 27.0 / 35.0) / sigma - 0.5
        Y = (4 * i + (v - 8 + 0.5) * 31.0 / 39.0) / sigma - 0.5
        X = np.clip(X, 0, W - 1)
        Y = np.clip(Y, 0, H - 1)
        assert np.all(np.abs(px - X[None, :]) <= 0.5 + 2.0 ** -11 + 1e-9)
        assert np.all(np.abs(py - Y[:, None]) <= 0.5 + 2.0 ** -11 + 1e-9)


def test_patch_corner_replication_and_constant():
    fx, _ = _ramp_frames()
    p = oracle.extract_patch(fx, 1.0, 0, 0)
    assert np.all(p[:, :6] == 0)                  # S:300 replicated left edge
    const = np.full((100, 120), 77, np.uint8)
    assert np.all(oracle.extract_patch(const, 0.9, 3, 4) == 77)


def test_equalize_examples(golden):
    ramp = np.repeat(np.arange(256, dtype=np.uint8), 11)
    assert np.array_equal(oracle.equalize(ramp), ramp)
    c = np.full(2805, 93, np.uint8)
    assert np.array_equal(oracle.equalize(c), c)
    ex = golden["equalize_examples"]["two_valued"]
    img = np.array([ex["in"][0]] * 50 + [ex["in"][1]] * 50, np.uint8)
    out = oracle.equalize(img)
    assert sorted(set(out.tolist())) == ex["out"]
    assert np.all(out[:50] == ex["out"][0]) and np.all(out[50:] == ex["out"][1])


def test_equalize_properties():
    for _ in range(50):
        n = int(RNG.integers(2, 3000))
        img = RNG.integers(int(RNG.integers(0, 100)), int(RNG.integers(150, 256)), size=n,
                           dtype=np.uint8)
        if img.min() == img.max():
            continue
        out = oracle.equalize(img)
        order = np.argsort(img, kind="stable")
        assert np.all(np.diff(out[order].astype(int)) >= 0)       # monotone map
        assert out[img == img.min()].max() == 0 and out[img == img.max()].min() == 255
        # near-uniform CDF: out(v) within 0.5 of 255*(cdf-cmin)/(N-cmin)
        vals, counts = np.unique(img, return_counts=True)
        cdf = np.cumsum(counts)
        exact = 255.0 * (cdf - cdf[0]) / (n - cdf[0])
        got = np.array([out[img == v][0] for v in vals])
        assert np.all(np.abs(got - exact) <= 0.5)


def test_mirror():
    p = RNG.integers(0, 256, size=(55, 51), dtype=np.uint8)
    m = oracle.mirror(p)
    assert np.array_equal(oracle.mirror(m), p)
    assert np.array_equal(m, p[:, ::-1])
    sym = np.concatenate([p[:, :25], p[:, 25:26], p[:, :25][:, ::-1]], axis=1)
    assert np.array_equal(oracle.mirror(sym), sym)


def test_decision_rule_examples(golden):
    for c in golden["decision_examples"]["cases"]:
        assert oracle.decision(c["K2"], c["K3"], c["Tnn"], 0) == c["strict"]
        assert oracle.decision(c["K2"], c["K3"], c["Tnn"], 1) == c["weak"]


def test_decision_rule_exhaustive():
    # S:606 AC11: K2, K3 in [0, 50], T in [1, 5]; Eq. 2 and Eq. 3
    for T in range(1, 6):
        for K2 in range(51):
            for K3 in range(51):
                s = oracle.decision(K2, K3, T, 0)
                w = oracle.decision(K2, K3, T, 1)
                assert s == int((K2 >= T and K3 > 0) or (K2 > 0 and K3 >= T))
                assert w == int(K2 >= T or K3 >= T)
                if s:
                    assert w
                if T < 5:                                           # S:350 monotone in T
                    assert oracle.decision(K2, K3, T + 1, 0) <= s
                    assert oracle.decision(K2, K3, T + 1, 1) <= w
                if K2 == 0:
                    assert s == 0                                   # P:99 early stop is safe


def _K(r, T):
    return int(np.sum(r.astype(np.float32) > np.float32(T)))


def test_classify_definition_and_mirror_invariance(cascade):
    cnn2, cnn3 = cascade.nets[1], cascade.nets[2]
    for trial in range(12):
        patch = RNG.integers(0, 256, size=(55, 51), dtype=np.uint8)
        E = oracle.equalize(patch)
        r2 = np.concatenate([oracle.forward(cnn2, oracle.normalise(E))[0].ravel(),
                             oracle.forward(cnn2, oracle.normalise(E[:, ::-1]))[0].ravel()])
        r3 = np.concatenate([oracle.forward(cnn3, oracle.normalise(E))[0].ravel(),
                             oracle.forward(cnn3, oracle.normalise(E[:, ::-1]))[0].ravel()])
        T2 = (float(np.sort(r2)[-int(RNG.integers(1, 30))] - 1e-7),
              float(np.sort(r3)[-int(RNG.integers(1, 30))] - 1e-7))
        for rule in (0, 1):
            for Tnn in (1, 2, 3):
                p = oracle.make_params(0.0, T2, Tnn, rule)
                c = oracle.classify(cnn2, cnn3, patch, p)
                K2 = _K(r2, T2[0])
                assert c.K2 == K2
                assert np.allclose(np.array(c.r2[:]), r2, atol=0, rtol=0)
                if c.cnn3_ran:
                    assert c.K3 == _K(r3, T2[1])
                    assert c.delta == oracle.decision(K2, c.K3, Tnn, rule)
                    assert c.score == r3.max()
                else:
                    assert (rule == 0 and K2 == 0) or (rule == 1 and K2 >= Tnn)
                    assert c.delta == (1 if rule == 1 else 0)
                cm = oracle.classify(cnn2, cnn3, patch[:, ::-1].copy(), p)
                assert (cm.K2, cm.K3, cm.delta) == (c.K2, c.K3, c.delta)


def test_raw_box():
    assert oracle.raw_box(1.0, 3, 5) == (20, 12, 27, 31)           # sigma = 1: box = window
    x, y, w, h = oracle.raw_box(0.5, 3, 5)
    assert (x, y, w, h) == (40, 24, 54, 62)
    x, y, w, h = oracle.raw_box(27.0 / 60.0, 0, 1)                 # 4K level 0 (min face 60)
    assert (w, h) == (60, 69) and x == 9
