"""Random-init weights for the three cascade CNNs (an input; §3.2 training is OUT).

Trained weights are unavailable (P:73-79 needs the YouTube Faces corpus), so both
the oracle and the CUDA path consume the same seeded random weights
(BASELINE.json north_star: "the networks use random-init weights of the paper's
architecture").

Recipe (DESIGN.md "Inputs" W1):
* generator: splitmix64 with state ``seed + net_index``; every float takes the top
  24 bits of one 64-bit output, u = bits / 2**24 in [0, 1);
* kernels: LeCun-uniform, w = (2u - 1) * sqrt(3 / fan_in), fan_in = in*kw*kh;
* biases:  (2u - 1) * 0.5 * sqrt(3 / fan_in)  -- non-zero so a dropped bias term
  fails parity (SURVEY suggested 0; changed on purpose, W1);
* order per conv layer: kernels [out][in][kh][kw], then bias[out] (SPEC S:186
  model-file order), layers concatenated; float32.
"""
import numpy as np

from . import arch

DEFAULT_SEED = 150801292

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(state: int, n: int) -> np.ndarray:
    """n successive splitmix64 outputs from ``state`` (uint64 wrap-around arithmetic)."""
    with np.errstate(over="ignore"):
        i = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(state & 0xFFFFFFFFFFFFFFFF) + i * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z & _M64


def uniform01(state: int, n: int) -> np.ndarray:
    """Top 24 bits of each splitmix64 output, as float64 in [0, 1)."""
    return (splitmix64(state, n) >> np.uint64(40)).astype(np.float64) / float(1 << 24)


def n_weights(net) -> int:
    """Number of float32 values the weight blob of ``net`` holds (sizing only)."""
    return sum(o * (i * kw * kh + 1) for k, i, o, kw, kh in net if k == arch.CONV)


def make_net_weights(net, seed: int) -> np.ndarray:
    u = uniform01(seed, n_weights(net))
    out = np.empty(u.shape, np.float32)
    pos = 0
    for kind, i, o, kw, kh in net:
        if kind != arch.CONV:
            continue
        fan_in = i * kw * kh
        lim = np.sqrt(3.0 / fan_in)
        nk = o * fan_in
        out[pos:pos + nk] = ((2.0 * u[pos:pos + nk] - 1.0) * lim).astype(np.float32)
        pos += nk
        out[pos:pos + o] = ((2.0 * u[pos:pos + o] - 1.0) * 0.5 * lim).astype(np.float32)
        pos += o
    assert pos == out.size
    return out


def make_cascade_weights(seed: int = DEFAULT_SEED):
    """(w_cnn1, w_cnn2, w_cnn3) as float32 arrays for architecture R."""
    return tuple(make_net_weights(net, seed + k) for k, net in enumerate(arch.NETS))


def checksum(ws) -> str:
    import hashlib
    h = hashlib.sha256()
    for w in ws:
        h.update(np.ascontiguousarray(w, np.float32).tobytes())
    return h.hexdigest()[:16]
