"""Streaming stress (SURVEY §5 race detection): 100 seeded batches through ccnn_submit /
ccnn_collect with three batches in flight (the overlapped pyramid / stage-1 / tail streams and
the per-slot buffers of runtime.cu) must equal the synchronous ccnn_detect of each batch, bit
for bit; batch shapes change every few batches (replans while batches are in flight), and host
and device frames alternate.  Also run under compute-sanitizer (tools/profile_round.sh)."""
import numpy as np
import pytest

from synth import arch, configs, frames as synth_frames, weights

pytestmark = pytest.mark.gpu

SHAPES = [(320, 240), (333, 257), (320, 240), (640, 360)]


def _batch(seed):
    w, h = SHAPES[(seed // 7) % len(SHAPES)]
    n = 1 + seed % 3
    return synth_frames.make_video(n, w, h, configs.FRAME_SEED + 104729 * seed, 24)


def test_streamed_equals_synchronous_100_seeds():
    import torch
    from paper_1508_01292_b200 import Detector
    c = configs.C1
    T1, T2 = c.thresholds()
    # a low T1 so the selective unit and NMS see real work on every batch
    det = Detector(arch.NETS, weights.make_cascade_weights(), T1 - 0.35, T2, c.Tnn, c.rule,
                   max_w=640, max_h=360, max_batch=4, queue_capacity=8192)
    batches = [_batch(s) for s in range(100)]
    ref = [det.detect(b, 24, 1.2) for b in batches]
    assert sum(len(r) for r in ref) > 100
    inputs = [torch.from_numpy(b).cuda() if k % 2 else torch.from_numpy(b).pin_memory()
              for k, b in enumerate(batches)]
    got = []
    det.submit(inputs[0], 24, 1.2)
    det.submit(inputs[1], 24, 1.2)
    for k in range(2, len(inputs)):
        det.submit(inputs[k], 24, 1.2)
        got.append(det.collect())
    got.append(det.collect())
    got.append(det.collect())
    for k, (g, r) in enumerate(zip(got, ref)):
        assert np.array_equal(g, r), k
    det.close()
