"""Multi-rank host logic (world size 2, gloo): frame sharding covers every frame once, and the
single all_gather of detections reproduces the 1-rank result bit for bit -- with fake
detections, with the oracle detector on CPU, and (-m gpu) with the CUDA detector of two ranks
sharing one GPU."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1508_01292_b200 import BOX_DTYPE, dist as cdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fake_detect(frame_ids):
    """Deterministic per-frame 'detections' standing in for ccnn_detect output (batch-local
    frame index, as the ABI returns it)."""
    out = []
    for k, f in enumerate(frame_ids):
        rng = np.random.default_rng(1000 + int(f))
        for _ in range(int(rng.integers(0, 4))):
            out.append((k, int(rng.integers(0, 3000)), int(rng.integers(0, 2000)), 60, 69,
                        float(np.float32(rng.normal())), int(rng.integers(1, 5))))
    return np.array(out, dtype=BOX_DTYPE)


# a small workload every detector finishes in a second: 6 stills 96 x 80, min face 24
_N, _W, _H, _MF, _SF = 6, 96, 80, 24, 1.2


def _frames():
    from synth import frames as sf
    return sf.make_stills(_N, _W, _H, 424242, _MF)


def _oracle_setup():
    import oracle
    from synth import arch, weights
    from tests import parity
    cas = oracle.Cascade(arch.NETS, weights.make_cascade_weights())
    fr = _frames()
    # thresholds low enough that every stage and NMS see work on these frames
    _, maps = parity.oracle_maps(cas, fr, _MF, _SF)
    allv = np.concatenate([m.ravel() for m in maps.values()])
    T1 = float(np.float32(np.quantile(allv, 0.9)))
    return cas, fr, T1, (0.3, 0.3)


def _as_abi_boxes(ob):
    """oracle boxes (score in fp64) -> the ABI's box layout (BOX_DTYPE, score fp32)."""
    out = np.zeros(len(ob), BOX_DTYPE)
    for k in ("frame", "x", "y", "w", "h", "neighbors"):
        out[k] = ob[k]
    out["score"] = ob["score"].astype(np.float32)
    return out


def _detect(kind, ids):
    if kind == "fake":
        return _fake_detect(ids)
    fr = _frames()[ids]
    if kind == "oracle":
        import oracle
        cas, _, T1, T2 = _oracle_setup()
        return _as_abi_boxes(oracle.detect(cas, fr, _MF, _SF, T1, T2, 1, 0)[1])
    from paper_1508_01292_b200 import Detector        # kind == "cuda": ranks share cuda:0
    from synth import arch, weights
    _, _, T1, T2 = _oracle_setup()
    det = Detector(arch.NETS, weights.make_cascade_weights(), T1, T2, 1, 0, max_w=_W, max_h=_H,
                   max_batch=_N, device=0)
    b = det.detect(fr, _MF, _SF) if len(ids) else np.zeros(0, BOX_DTYPE)
    det.close()
    return b


def _worker(rank, world, port, n_frames, q, kind="fake"):
    import sys
    import torch.distributed as dist
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids = cdist.shard_frames(n_frames, world, rank)
    local = cdist.to_global(_detect(kind, ids), ids)
    merged = cdist.gather_boxes(local)
    q.put((rank, merged.tobytes()))
    dist.destroy_process_group()


def _run_world2(n_frames, kind):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_frames, q, kind)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    return [np.frombuffer(results[r], dtype=BOX_DTYPE) for r in range(world)]


def test_shard_frames_partition():
    for n in (0, 1, 7, 32, 33):
        for world in (1, 2, 3, 8):
            parts = [cdist.shard_frames(n, world, r) for r in range(world)]
            allf = np.sort(np.concatenate(parts))
            assert np.array_equal(allf, np.arange(n))
    with pytest.raises(ValueError):
        cdist.shard_frames(4, 2, 2)


def test_gather_world2_equals_single_rank():
    n_frames = 13
    ids = np.arange(n_frames)
    ref = cdist.sort_boxes(cdist.to_global(_fake_detect(ids), ids))
    for got in _run_world2(n_frames, "fake"):
        assert np.array_equal(got, ref)


def test_gather_world2_oracle_detector():
    """Each rank runs the oracle detector on its frame shard; the gathered boxes equal the
    1-rank oracle detection of all frames."""
    ids = np.arange(_N)
    ref = cdist.sort_boxes(cdist.to_global(_detect("oracle", ids), ids))
    assert len(ref) > 0
    for got in _run_world2(_N, "oracle"):
        assert np.array_equal(got, ref)


@pytest.mark.gpu
def test_gather_world2_cuda_detector_shared_gpu():
    """Two ranks on one GPU (gloo), each with its own ccnn context on its frame shard: the
    gathered boxes equal one rank's detection of all frames, bit for bit."""
    ids = np.arange(_N)
    ref = cdist.sort_boxes(cdist.to_global(_detect("cuda", ids), ids))
    assert len(ref) > 0
    for got in _run_world2(_N, "cuda"):
        assert np.array_equal(got, ref)
