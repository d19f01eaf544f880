"""Multi-rank host logic on CPU (world size 2, gloo): frame sharding covers every frame once,
and the single all_gather of detections reproduces the 1-rank result bit for bit."""
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


def _worker(rank, world, port, n_frames, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids = cdist.shard_frames(n_frames, world, rank)
    local = cdist.to_global(_fake_detect(ids), ids)
    merged = cdist.gather_boxes(local)
    q.put((rank, merged.tobytes()))
    dist.destroy_process_group()


def test_shard_frames_partition():
    for n in (0, 1, 7, 32, 33):
        for world in (1, 2, 3, 8):
            parts = [cdist.shard_frames(n, world, r) for r in range(world)]
            allf = np.sort(np.concatenate(parts))
            assert np.array_equal(allf, np.arange(n))
    with pytest.raises(ValueError):
        cdist.shard_frames(4, 2, 2)


def test_gather_world2_equals_single_rank():
    n_frames, world = 13, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_frames, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    ids = np.arange(n_frames)
    ref = cdist.sort_boxes(cdist.to_global(_fake_detect(ids), ids))
    for r in range(world):
        got = np.frombuffer(results[r], dtype=BOX_DTYPE)
        assert np.array_equal(got, ref)
