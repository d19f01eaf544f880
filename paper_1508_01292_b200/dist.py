"""Frame sharding and the final detection gather across ranks.

Video frames are independent (BASELINE.json north_star), so rank r of N owns the frames
f with f % N == r and runs ccnn_detect on them alone -- no collective on the data path.
After the last batch, ONE exchange: all_gather of the per-rank box counts, then of the
boxes padded to the largest count (NCCL over NVLink on GPUs, gloo on CPU for tests).
This module is host-side plumbing only; the detector arithmetic is in libccnn.so.
"""
import numpy as np

from .ccnn import BOX_DTYPE

_FIELDS = 7  # int32 words per box: frame, x, y, w, h, score (bits), neighbors


def shard_frames(n_frames: int, world: int, rank: int) -> np.ndarray:
    """Global frame indices owned by `rank` (round robin: f % world == rank)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return np.arange(rank, n_frames, world, dtype=np.int64)


def to_global(boxes: np.ndarray, frame_ids: np.ndarray) -> np.ndarray:
    """Rewrite the batch-local `frame` field of ccnn boxes to global frame ids."""
    out = boxes.copy()
    out["frame"] = np.asarray(frame_ids)[boxes["frame"]].astype(np.int32)
    return out


def sort_boxes(boxes: np.ndarray) -> np.ndarray:
    """The ABI's output order: (frame, score desc, y, x, w, h)."""
    if len(boxes) == 0:
        return boxes
    order = np.lexsort((boxes["h"], boxes["w"], boxes["x"], boxes["y"], -boxes["score"],
                        boxes["frame"]))
    return boxes[order]


def gather_boxes(boxes: np.ndarray, device=None, group=None) -> np.ndarray:
    """all_gather every rank's boxes (global frame ids) and return the merged, sorted set
    on every rank.  Two collectives: counts, then boxes padded to the maximum count."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    boxes = np.ascontiguousarray(boxes, BOX_DTYPE)
    words = boxes.view(np.int32).reshape(-1, _FIELDS)
    dev = torch.device("cpu") if device is None else device
    cnt = torch.tensor([words.shape[0]], dtype=torch.int64, device=dev)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    counts = [int(c.item()) for c in cnts]
    mx = max(1, max(counts))
    pad = torch.zeros((mx, _FIELDS), dtype=torch.int32, device=dev)
    if words.shape[0]:
        pad[:words.shape[0]] = torch.from_numpy(words).to(dev)
    gathered = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(gathered, pad, group=group)
    parts = [g[:c].cpu().numpy() for g, c in zip(gathered, counts)]
    merged = np.ascontiguousarray(np.concatenate(parts, axis=0), np.int32)
    return sort_boxes(merged.view(BOX_DTYPE).reshape(-1))
