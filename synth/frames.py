"""Seeded synthetic grayscale frames (an input).

The paper's workloads are real video / FDDB / AFW images, which are OUT
of scope; these frames only reproduce their *shape*: resolution, 8-bit grayscale
(P:77), textured background, frontal-face-like blobs of the searched sizes, and a
cluttered variant.  Everything is integer arithmetic so host and device bytes are
identical by construction (SURVEY.md §8(d) "Synthetic inputs").

* background: 3 octaves of hash-lattice value noise, cells 64/16/4 px, integer
  bilinear interpolation, amplitude weights 5:3:2, contrast x3/2 about 128;
* faces: SPEC S:583 template -- bright oval, two dark eye blobs, dark mouth bar --
  at widths U[min_face, 4*min_face];
* video: one canvas per stream, frame f = canvas shifted by (2f, f) px;
* clutter: + octaves at 4 and 2 px with weight 0.6 and 300 extra templates.
"""
import numpy as np

_U32 = np.uint32


def _hash8(gx: np.ndarray, gy: np.ndarray, seed: int) -> np.ndarray:
    """32-bit integer hash of lattice coordinates -> 0..255 (int32)."""
    with np.errstate(over="ignore"):
        h = gx.astype(_U32) * _U32(0x8DA6B343) + gy.astype(_U32) * _U32(0xD8163841) \
            + _U32(seed & 0xFFFFFFFF) * _U32(0xCB1AB31F)
        h ^= h >> _U32(16)
        h *= _U32(0x7FEB352D)
        h ^= h >> _U32(15)
        h *= _U32(0x846CA68B)
        h ^= h >> _U32(16)
    return (h & _U32(0xFF)).astype(np.int32)


def value_noise(w: int, h: int, cell: int, seed: int) -> np.ndarray:
    """Integer value noise in 0..255, shape (h, w), int32."""
    xs = np.arange(w, dtype=np.int32)
    ys = np.arange(h, dtype=np.int32)
    gx, fx = xs // cell, xs % cell
    gy, fy = ys // cell, ys % cell
    nlx, nly = w // cell + 2, h // cell + 2
    lat = _hash8(np.arange(nlx)[None, :], np.arange(nly)[:, None], seed)  # (nly, nlx)
    # horizontal interpolation on every lattice row, kept at scale `cell`
    row = lat[:, gx] * (cell - fx)[None, :] + lat[:, gx + 1] * fx[None, :]  # (nly, w)
    v = row[gy, :] * (cell - fy)[:, None] + row[gy + 1, :] * fy[:, None]
    c2 = cell * cell
    return (v + c2 // 2) // c2


def background(w: int, h: int, seed: int, clutter: bool = False) -> np.ndarray:
    acc = 5 * (value_noise(w, h, 64, seed) - 128)
    acc += 3 * (value_noise(w, h, 16, seed + 1) - 128)
    acc += 2 * (value_noise(w, h, 4, seed + 2) - 128)
    if clutter:
        acc += 6 * (value_noise(w, h, 4, seed + 3) - 128)
        acc += 6 * (value_noise(w, h, 2, seed + 4) - 128)
    img = 128 + (acc * 3) // 20
    return np.clip(img, 0, 255).astype(np.int32)


def draw_face(img: np.ndarray, x: int, y: int, fw: int, contrast: int) -> None:
    """SPEC S:583 face template at top-left (x, y), width fw, height ~ 1.15 fw (in place)."""
    fh = (fw * 23) // 20
    H, W = img.shape
    x0, y0, x1, y1 = max(x, 0), max(y, 0), min(x + fw, W), min(y + fh, H)
    if x1 <= x0 or y1 <= y0:
        return
    yy, xx = np.mgrid[y0:y1, x0:x1]
    # coordinates relative to the template, scaled by 1000/fw and 1000/fh (integers)
    u = ((xx - x) * 2000 + 1000) // (2 * fw) - 500          # -500..500 across the width
    v = ((yy - y) * 2000 + 1000) // (2 * fh) - 500
    sub = img[y0:y1, x0:x1]
    oval = u * u + v * v <= 500 * 500
    sub[oval] = np.clip(sub[oval] + contrast, 0, 255)
    dark = max(contrast, 40)
    for ex in (-180, 180):                                  # eye blobs
        eye = (u - ex) ** 2 + (v + 120) ** 2 <= 90 * 90
        sub[eye] = np.clip(sub[eye] - dark, 0, 255)
    mouth = (np.abs(u) <= 200) & (np.abs(v - 230) <= 35)     # mouth bar
    sub[mouth] = np.clip(sub[mouth] - dark, 0, 255)


def plant_faces(img: np.ndarray, rng: np.random.Generator, n: int, min_face: int,
                max_face: int) -> list:
    H, W = img.shape
    boxes = []
    for _ in range(n):
        fw = int(rng.integers(min_face, max(min_face + 1, max_face + 1)))
        fh = (fw * 23) // 20
        if fw >= W or fh >= H:
            continue
        x = int(rng.integers(0, W - fw))
        y = int(rng.integers(0, H - fh))
        draw_face(img, x, y, fw, int(rng.integers(40, 110)))
        boxes.append((x, y, fw, fh))
    return boxes


def make_still_gt(w: int, h: int, seed: int, min_face: int, n_faces=None,
                  clutter: bool = False):
    """One synthetic grayscale frame, uint8 (h, w), and its planted faces as rectangles
    [(x, y, w, h)] (the ground truth of the NEXT #3 evaluation; clutter templates, when
    requested, are planted too and counted as faces)."""
    rng = np.random.default_rng(seed)
    img = background(w, h, seed, clutter)
    if n_faces is None:
        n_faces = int(rng.integers(1, 6))
    gt = plant_faces(img, rng, n_faces, min_face, 4 * min_face)
    if clutter:
        gt += plant_faces(img, rng, 300, max(8, min_face // 2), 4 * min_face)
    return img.astype(np.uint8), gt


def make_still(w: int, h: int, seed: int, min_face: int, n_faces=None,
               clutter: bool = False) -> np.ndarray:
    """One synthetic grayscale frame, uint8 (h, w)."""
    return make_still_gt(w, h, seed, min_face, n_faces, clutter)[0]


def make_video(n: int, w: int, h: int, seed: int, min_face: int, n_faces: int = 12,
               clutter: bool = False) -> np.ndarray:
    """n frames (n, h, w) uint8 of one stream: content translated by (2, 1) px per frame."""
    cw, ch = w + 2 * n, h + n
    canvas = make_still(cw, ch, seed, min_face, n_faces=n_faces, clutter=clutter)
    out = np.empty((n, h, w), np.uint8)
    for f in range(n):
        out[f] = canvas[f:f + h, 2 * f:2 * f + w]
    return out


def make_video_frames(indices, n_total: int, w: int, h: int, seed: int, min_face: int,
                      n_faces: int = 12, clutter: bool = False) -> np.ndarray:
    """Frames `indices` of the n_total-frame stream make_video(n_total, ...) would return
    (a rank's shard of a stream: identical bytes, without materialising the other frames)."""
    cw, ch = w + 2 * n_total, h + n_total
    canvas = make_still(cw, ch, seed, min_face, n_faces=n_faces, clutter=clutter)
    idx = [int(f) for f in indices]
    out = np.empty((len(idx), h, w), np.uint8)
    for k, f in enumerate(idx):
        if not 0 <= f < n_total:
            raise ValueError("frame index out of range")
        out[k] = canvas[f:f + h, 2 * f:2 * f + w]
    return out


def make_stills(n: int, w: int, h: int, seed: int, min_face: int) -> np.ndarray:
    return np.stack([make_still(w, h, seed + k, min_face) for k in range(n)])
