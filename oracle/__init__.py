"""CPU oracle of the compact CNN cascade hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1508_01292_b200``) never imports it and shares no code with it.

This module is argument marshalling over ``libccnn_oracle.so`` (plain C, fp64,
``-ffp-contract=off``; ``oracle/ccnn_oracle.c`` holds the arithmetic with its
PAPER.md citations).  Parity status of each function: DESIGN.md "Oracle pins".
"""
import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libccnn_oracle.so")
SRC = os.path.join(HERE, "ccnn_oracle.c")


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc -O2 -ffp-contract=off); idempotent."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "ccnn_oracle.h"))):
        tmp = LIB_PATH + ".tmp.%d" % os.getpid()
        subprocess.check_call(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-pthread", SRC, "-o", tmp, "-lm"])
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


class Layer(C.Structure):
    _fields_ = [("kind", C.c_int), ("in_maps", C.c_int), ("out_maps", C.c_int),
                ("kw", C.c_int), ("kh", C.c_int)]


class Net(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("layers", C.POINTER(Layer)),
                ("weights", C.POINTER(C.c_float))]


class Box(C.Structure):
    _fields_ = [("frame", C.c_int32), ("x", C.c_int32), ("y", C.c_int32), ("w", C.c_int32),
                ("h", C.c_int32), ("score", C.c_double), ("neighbors", C.c_int32)]


class Cand(C.Structure):
    _fields_ = [("frame", C.c_int32), ("level", C.c_int32), ("ix", C.c_int32), ("iy", C.c_int32),
                ("s1", C.c_double), ("K2", C.c_int32), ("K3", C.c_int32), ("delta", C.c_int32),
                ("cnn3_ran", C.c_int32), ("score", C.c_double), ("r2", C.c_double * 50),
                ("r3", C.c_double * 50), ("bx", C.c_int32), ("by", C.c_int32),
                ("bw", C.c_int32), ("bh", C.c_int32)]


class Params(C.Structure):
    _fields_ = [("T1", C.c_float), ("T2", C.c_float * 2), ("Tnn", C.c_int32),
                ("rule", C.c_int32), ("nms_min_cluster", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("windows", C.c_int64), ("stage1", C.c_int64), ("stage2", C.c_int64),
                ("stage3", C.c_int64), ("nms", C.c_int64)]


_lib = None
_P = C.POINTER


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        dp, fp, ip, u8p = _P(C.c_double), _P(C.c_float), _P(C.c_int), _P(C.c_uint8)
        L.or_activation.restype = C.c_double
        L.or_activation.argtypes = [C.c_double]
        L.or_conv2d_valid.argtypes = [dp, C.c_int, C.c_int, C.c_int, fp, fp, C.c_int, C.c_int,
                                      C.c_int, dp]
        L.or_pool2.argtypes = [dp, C.c_int, C.c_int, C.c_int, dp]
        L.or_param_count.restype = C.c_long
        L.or_param_count.argtypes = [_P(Net)]
        L.or_forward_shape.argtypes = [_P(Net), C.c_int, C.c_int, ip, ip, ip]
        L.or_forward.argtypes = [_P(Net), dp, C.c_int, C.c_int, dp, ip, ip, ip]
        L.or_receptive_field.argtypes = [_P(Net), ip, ip]
        L.or_output_stride.argtypes = [_P(Net)]
        L.or_level_table.argtypes = [C.c_int, C.c_int, C.c_int, C.c_float, C.c_int, C.c_int,
                                     C.c_int, dp, ip, ip]
        L.or_resample.argtypes = [u8p, C.c_int, C.c_int, C.c_long, C.c_double, C.c_int, C.c_int,
                                  u8p]
        L.or_to_gray.argtypes = [u8p, C.c_int, C.c_int, C.c_long, u8p]
        L.or_normalise.restype = C.c_double
        L.or_normalise.argtypes = [C.c_uint8]
        L.or_stage1_window.restype = C.c_double
        L.or_stage1_window.argtypes = [_P(Net), u8p, C.c_int, C.c_int, C.c_int, C.c_int]
        L.or_stage1_dense.argtypes = [_P(Net), u8p, C.c_int, C.c_int, dp]
        L.or_window_grid.argtypes = [C.c_int, C.c_int, ip, ip]
        L.or_extract_patch.argtypes = [u8p, C.c_int, C.c_int, C.c_long, C.c_double, C.c_int,
                                       C.c_int, u8p]
        L.or_equalize.argtypes = [u8p, C.c_int, u8p]
        L.or_mirror.argtypes = [u8p, C.c_int, C.c_int, u8p]
        L.or_decision.argtypes = [C.c_int] * 4
        L.or_classify.argtypes = [_P(Net), _P(Net), u8p, _P(Params), _P(Cand)]
        L.or_raw_box.argtypes = [C.c_double, C.c_int, C.c_int] + [_P(C.c_int32)] * 4
        L.or_iou_edge.argtypes = [_P(Box), _P(Box)]
        L.or_group.argtypes = [_P(Box), C.c_int, C.c_int, _P(Box)]
        L.or_detect.argtypes = [_P(Net), u8p, C.c_int, C.c_int, C.c_int, C.c_long, C.c_int,
                                C.c_float, _P(Params), C.c_int, C.c_int, _P(_P(Cand)),
                                _P(C.c_int64), _P(_P(Box)), _P(C.c_int64), _P(Stats)]
        L.or_free.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(_P(C.c_double))


def _u8(a):
    return a.ctypes.data_as(_P(C.c_uint8))


class OracleNet:
    """Keeps the ctypes layer array and weights alive alongside the Net struct."""

    def __init__(self, layers, weights):
        self.layer_arr = (Layer * len(layers))(*[Layer(*l) for l in layers])
        self.w = np.ascontiguousarray(weights, np.float32)
        self.net = Net(len(layers), self.layer_arr, self.w.ctypes.data_as(_P(C.c_float)))

    @property
    def ref(self):
        return C.byref(self.net)


def activation(x):
    x = np.asarray(x, np.float64)
    f = np.vectorize(lib().or_activation, otypes=[np.float64])
    return f(x)


def conv2d_valid(inp, kern, bias):
    """inp (in, h, w) f64, kern (out, in, kh, kw) f32, bias (out,) f32 -> (out, oh, ow)."""
    inp = np.ascontiguousarray(inp, np.float64)
    kern = np.ascontiguousarray(kern, np.float32)
    bias = np.ascontiguousarray(bias, np.float32)
    ni, h, w = inp.shape
    no, ni2, kh, kw = kern.shape
    assert ni == ni2
    out = np.empty((no, h - kh + 1, w - kw + 1), np.float64)
    rc = lib().or_conv2d_valid(_dp(inp), ni, w, h, kern.ctypes.data_as(_P(C.c_float)),
                               bias.ctypes.data_as(_P(C.c_float)), no, kw, kh, _dp(out))
    if rc != 0:
        raise ValueError("input smaller than kernel")
    return out


def pool2(inp):
    inp = np.ascontiguousarray(inp, np.float64)
    m, h, w = inp.shape
    out = np.empty((m, h // 2, w // 2), np.float64)
    lib().or_pool2(_dp(inp), m, w, h, _dp(out))
    return out


def forward(net: OracleNet, plane):
    plane = np.ascontiguousarray(plane, np.float64)
    h, w = plane.shape
    ow, oh, om = C.c_int(), C.c_int(), C.c_int()
    if lib().or_forward_shape(net.ref, w, h, C.byref(ow), C.byref(oh), C.byref(om)) != 0:
        raise ValueError("input smaller than receptive field")
    out = np.empty((om.value, oh.value, ow.value), np.float64)
    rc = lib().or_forward(net.ref, _dp(plane), w, h, _dp(out), C.byref(ow), C.byref(oh),
                          C.byref(om))
    if rc != 0:
        raise RuntimeError("or_forward failed %d" % rc)
    return out


def param_count(net: OracleNet) -> int:
    return lib().or_param_count(net.ref)


def receptive_field(net: OracleNet):
    rw, rh = C.c_int(), C.c_int()
    lib().or_receptive_field(net.ref, C.byref(rw), C.byref(rh))
    return rw.value, rh.value


def output_stride(net: OracleNet) -> int:
    return lib().or_output_stride(net.ref)


def level_table(W, H, min_face, scale_step, max_levels=512):
    sig = np.empty(max_levels, np.float64)
    lw = np.empty(max_levels, np.int32)
    lh = np.empty(max_levels, np.int32)
    n = lib().or_level_table(W, H, min_face, scale_step, 27, 31, max_levels, _dp(sig),
                             lw.ctypes.data_as(_P(C.c_int)), lh.ctypes.data_as(_P(C.c_int)))
    if n < 0:
        raise ValueError("bad pyramid arguments")
    return [(float(sig[k]), int(lw[k]), int(lh[k])) for k in range(n)]


def to_gray(img):
    """(h, w) uint8 -> itself; (h, w, 3) interleaved R,G,B -> Rec.601 luma (reading I1)."""
    img = np.ascontiguousarray(img, np.uint8)
    if img.ndim == 2:
        return img.copy()
    if img.ndim != 3 or img.shape[2] != 3:
        raise ValueError("expected (h, w) gray or (h, w, 3) RGB")
    h, w, _ = img.shape
    out = np.empty((h, w), np.uint8)
    lib().or_to_gray(_u8(img), w, h, 3 * w, _u8(out))
    return out


def resample(frame, sigma, lw, lh):
    frame = np.ascontiguousarray(frame, np.uint8)
    H, W = frame.shape
    out = np.empty((lh, lw), np.uint8)
    lib().or_resample(_u8(frame), W, H, W, sigma, lw, lh, _u8(out))
    return out


def normalise(v):
    return np.vectorize(lib().or_normalise, otypes=[np.float64])(np.asarray(v, np.uint8))


def window_grid(lw, lh):
    nx, ny = C.c_int(), C.c_int()
    lib().or_window_grid(lw, lh, C.byref(nx), C.byref(ny))
    return nx.value, ny.value


def stage1_window(cnn1: OracleNet, level, i, j):
    level = np.ascontiguousarray(level, np.uint8)
    lh, lw = level.shape
    return lib().or_stage1_window(cnn1.ref, _u8(level), lw, lh, i, j)


def stage1_dense(cnn1: OracleNet, level):
    level = np.ascontiguousarray(level, np.uint8)
    lh, lw = level.shape
    nx, ny = window_grid(lw, lh)
    out = np.empty((ny, nx), np.float64)
    if nx:
        rc = lib().or_stage1_dense(cnn1.ref, _u8(level), lw, lh, _dp(out))
        if rc != 0:
            raise RuntimeError("or_stage1_dense failed %d" % rc)
    return out


def extract_patch(frame, sigma, i, j):
    frame = np.ascontiguousarray(frame, np.uint8)
    H, W = frame.shape
    out = np.empty((55, 51), np.uint8)
    lib().or_extract_patch(_u8(frame), W, H, W, sigma, i, j, _u8(out))
    return out


def equalize(img):
    img = np.ascontiguousarray(img, np.uint8)
    out = np.empty_like(img)
    lib().or_equalize(_u8(img), img.size, _u8(out))
    return out


def mirror(img):
    img = np.ascontiguousarray(img, np.uint8)
    h, w = img.shape
    out = np.empty_like(img)
    lib().or_mirror(_u8(img), w, h, _u8(out))
    return out


def decision(K2, K3, Tnn, rule):
    return lib().or_decision(K2, K3, Tnn, rule)


def make_params(T1, T2, Tnn, rule, nms_min_cluster=1):
    return Params(T1, (C.c_float * 2)(*T2), Tnn, rule, nms_min_cluster)


def classify(cnn2: OracleNet, cnn3: OracleNet, patch, params: Params):
    patch = np.ascontiguousarray(patch, np.uint8)
    c = Cand()
    lib().or_classify(cnn2.ref, cnn3.ref, _u8(patch), C.byref(params), C.byref(c))
    return c


def raw_box(sigma, i, j):
    v = [C.c_int32() for _ in range(4)]
    lib().or_raw_box(sigma, i, j, *[C.byref(x) for x in v])
    return tuple(x.value for x in v)


def iou_edge(a, b):
    A = Box(0, *a[:4], 0.0, 1)
    B = Box(0, *b[:4], 0.0, 1)
    return bool(lib().or_iou_edge(C.byref(A), C.byref(B)))


def group(boxes, min_cluster=1):
    """boxes: iterable of (x, y, w, h, score) for one frame -> list of (x,y,w,h,score,neighbors)."""
    boxes = list(boxes)
    arr = (Box * max(1, len(boxes)))(*[Box(0, b[0], b[1], b[2], b[3], b[4], 1) for b in boxes])
    out = (Box * max(1, len(boxes)))()
    n = lib().or_group(arr, len(boxes), min_cluster, out)
    return [(o.x, o.y, o.w, o.h, o.score, o.neighbors) for o in out[:n]]


CAND_DTYPE = np.dtype([("frame", np.int32), ("level", np.int32), ("ix", np.int32),
                       ("iy", np.int32), ("s1", np.float64), ("K2", np.int32),
                       ("K3", np.int32), ("delta", np.int32), ("cnn3_ran", np.int32),
                       ("score", np.float64), ("r2", np.float64, (50,)),
                       ("r3", np.float64, (50,)), ("bx", np.int32), ("by", np.int32),
                       ("bw", np.int32), ("bh", np.int32)])
BOX_DTYPE = np.dtype([("frame", np.int32), ("x", np.int32), ("y", np.int32), ("w", np.int32),
                      ("h", np.int32), ("score", np.float64), ("neighbors", np.int32)],
                     align=True)


class Cascade:
    """The three nets (architecture + float32 weights) as the oracle sees them."""

    def __init__(self, layer_lists, weight_arrays):
        self.nets = [OracleNet(l, w) for l, w in zip(layer_lists, weight_arrays)]
        self.arr = (Net * 3)(*[n.net for n in self.nets])


def detect(cascade: Cascade, frames, min_face, scale_step, T1, T2, Tnn, rule,
           nms_min_cluster=1, dense=True, n_threads=0):
    """Full oracle pipeline over frames (n, H, W) uint8.

    Returns (candidates structured array, boxes structured array, stats dict)."""
    frames = np.ascontiguousarray(frames, np.uint8)
    if frames.ndim == 2:
        frames = frames[None]
    n, H, W = frames.shape
    p = make_params(T1, T2, Tnn, rule, nms_min_cluster)
    cp, bp = _P(Cand)(), _P(Box)()
    nc, nb = C.c_int64(), C.c_int64()
    st = Stats()
    rc = lib().or_detect(cascade.arr, _u8(frames), n, W, H, W, min_face, scale_step, C.byref(p),
                         1 if dense else 0, n_threads, C.byref(cp), C.byref(nc), C.byref(bp),
                         C.byref(nb), C.byref(st))
    if rc != 0:
        raise ValueError("or_detect failed %d" % rc)
    assert C.sizeof(Cand) == CAND_DTYPE.itemsize, (C.sizeof(Cand), CAND_DTYPE.itemsize)
    cands = np.frombuffer(C.string_at(cp, nc.value * C.sizeof(Cand)), CAND_DTYPE).copy() \
        if nc.value else np.zeros(0, CAND_DTYPE)
    assert C.sizeof(Box) == BOX_DTYPE.itemsize, (C.sizeof(Box), BOX_DTYPE.itemsize)
    boxes = np.frombuffer(C.string_at(bp, nb.value * C.sizeof(Box)), BOX_DTYPE).copy() \
        if nb.value else np.zeros(0, BOX_DTYPE)
    lib().or_free(cp)
    lib().or_free(bp)
    stats = dict(windows=st.windows, stage1=st.stage1, stage2=st.stage2, stage3=st.stage3,
                 nms=st.nms)
    return cands, boxes, stats
