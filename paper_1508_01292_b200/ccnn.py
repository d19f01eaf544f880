"""Thin ctypes binding of libccnn.so (include/ccnn.h) -- argument marshalling only.

Every step of the detector runs in the library's sm_100a kernels; this module never
computes anything itself and has no fallback: if libccnn.so is missing or cannot be
loaded, importing it raises.  PyTorch is used only to hand over device pointers and
the current CUDA stream.
"""
import ctypes as C
import os

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libccnn.so")
if os.environ.get("CCNN_LIB_VARIANT"):      # experiments only: an in-tree variant build
    LIB_PATH = os.path.join(os.path.dirname(LIB_PATH), "libccnn_%s.so" % os.environ["CCNN_LIB_VARIANT"])

CCNN_OK, CCNN_E_ARG, CCNN_E_ARCH, CCNN_E_WEIGHTS = 0, -1, -2, -3
CCNN_E_CAPACITY, CCNN_E_QUEUE, CCNN_E_CUDA, CCNN_E_STATE = -4, -5, -6, -7
CCNN_DEBUG_LEVELS, CCNN_DEBUG_STAGE1, CCNN_DEBUG_PYR_TEX = 1, 2, 4

# every entry point declared in include/ccnn.h
EXPORTS = ("ccnn_create", "ccnn_set_stream", "ccnn_detect", "ccnn_detect_frames",
           "ccnn_submit", "ccnn_collect", "ccnn_submit_frames", "ccnn_last_boxes", "ccnn_destroy", "ccnn_last_error",
           "ccnn_abi_version", "ccnn_set_debug", "ccnn_debug_levels", "ccnn_debug_level",
           "ccnn_debug_stage1_map", "ccnn_debug_candidates", "ccnn_debug_counters", "ccnn_debug_group")


class CcnnError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("ccnn error %d: %s" % (code, msg))
        self.code = code


class Layer(C.Structure):
    _fields_ = [("kind", C.c_int32), ("in_maps", C.c_int32), ("out_maps", C.c_int32),
                ("kw", C.c_int32), ("kh", C.c_int32)]


class Net(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("layers", C.POINTER(Layer)),
                ("weights", C.POINTER(C.c_float)), ("n_weights", C.c_int64)]


class Params(C.Structure):
    _fields_ = [("net", Net * 3), ("T1", C.c_float), ("T2", C.c_float * 2), ("Tnn", C.c_int32),
                ("rule", C.c_int32), ("nms_min_cluster", C.c_int32), ("max_w", C.c_int32),
                ("max_h", C.c_int32), ("max_batch", C.c_int32), ("queue_capacity", C.c_int32),
                ("segment_rows", C.c_int32)]


class Box(C.Structure):
    _fields_ = [("frame", C.c_int32), ("x", C.c_int32), ("y", C.c_int32), ("w", C.c_int32),
                ("h", C.c_int32), ("score", C.c_float), ("neighbors", C.c_int32)]


class Frame(C.Structure):
    _fields_ = [("data", C.c_void_p), ("w", C.c_int32), ("h", C.c_int32), ("pitch", C.c_int64),
                ("channels", C.c_int32), ("reserved", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("windows", C.c_int64), ("stage1", C.c_int64), ("stage2", C.c_int64),
                ("stage3", C.c_int64), ("nms", C.c_int64), ("ms", C.c_float * 5),
                ("kernel_launches", C.c_int64), ("s1_mma_flops", C.c_double)]


class Candidate(C.Structure):
    _fields_ = [("frame", C.c_int32), ("level", C.c_int32), ("ix", C.c_int32), ("iy", C.c_int32),
                ("s1", C.c_float), ("K2", C.c_int32), ("K3", C.c_int32), ("delta", C.c_int32),
                ("cnn3_ran", C.c_int32), ("score", C.c_float), ("r2", C.c_float * 50),
                ("r3", C.c_float * 50), ("bx", C.c_int32), ("by", C.c_int32), ("bw", C.c_int32),
                ("bh", C.c_int32)]


BOX_DTYPE = np.dtype([("frame", np.int32), ("x", np.int32), ("y", np.int32), ("w", np.int32),
                      ("h", np.int32), ("score", np.float32), ("neighbors", np.int32)])
CAND_DTYPE = np.dtype([("frame", np.int32), ("level", np.int32), ("ix", np.int32),
                       ("iy", np.int32), ("s1", np.float32), ("K2", np.int32), ("K3", np.int32),
                       ("delta", np.int32), ("cnn3_ran", np.int32), ("score", np.float32),
                       ("r2", np.float32, (50,)), ("r3", np.float32, (50,)), ("bx", np.int32),
                       ("by", np.int32), ("bw", np.int32), ("bh", np.int32)])

_lib = None
_P = C.POINTER


def load():
    """Load libccnn.so and declare its signatures (raises if absent: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError("libccnn.so not built (run __graft_entry__.build()); no CPU fallback")
    L = C.CDLL(LIB_PATH)
    L.ccnn_create.argtypes = [_P(Params), C.c_int, _P(C.c_void_p)]
    L.ccnn_set_stream.argtypes = [C.c_void_p, C.c_void_p]
    L.ccnn_detect.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int64,
                              C.c_int, C.c_int, C.c_float, _P(Box), C.c_int64, _P(C.c_int64),
                              _P(Stats)]
    L.ccnn_detect_frames.argtypes = [C.c_void_p, _P(Frame), C.c_int, C.c_int, C.c_int, C.c_float,
                                     _P(Box), C.c_int64, _P(C.c_int64), _P(Stats)]
    L.ccnn_submit_frames.argtypes = [C.c_void_p, _P(Frame), C.c_int, C.c_int, C.c_int, C.c_float,
                                     C.c_int]
    L.ccnn_last_boxes.argtypes = [C.c_void_p, _P(Box), C.c_int64, _P(C.c_int64)]
    L.ccnn_submit.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int64,
                              C.c_int, C.c_int, C.c_float, C.c_int]
    L.ccnn_collect.argtypes = [C.c_void_p, _P(Box), C.c_int64, _P(C.c_int64), _P(Stats)]
    L.ccnn_destroy.argtypes = [C.c_void_p]
    L.ccnn_destroy.restype = None
    L.ccnn_last_error.argtypes = [C.c_void_p]
    L.ccnn_last_error.restype = C.c_char_p
    L.ccnn_abi_version.argtypes = []
    L.ccnn_set_debug.argtypes = [C.c_void_p, C.c_int]
    L.ccnn_debug_levels.argtypes = [C.c_void_p, C.c_int, _P(C.c_double), _P(C.c_int32), _P(C.c_int32),
                                    C.c_int]
    L.ccnn_debug_level.argtypes = [C.c_void_p, C.c_int, C.c_int, _P(C.c_uint8), C.c_int64]
    L.ccnn_debug_stage1_map.argtypes = [C.c_void_p, C.c_int, C.c_int, _P(C.c_float), C.c_int64]
    L.ccnn_debug_candidates.argtypes = [C.c_void_p, _P(Candidate), C.c_int64, _P(C.c_int64)]
    L.ccnn_debug_counters.argtypes = [C.c_void_p, _P(C.c_uint32), C.c_int]
    L.ccnn_debug_group.argtypes = [C.c_void_p, _P(Box), C.c_int64, C.c_int, _P(Box), C.c_int64,
                                   _P(C.c_int64)]
    _lib = L
    return L


class Detector:
    """One ccnn_ctx: ccnn_create(architecture, weights, thresholds) / ccnn_detect."""

    def __init__(self, layer_lists, weight_arrays, T1, T2, Tnn, rule=0, nms_min_cluster=1,
                 max_w=3840, max_h=2160, max_batch=64, queue_capacity=4096, segment_rows=0,
                 device=0):
        L = load()
        self._layers = [(Layer * len(ls))(*[Layer(*l) for l in ls]) for ls in layer_lists]
        self._w = [np.ascontiguousarray(w, np.float32) for w in weight_arrays]
        nets = (Net * 3)(*[Net(len(ls), self._layers[k], self._w[k].ctypes.data_as(_P(C.c_float)),
                               self._w[k].size) for k, ls in enumerate(layer_lists)])
        self.params = Params(nets, T1, (C.c_float * 2)(*T2), Tnn, rule, nms_min_cluster, max_w,
                             max_h, max_batch, queue_capacity, segment_rows)
        self.device = device
        h = C.c_void_p()
        rc = L.ccnn_create(C.byref(self.params), device, C.byref(h))
        if rc != CCNN_OK:
            raise CcnnError(rc, "ccnn_create failed")
        self.h = h
        self.last_stats = None
        self._cap = 1024
        self._inflight = []

    def close(self):
        if getattr(self, "h", None):
            load().ccnn_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != CCNN_OK:
            raise CcnnError(rc, load().ccnn_last_error(self.h).decode())

    def set_stream(self, stream_handle):
        self._check(load().ccnn_set_stream(self.h, C.c_void_p(stream_handle)))

    def set_debug(self, flags):
        self._check(load().ccnn_set_debug(self.h, flags))

    def _frames(self, frames, stream):
        """(ptr, n, H, W, pitch, on_device, keepalive) for a torch tensor or numpy array."""
        if hasattr(frames, "data_ptr"):                  # torch tensor
            import torch
            t = frames if frames.dim() == 3 else frames.unsqueeze(0)
            assert t.dtype == torch.uint8
            n, H, W = t.shape
            pitch = t.stride(1)
            assert t.stride(2) == 1 and t.stride(0) == H * pitch
            if t.is_cuda and stream is None:
                stream = torch.cuda.current_stream(t.device).cuda_stream
            return t.data_ptr(), n, H, W, pitch, 1 if t.is_cuda else 0, t, stream
        a = np.ascontiguousarray(frames, np.uint8)
        if a.ndim == 2:
            a = a[None]
        n, H, W = a.shape
        return a.ctypes.data, n, H, W, W, 0, a, stream

    def _result(self, rc, nb, st, box_cap, out):
        L = load()
        if rc == CCNN_E_CAPACITY and box_cap is None:      # fetch, do not detect again
            cap = int(nb.value)
            self._cap = max(self._cap, cap)
            out = np.zeros(cap, BOX_DTYPE)
            rc = L.ccnn_last_boxes(self.h, out.ctypes.data_as(_P(Box)), cap, C.byref(nb))
        self._check(rc)
        self.last_stats = dict(windows=st.windows, stage1=st.stage1, stage2=st.stage2,
                               stage3=st.stage3, nms=st.nms, ms=list(st.ms),
                               kernel_launches=st.kernel_launches, s1_mma_flops=st.s1_mma_flops)
        return out[:nb.value].copy()

    def detect(self, frames, min_face, scale_step, box_cap=None, stream=None):
        """frames: torch uint8 tensor (n, H, W) on the ctx device or on the host, or a numpy
        uint8 array (n, H, W).  Returns a numpy structured array of boxes (BOX_DTYPE)."""
        L = load()
        ptr, n, H, W, pitch, on_device, keep, stream = self._frames(frames, stream)
        if stream is not None:
            self.set_stream(stream)
        cap = box_cap if box_cap is not None else max(self._cap, 64 * n)
        nb = C.c_int64()
        st = Stats()
        out = np.zeros(cap, BOX_DTYPE)
        rc = L.ccnn_detect(self.h, C.c_void_p(ptr), n, W, H, pitch, on_device, min_face,
                           scale_step, out.ctypes.data_as(_P(Box)), cap, C.byref(nb), C.byref(st))
        res = self._result(rc, nb, st, box_cap, out)
        del keep
        return res

    def submit(self, frames, min_face, scale_step, stream=None, timed=True):
        """Enqueue one batch (ccnn_submit); the frames are kept alive until collect()."""
        L = load()
        ptr, n, H, W, pitch, on_device, keep, stream = self._frames(frames, stream)
        if stream is not None:
            self.set_stream(stream)
        self._check(L.ccnn_submit(self.h, C.c_void_p(ptr), n, W, H, pitch, on_device, min_face,
                                  scale_step, 1 if timed else 0))
        self._inflight.append((keep, n))

    def _frame_list(self, frames, stream):
        """ccnn_frame array for a list of uint8 images of individual sizes -- (h, w) gray or
        (h, w, 3) interleaved R,G,B -- numpy arrays or torch tensors, all on the host or all
        on the ctx device."""
        if len(frames) == 0:
            raise ValueError("empty frame list")
        keep, descs, dev = [], [], set()
        for f in frames:
            if hasattr(f, "data_ptr"):
                import torch
                assert f.dtype == torch.uint8 and f.dim() in (2, 3)
                ch = 1 if f.dim() == 2 else f.shape[2]
                assert (f.stride(1) == 1) if ch == 1 else (f.stride(2) == 1 and f.stride(1) == ch)
                if f.is_cuda and stream is None:
                    stream = torch.cuda.current_stream(f.device).cuda_stream
                dev.add(bool(f.is_cuda))
                keep.append(f)
                descs.append(Frame(f.data_ptr(), f.shape[1], f.shape[0], f.stride(0), ch, 0))
            else:
                a = np.asarray(f)
                ch = 1 if a.ndim == 2 else a.shape[2]
                ok = a.dtype == np.uint8 and a.ndim in (2, 3) and \
                    ((a.strides[1] == 1) if a.ndim == 2 else (a.strides[2] == 1 and a.strides[1] == ch))
                if not ok:
                    a = np.ascontiguousarray(a, np.uint8)
                dev.add(False)
                keep.append(a)
                descs.append(Frame(a.ctypes.data, a.shape[1], a.shape[0], a.strides[0], ch, 0))
        if len(dev) != 1:
            raise ValueError("frames must be all on the host or all on the device")
        arr = (Frame * len(descs))(*descs)
        return arr, len(descs), 1 if dev.pop() else 0, keep, stream

    def detect_frames(self, frames, min_face, scale_step, box_cap=None, stream=None):
        """ccnn_detect_frames: a list of 2-D uint8 frames of individual sizes.  box.frame
        indexes the list."""
        L = load()
        arr, n, on_device, keep, stream = self._frame_list(frames, stream)
        if stream is not None:
            self.set_stream(stream)
        cap = box_cap if box_cap is not None else max(self._cap, 64 * n)
        nb = C.c_int64()
        st = Stats()
        out = np.zeros(cap, BOX_DTYPE)
        rc = L.ccnn_detect_frames(self.h, arr, n, on_device, min_face, scale_step,
                                  out.ctypes.data_as(_P(Box)), cap, C.byref(nb), C.byref(st))
        res = self._result(rc, nb, st, box_cap, out)
        del keep
        return res

    def submit_frames(self, frames, min_face, scale_step, stream=None, timed=True):
        """Enqueue a list of frames of individual sizes (ccnn_submit_frames)."""
        L = load()
        arr, n, on_device, keep, stream = self._frame_list(frames, stream)
        if stream is not None:
            self.set_stream(stream)
        self._check(L.ccnn_submit_frames(self.h, arr, n, on_device, min_face, scale_step,
                                         1 if timed else 0))
        self._inflight.append((keep, n))

    def collect(self, box_cap=None):
        """Boxes of the oldest submitted batch (ccnn_collect)."""
        L = load()
        keep, n = self._inflight[0]
        cap = box_cap if box_cap is not None else max(self._cap, 64 * n)
        nb = C.c_int64()
        st = Stats()
        out = np.zeros(cap, BOX_DTYPE)
        rc = L.ccnn_collect(self.h, out.ctypes.data_as(_P(Box)), cap, C.byref(nb), C.byref(st))
        self._inflight.pop(0)
        return self._result(rc, nb, st, box_cap, out)

    # ---- test hooks ----
    def levels(self, frame=0):
        """(sigma, lw, lh) of every level of `frame` of the last submitted batch."""
        L = load()
        n = L.ccnn_debug_levels(self.h, frame, None, None, None, 0)
        if n < 0:
            self._check(n)
        sig = np.zeros(max(n, 1), np.float64)
        lw = np.zeros(max(n, 1), np.int32)
        lh = np.zeros(max(n, 1), np.int32)
        L.ccnn_debug_levels(self.h, frame, sig.ctypes.data_as(_P(C.c_double)),
                            lw.ctypes.data_as(_P(C.c_int32)), lh.ctypes.data_as(_P(C.c_int32)), n)
        return [(float(sig[k]), int(lw[k]), int(lh[k])) for k in range(n)]

    def level_image(self, frame, level):
        _, lw, lh = self.levels(frame)[level]
        out = np.zeros((lh, lw), np.uint8)
        self._check(load().ccnn_debug_level(self.h, frame, level, out.ctypes.data_as(_P(C.c_uint8)),
                                            out.size))
        return out

    def stage1_map(self, frame, level):
        _, lw, lh = self.levels(frame)[level]
        nx, ny = (lw - 27) // 4 + 1, (lh - 31) // 4 + 1
        out = np.zeros((ny, nx), np.float32)
        self._check(load().ccnn_debug_stage1_map(self.h, frame, level,
                                                 out.ctypes.data_as(_P(C.c_float)), out.size))
        return out

    def counters(self):
        out = (C.c_uint32 * 16)()
        n = load().ccnn_debug_counters(self.h, out, 16)
        return list(out[:max(n, 0)])

    def candidates(self):
        L = load()
        n = C.c_int64()
        self._check(L.ccnn_debug_candidates(self.h, None, 0, C.byref(n)))
        if n.value == 0:
            return np.zeros(0, CAND_DTYPE)
        buf = (Candidate * n.value)()
        self._check(L.ccnn_debug_candidates(self.h, buf, n.value, C.byref(n)))
        assert C.sizeof(Candidate) == CAND_DTYPE.itemsize
        return np.frombuffer(bytes(buf), CAND_DTYPE).copy()

    def group(self, raw, n_frames):
        """ccnn_debug_group: the device NMS alone on raw boxes (BOX_DTYPE array; `neighbors`
        ignored) of n_frames frames -> grouped boxes in the ccnn_detect output order."""
        L = load()
        raw = np.ascontiguousarray(raw, BOX_DTYPE)
        cap = max(1, len(raw))
        out = np.zeros(cap, BOX_DTYPE)
        n = C.c_int64()
        self._check(L.ccnn_debug_group(self.h, raw.ctypes.data_as(_P(Box)), len(raw), n_frames,
                                       out.ctypes.data_as(_P(Box)), cap, C.byref(n)))
        return out[:n.value].copy()
