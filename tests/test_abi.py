"""CPU-side checks of the C-ABI boundary (no GPU compute).

* libccnn.so builds for sm_100a, loads, and exports every function include/ccnn.h declares;
* the ctypes mirrors have the header's struct layouts (sizeof/offsetof from a C program
  compiled against include/ccnn.h with gcc);
* ccnn_create validates architecture / weights / arguments before touching a device.
"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1508_01292_b200 import build as pkg_build
from paper_1508_01292_b200 import ccnn
from synth import arch, weights

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ccnn.h")


@pytest.fixture(scope="module")
def lib():
    pkg_build.build()
    return ccnn.load()


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(ccnn_\w+)\s*\(", src, flags=re.M))
    return names


def test_exports_every_declared_symbol(lib):
    declared = _declared_functions()
    assert declared == set(ccnn.EXPORTS), (declared ^ set(ccnn.EXPORTS))
    out = subprocess.check_output(["nm", "-D", "--defined-only", ccnn.LIB_PATH]).decode()
    exported = set(re.findall(r" T (ccnn_\w+)", out))
    assert declared <= exported, declared - exported
    for name in declared:
        getattr(lib, name)
    assert lib.ccnn_abi_version() == 5


def test_sm100a_code_present():
    out = subprocess.check_output(["cuobjdump", "--list-elf", ccnn.LIB_PATH]).decode()
    assert "sm_100a" in out


def test_struct_layouts_match_header(tmp_path):
    prog = tmp_path / "sizes.c"
    prog.write_text("""
#include <stdio.h>
#include <stddef.h>
#include "ccnn.h"
int main(void){
 printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(ccnn_layer), sizeof(ccnn_net), sizeof(ccnn_params),
        sizeof(ccnn_box), sizeof(ccnn_stats), sizeof(ccnn_candidate), sizeof(ccnn_frame));
 printf("%zu %zu %zu %zu %zu %zu %zu\\n", offsetof(ccnn_params, T1), offsetof(ccnn_params, Tnn),
        offsetof(ccnn_params, segment_rows), offsetof(ccnn_stats, ms), offsetof(ccnn_candidate, r3),
        offsetof(ccnn_frame, pitch), offsetof(ccnn_frame, channels));
 return 0;}
""")
    exe = tmp_path / "sizes"
    subprocess.check_call(["gcc", "-I", os.path.dirname(HEADER), str(prog), "-o", str(exe)])
    a, b = subprocess.check_output([str(exe)]).decode().split("\n")[:2]
    sizes = list(map(int, a.split()))
    offs = list(map(int, b.split()))
    assert sizes == [C.sizeof(ccnn.Layer), C.sizeof(ccnn.Net), C.sizeof(ccnn.Params),
                     C.sizeof(ccnn.Box), C.sizeof(ccnn.Stats), C.sizeof(ccnn.Candidate),
                     C.sizeof(ccnn.Frame)]
    assert offs == [ccnn.Params.T1.offset, ccnn.Params.Tnn.offset, ccnn.Params.segment_rows.offset,
                    ccnn.Stats.ms.offset, ccnn.Candidate.r3.offset, ccnn.Frame.pitch.offset,
                    ccnn.Frame.channels.offset]
    assert ccnn.BOX_DTYPE.itemsize == C.sizeof(ccnn.Box)
    assert ccnn.CAND_DTYPE.itemsize == C.sizeof(ccnn.Candidate)


def _params(layers=arch.NETS, ws=None, **kw):
    ws = ws if ws is not None else weights.make_cascade_weights()
    keep = [[ccnn.Layer(*l) for l in ls] for ls in layers]
    arrs = [(ccnn.Layer * len(k))(*k) for k in keep]
    wa = [np.ascontiguousarray(w, np.float32) for w in ws]
    nets = (ccnn.Net * 3)(*[ccnn.Net(len(layers[k]), arrs[k], wa[k].ctypes.data_as(C.POINTER(C.c_float)),
                                     wa[k].size) for k in range(3)])
    d = dict(T1=0.5, T2=(0.5, 0.5), Tnn=2, rule=0, nms_min_cluster=1, max_w=640, max_h=480,
             max_batch=4, queue_capacity=1024, segment_rows=0)
    d.update(kw)
    p = ccnn.Params(nets, d["T1"], (C.c_float * 2)(*d["T2"]), d["Tnn"], d["rule"],
                    d["nms_min_cluster"], d["max_w"], d["max_h"], d["max_batch"],
                    d["queue_capacity"], d["segment_rows"])
    return p, (arrs, wa)


def test_create_validation_without_gpu(lib):
    h = C.c_void_p()
    bad = list(arch.NETS)
    bad[0] = tuple(list(arch.CNN1[:4]) + [(0, 6, 2, 5, 5)] + list(arch.CNN1[5:]))  # 27x30 window
    p, keep = _params(layers=bad)
    assert lib.ccnn_create(C.byref(p), 0, C.byref(h)) == ccnn.CCNN_E_ARCH
    ws = list(weights.make_cascade_weights())
    ws[1] = ws[1].copy()
    ws[1][7] = np.nan
    p, keep = _params(ws=ws)
    assert lib.ccnn_create(C.byref(p), 0, C.byref(h)) == ccnn.CCNN_E_WEIGHTS
    ws = list(weights.make_cascade_weights())
    ws[2] = ws[2][:-1]
    p, keep = _params(ws=ws)
    assert lib.ccnn_create(C.byref(p), 0, C.byref(h)) == ccnn.CCNN_E_WEIGHTS
    p, keep = _params(Tnn=0)
    assert lib.ccnn_create(C.byref(p), 0, C.byref(h)) == ccnn.CCNN_E_ARG
    p, keep = _params(T1=float("inf"))
    assert lib.ccnn_create(C.byref(p), 0, C.byref(h)) == ccnn.CCNN_E_WEIGHTS
    assert lib.ccnn_create(None, 0, C.byref(h)) == ccnn.CCNN_E_ARG
    assert b"NULL context" in lib.ccnn_last_error(None)
    if not _has_gpu():
        p, keep = _params()
        assert lib.ccnn_create(C.byref(p), 0, C.byref(h)) == ccnn.CCNN_E_CUDA
        assert not h.value


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1508_01292_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "ccnn_oracle" not in txt, f
