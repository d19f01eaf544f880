"""bench.py's host-side arithmetic (CPU): the level table it reports matches the oracle's (O1),
the algorithmic stage-1 FLOPs are 2 x the dense CNN1 MACs over the conv outputs the windows
need (K2: 2.1346 GFLOP per 4K frame at C4), and the clock / CPU-list
helpers parse what they are given."""
import numpy as np

import bench
import oracle
from synth import configs


def test_level_table_matches_oracle():
    for c in (configs.C1, configs.C3, configs.C4):
        mine = bench.level_table(c.width, c.height, c.min_face, c.scale_step)
        ref = oracle.level_table(c.width, c.height, c.min_face, c.scale_step)
        assert [(w, h) for _, w, h in mine] == [(w, h) for _, w, h in ref]


def test_stage1_alg_flops_c4():
    c = configs.C4
    lv = bench.level_table(c.width, c.height, c.min_face, c.scale_step)
    assert len(lv) == 19
    flops = bench.stage1_alg_flops(lv)
    assert abs(flops - 2.1346e9) / 2.1346e9 < 1e-4
    windows = sum(((w - 27) // 4 + 1) * ((h - 31) // 4 + 1) for _, w, h in lv)
    assert windows == 316848


def test_stage1_alg_flops_brute_force_small():
    """The closed form equals counting the MACs of every conv output some window needs."""
    lw, lh = 47, 51                                   # 6 x 6 windows
    nx, ny = (lw - 27) // 4 + 1, (lh - 31) // 4 + 1
    need1, need2, need3 = set(), set(), set()
    for i in range(ny):
        for j in range(nx):
            need3.add((i, j))
            for y2 in range(2 * i, 2 * i + 12):     # layer-2 conv outputs under the window
                for x2 in range(2 * j, 2 * j + 10):
                    need2.add((y2, x2))
            for y1 in range(4 * i, 4 * i + 28):     # layer-1 conv outputs under the window
                for x1 in range(4 * j, 4 * j + 24):
                    need1.add((y1, x1))
    macs = len(need1) * 6 * 16 + len(need2) * 6 * 54 + len(need3) * (2 * 180 + 2)
    assert bench.stage1_alg_flops([(1.0, lw, lh)]) == 2 * macs


def test_parse_cpulist():
    assert bench.parse_cpulist("0-3,8,10-11\n") == {0, 1, 2, 3, 8, 10, 11}
    assert bench.parse_cpulist("") == set()


def test_split_mma_factor_between_2_and_3():
    """FLOP-weighted MMAs per fp32-accurate product: 2 for layer 1 (exact pixels x hi+lo
    weights), 3 for layers 2-4; the C4 pyramid's weighting equals the per-layer closed form."""
    lv = bench.level_table(3840, 2160, 60, 1.2)
    f = bench.split_mma_factor(lv)
    l1 = l23 = 0
    for _, w, h in lv:
        nx, ny = (w - 27) // 4 + 1, (h - 31) // 4 + 1
        l1 += (4 * nx + 20) * (4 * ny + 24) * 96
        l23 += (2 * nx + 8) * (2 * ny + 10) * 324 + nx * ny * 362
    assert abs(f - (2 * l1 + 3 * l23) / (l1 + l23)) < 1e-12
    assert 2.0 < f < 3.0 and abs(f - 2.513) < 5e-3       # layer 1 is ~49% of the FLOPs
