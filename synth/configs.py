"""The five BASELINE.json workloads (configs[0..4]) as plain parameter records.

Settings follow SURVEY.md §8 "Configs": C2 uses the FDDB protocol settings of
§4.1 (minSize 15, scaleFactor 1.05, T_nn 1), C4/C5 the Fig. 12 settings
(minSize 60, scaleFactor 1.2, minNeighbors = T_nn 2), C3 the "typical
search settings" of P:237 (40 px, 1.2).  Thresholds come from calib/*.json,
written by oracle/calibrate.py (oracle-only script).
"""
import json
import os
from dataclasses import dataclass

import numpy as np

from . import frames

CALIB_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "calib")
FRAME_SEED = 150801292
CALIB_SEED_OFFSET = 1_000_000


@dataclass(frozen=True)
class Config:
    name: str
    width: int
    height: int
    batch: int          # frames per ccnn_detect call (one bench step)
    min_face: int
    scale_step: float
    Tnn: int
    rule: int           # 0 = Eq. 2 strict, 1 = Eq. 3 weak
    kind: str           # "video" | "stills" | "clutter"
    calib: str          # calib/<calib>.json

    def make_frames(self, n=None, seed=FRAME_SEED):
        n = self.batch if n is None else n
        if self.kind == "stills":
            return frames.make_stills(n, self.width, self.height, seed, self.min_face)
        return frames.make_video(n, self.width, self.height, seed, self.min_face,
                                 clutter=(self.kind == "clutter"))

    def make_frames_at(self, indices, n_total, seed=FRAME_SEED):
        """Frames `indices` of the n_total-frame workload make_frames(n_total) returns (the
        shard of one rank: frame g of the global stream, identical bytes)."""
        if self.kind == "stills":
            return np.stack([frames.make_still(self.width, self.height, seed + int(g), self.min_face)
                             for g in indices])
        return frames.make_video_frames(indices, n_total, self.width, self.height, seed,
                                        self.min_face, clutter=(self.kind == "clutter"))

    def thresholds(self):
        with open(os.path.join(CALIB_DIR, self.calib + ".json")) as f:
            c = json.load(f)
        return float(c["T1"]), (float(c["T2"][0]), float(c["T2"][1]))


C1 = Config("c1_320x240_min24", 320, 240, 1, 24, 1.2, 2, 0, "video", "c4")
C2 = Config("c2_fddb_450x450x256_min15", 450, 450, 256, 15, 1.05, 1, 0, "stills", "c4")
C3 = Config("c3_1080p_min40", 1920, 1080, 32, 40, 1.2, 2, 0, "video", "c4")
C4 = Config("c4_4k_min60", 3840, 2160, 32, 60, 1.2, 2, 0, "video", "c4")
C5 = Config("c5_4k_clutter_min60", 3840, 2160, 16, 60, 1.2, 2, 0, "clutter", "c5")

CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5)}
BY_ID = {"c1": C1, "c2": C2, "c3": C3, "c4": C4, "c5": C5}
