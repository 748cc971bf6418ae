"""Batched K2-K4 detection vs the reference, repeated (looks for
batch-size-dependent or nondeterministic corner sets).

    python tools/diag_detect_batch.py c1 [reps]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1701_03572_b200 import stab  # noqa: E402
from paper_1701_03572_b200.synth import CONFIGS, Video  # noqa: E402
from tests import _oracle  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = CONFIGS[name]
n = min(cfg.video.frames, 300)
y = Video(cfg.video, threads=os.cpu_count()).render(0, n)[0]
R = cfg.stab.flow.redetect_interval
det = y[0:n - 1:R]
ref = _oracle.reference()
from concurrent.futures import ThreadPoolExecutor
with ThreadPoolExecutor(os.cpu_count()) as ex:
    cpu = list(ex.map(lambda f: ref.detect_corners(f, cfg.stab.detect), det))
for rep in range(reps):
    for nb in (1, 2, 12, len(det)):
        bad = []
        for b0 in range(0, len(det), nb):
            out = stab.detect_corners_batch(det[b0:b0 + nb], cfg.stab.detect)
            for i, (gxy, gsc) in enumerate(out):
                oxy, osc = cpu[b0 + i]
                if not (np.array_equal(gxy, oxy) and np.array_equal(gsc, osc)):
                    same = len(gxy) == len(oxy)
                    nd = int((np.abs(gxy - oxy).max(1) > 0).sum()) if same else -1
                    bad.append((b0 + i, len(gxy), len(oxy), nd))
        print(f"rep {rep} batch {nb}: {len(bad)} of {len(det)} frames differ {bad[:8]}", flush=True)
