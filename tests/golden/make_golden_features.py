"""Golden vectors for the feature front end, generated
from the REAL reference (/root/reference/proj/src/features/features.cpp,
compiled unmodified into oracle/_ref/libss_ref.so by ``make -C oracle``).
Runs only where /root/reference exists; the fixtures are committed.

  features_tex.npz   256x160 textured stereo pair (d in [0,15]): corners
                     (max_count 500, threshold 20) of both views, their
                     descriptors, mutual matches (max_hamming 64) and the
                     histogram_vote order (bin 4 px)
  features_kats.npz  a white square on black (4 corners), a uniform image
                     (no corners), threshold 1 on noise (many corners, capped)
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402
from paper_2007_12623_b200.synth import stereo_pair  # noqa: E402


def main():
    ref = Oracle("ref")
    L, R, _ = stereo_pair("textured", 256, 160, 16, seed=21)
    out = {"left": L, "right": R, "cfg": np.array([500, 20, 64, 4.0])}
    for tag, img in (("l", L), ("r", R)):
        c = ref.detect_corners(img, 500, 20)
        pos, desc = ref.describe(img, c)
        out[f"corners_{tag}"], out[f"pos_{tag}"], out[f"desc_{tag}"] = c, pos, desc
    m = ref.match_features(out["pos_l"], out["desc_l"], out["pos_r"], out["desc_r"], 64)
    for k, v in m.items():
        out["match_" + k] = v
    out["vote_order"] = ref.histogram_vote(m, 4.0)
    np.savez_compressed(os.path.join(HERE, "features_tex.npz"), **out)

    sq = np.zeros((64, 64), np.uint8)
    sq[20:44, 20:44] = 255
    uni = np.full((48, 48), 90, np.uint8)
    rng = np.random.default_rng(5)
    noise = rng.integers(0, 256, (72, 96), dtype=np.uint8)
    k = {"square": sq, "uniform": uni, "noise": noise}
    k["square_corners"] = ref.detect_corners(sq, 100, 30)
    k["uniform_corners"] = ref.detect_corners(uni, 100, 1)
    k["noise_corners"] = ref.detect_corners(noise, 300, 1)
    np.savez_compressed(os.path.join(HERE, "features_kats.npz"), **k)
    print("square corners:", k["square_corners"].tolist())
    print("noise corners:", len(k["noise_corners"]), "tex corners:", len(out["corners_l"]),
          "matches:", len(m["index_a"]))


if __name__ == "__main__":
    main()
