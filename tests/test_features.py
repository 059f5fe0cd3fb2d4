"""Feature front end (segment-test corners, 256-bit
descriptors, mutual Hamming matching, histogram vote).

Oracle: the reference's own features.cpp, compiled unmodified into
oracle/_ref (tests/golden/make_golden_features.py made the fixtures from it).
detect_corners / describe / match_features run on the B200 through the C-ABI
and must be bit-identical (integer work); histogram_vote is a host utility
checked against the reference on CPU.
"""
import numpy as np
import pytest

from conftest import load_golden
from paper_2007_12623_b200.synth import stereo_pair


def test_golden_features_pinned_to_reference(ref):
    g = load_golden("features_tex")
    mc, thr, mh, _ = g["cfg"]
    for tag, img in (("l", g["left"]), ("r", g["right"])):
        c = ref.detect_corners(img, int(mc), int(thr))
        assert np.array_equal(c, g[f"corners_{tag}"])
        pos, desc = ref.describe(img, c)
        assert np.array_equal(pos, g[f"pos_{tag}"]) and np.array_equal(desc, g[f"desc_{tag}"])


def test_histogram_vote_host_matches_reference(ref):
    import paper_2007_12623_b200 as ss
    g = load_golden("features_tex")
    m = {k[len("match_"):]: g[k] for k in g if k.startswith("match_")}
    out = ss.features.histogram_vote(m, float(g["cfg"][3]))
    assert np.array_equal(out["order"], g["vote_order"])
    rng = np.random.default_rng(3)
    for _ in range(5):
        n = 200
        mm = {"index_a": np.arange(n, dtype=np.int32), "index_b": rng.permutation(n).astype(np.int32),
              "hamming": rng.integers(0, 40, n).astype(np.int32),
              "displacement": np.round(rng.normal(0, 6, (n, 2)))}
        assert np.array_equal(ss.features.histogram_vote(mm, 3.0)["order"],
                              ref.histogram_vote(mm, 3.0))


def test_histogram_vote_contract():
    import paper_2007_12623_b200 as ss
    with pytest.raises(ValueError):
        ss.features.histogram_vote({"displacement": np.zeros((1, 2)), "hamming": [0]}, 0.0)


# ---------------- GPU ----------------

@pytest.fixture(scope="module")
def ss():
    import paper_2007_12623_b200 as ss
    from paper_2007_12623_b200.build import build
    build(verbose=False)
    if ss.device_count() < 1:
        pytest.fail("no CUDA device visible to the GPU tests")
    return ss


@pytest.mark.gpu
def test_gpu_features_golden(ss):
    g = load_golden("features_tex")
    mc, thr, mh, _ = (int(x) for x in g["cfg"])
    got = {}
    for tag, img in (("l", g["left"]), ("r", g["right"])):
        c = ss.features.detect_corners(img, mc, thr)
        assert np.array_equal(c, g[f"corners_{tag}"]), f"corners {tag}"
        pos, desc = ss.features.describe(img, c)
        assert np.array_equal(pos, g[f"pos_{tag}"]) and np.array_equal(desc, g[f"desc_{tag}"])
        got[tag] = (pos, desc)
    m = ss.features.match_features(*got["l"], *got["r"], mh)
    for k in ("index_a", "index_b", "hamming", "displacement"):
        assert np.array_equal(m[k], g["match_" + k]), k


@pytest.mark.gpu
def test_gpu_features_kats(ss):
    k = load_golden("features_kats")
    assert np.array_equal(ss.features.detect_corners(k["square"], 100, 30), k["square_corners"])
    assert len(ss.features.detect_corners(k["uniform"], 100, 1)) == 0
    assert np.array_equal(ss.features.detect_corners(k["noise"], 300, 1), k["noise_corners"])
    with pytest.raises(ss.InvalidArgument, match="threshold must be >= 1"):
        ss.features.detect_corners(k["square"], 10, 0)
    assert len(ss.features.detect_corners(k["square"], 0, 30)) == 0
    assert len(ss.features.detect_corners(np.zeros((5, 5), np.uint8), 10, 5)) == 0
    pos, desc = ss.features.describe(k["square"], np.zeros((0, 3), np.int32))
    assert len(pos) == 0
    m = ss.features.match_features(pos, desc, pos, desc, 64)
    assert len(m["index_a"]) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("kind,W,H,mc,thr", [("textured", 960, 540, 2000, 20),
                                             ("lowtex", 640, 360, 1000, 5),
                                             ("textured", 1920, 1080, 4000, 30)])
def test_gpu_features_vs_reference(ss, ref, kind, W, H, mc, thr):
    L, R, _ = stereo_pair(kind, W, H, 32, seed=9)
    fa, fb = [], []
    for img, acc in ((L, fa), (R, fb)):
        c = ss.features.detect_corners(img, mc, thr)
        assert np.array_equal(c, ref.detect_corners(img, mc, thr))
        pos, desc = ss.features.describe(img, c)
        rp, rd = ref.describe(img, c)
        assert np.array_equal(pos, rp) and np.array_equal(desc, rd)
        acc += [pos, desc]
    for mh in (40, 256):
        m = ss.features.match_features(*fa, *fb, mh)
        r = ref.match_features(*fa, *fb, mh)
        for k in r:
            assert np.array_equal(m[k], r[k]), (k, mh)


@pytest.mark.gpu
def test_gpu_describe_arbitrary_corner_order(ss, ref):
    rng = np.random.default_rng(17)
    img = rng.integers(0, 256, (120, 150), dtype=np.uint8)
    c = np.stack([rng.integers(0, 150, 400), rng.integers(0, 120, 400),
                  rng.integers(1, 99, 400)], axis=1).astype(np.int32)
    pos, desc = ss.features.describe(img, c)
    rp, rd = ref.describe(img, c)
    assert np.array_equal(pos, rp) and np.array_equal(desc, rd)
