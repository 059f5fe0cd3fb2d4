"""SPEC.md:610 acceptance #2 (synthetic disparity accuracy): on a rendered
textured slanted plane and a sphere (+-0.5 gray-level noise), >= 95% of the
valid pixels lie within 1 px of the ground-truth disparity after the full
stereo stage (compute_disparity -> cleanup_pass -> refine_disparities).
Generator: paper_2007_12623_b200/synth.py kinds "plane" and "sphere"."""
import numpy as np
import pytest


def _within_1px(d, v, gt):
    m = v == 1
    assert m.mean() > 0.9, f"only {m.mean():.3f} valid"
    return float((np.abs(d[m] - gt[m]) <= 1.0).mean())


@pytest.mark.parametrize("kind", ["plane", "sphere"])
def test_accuracy_restatement(orc, kind):
    """The CPU restatement (held bit-exact to the reference elsewhere)."""
    from paper_2007_12623_b200.synth import params_for, stereo_pair
    L, R, gt = stereo_pair(kind, 320, 240, 32, seed=5)
    p = params_for(32)
    d, v = orc.refine_disparities(*orc.cleanup_pass(*orc.compute_disparity(L, R, p), p), L, R, p)
    assert _within_1px(d, v, gt) >= 0.95


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["plane", "sphere"])
def test_accuracy_gpu_batch_api(kind):
    """The B200 chain through the batch API at 960x540, D = 64."""
    import paper_2007_12623_b200 as ss
    from paper_2007_12623_b200.synth import as_rgb, params_for, stereo_pair
    L, R, gt = stereo_pair(kind, 960, 540, 64, seed=5)
    ctx = ss.StereoContext(0, 960, 540, 1, ss.StereoParams(**params_for(64)))
    out = ctx.run(as_rgb(L)[None], as_rgb(R)[None], ss.SS_OUT_DISPARITY)
    ctx.close()
    assert _within_1px(out["disparity"][0], out["valid"][0], gt) >= 0.95
