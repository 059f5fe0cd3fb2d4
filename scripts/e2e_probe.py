"""Where does the end-to-end (host buffers) time go? Times ss_stereo_batch for
output-flag variants against the device-resident run (same frames)."""
import time

import torch

import paper_2007_12623_b200 as ss
from bench import H, W, D, make_frames
from paper_2007_12623_b200.synth import default_rig, params_for

F, B = 256, 16
L, R = make_frames(0, 1, F, 32)
Lh, Rh = torch.from_numpy(L).pin_memory(), torch.from_numpy(R).pin_memory()
ctx = ss.StereoContext(0, W, H, B, ss.StereoParams(**params_for(D)), ss.StereoRig(**default_rig(W, H)))
full = ss.SS_OUT_DISPARITY | ss.SS_OUT_CLOUD | ss.SS_OUT_NORMALS
for name, flags in (("full", full), ("disp+cloud", ss.SS_OUT_DISPARITY | ss.SS_OUT_CLOUD),
                    ("disp", ss.SS_OUT_DISPARITY)):
    ho = ss.StereoContext.alloc_outputs(F, H, W, flags, alloc=lambda s, dt: ss.pinned_empty(s, dt))
    ctx.run(Lh.numpy()[:B], Rh.numpy()[:B], flags, out={k: v[:B] for k, v in ho.items()})
    torch.cuda.synchronize()
    t = time.perf_counter()
    ctx.run(Lh.numpy(), Rh.numpy(), flags, out=ho)
    dt = time.perf_counter() - t
    print(f"{name:12s} {F / dt:8.1f} pairs/s  ({dt * 1e3 / F:.3f} ms/pair)")
