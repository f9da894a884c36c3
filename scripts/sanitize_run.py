"""Small whole-path runs for compute-sanitizer (memcheck / racecheck / synccheck): c1 with translation (32^3,
T=3, W=4), a 64-particle c2 batch (64^3, L0=8 -> 32; stage 1 on the tensor-core ring kernel), and the f-row paths
(upsampled subpixel, multi-template, reconstruct, ball basis) at c1 size.

usage: compute-sanitizer --tool memcheck python scripts/sanitize_run.py [c1|c2|extras]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2603_15285_b200 as mt  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "c1"
dev = torch.device("cuda", 0)
if what == "c1":
    b = gen.particles(32, 4, float("inf"), seed=12, shift_mode=gen.SHIFT_FIXED, fixed_shift=(1.0, -2.0, 1.0))
    h = mt.Handle(N=32, L_max=8, max_batch=4)
    p = h.align_batch(torch.from_numpy(b.vols).to(dev), torch.from_numpy(b.ref).to(dev),
                      mt.Params(bands=[4, 6, 8], n_cand=4, n_alternations=3, shift_window=4))
elif what == "c2":
    b = gen.particles(64, 64, 0.1, seed=1)
    h = mt.Handle(N=64, L_max=32, max_batch=64)
    p = h.align_batch(torch.from_numpy(b.vols).to(dev), torch.from_numpy(b.ref).to(dev),
                      mt.Params(bands=[8, 12, 16, 24, 32], n_cand=10))
else:
    b = gen.particles(32, 6, 0.5, seed=13, shift_mode=gen.SHIFT_UNIFORM, shift_max=2.0)
    h = mt.Handle(N=32, L_max=8, max_batch=6)
    v, r = torch.from_numpy(b.vols).to(dev), torch.from_numpy(b.ref).to(dev)
    h.align_batch(v, r, mt.Params(bands=[4, 6, 8], n_cand=4, n_alternations=2, shift_window=4, upsample=16))
    pm = h.align_multi(v, torch.stack([r, r.flip(0)]), mt.Params(bands=[4, 6, 8], n_cand=4, n_alternations=2,
                                                                 shift_window=4))
    h.reconstruct(v, pm, n_classes=2, class_col=8)
    h.align_batch(v, r, mt.Params(bands=[4, 6, 8], n_cand=4, radial=1))
    h.synth_particles(3, 0.1, shift_max=2.0)
    p = pm
h.status()
torch.cuda.synchronize()
print(what, "ok", np.round(p.cpu().numpy()[0], 4).tolist())
