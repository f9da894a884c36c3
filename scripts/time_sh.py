"""Time stage 1 (matcha_sh_analysis) alone on c2-shaped particles (TS_N / TS_L / TS_B for other shapes), optionally under several MATCHA_SH_DBG values.

usage (GPU box): python scripts/time_sh.py [dbg ...]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15285_b200 as mt  # noqa: E402

N, L, B = int(os.environ.get("TS_N", "64")), int(os.environ.get("TS_L", "32")), int(os.environ.get("TS_B", "1000"))
h = mt.Handle(N=N, L_max=L, quad_oversample=2, max_batch=B)
vols = torch.randn(B, N, N, N, device="cuda")
out = torch.empty(B, mt.ncoef(L), N // 2, dtype=torch.complex64, device="cuda")
for dbg in (sys.argv[1:] or ["0"]):
    os.environ["MATCHA_SH_DBG"] = dbg
    for _ in range(3):
        h.sh_analysis(vols, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        h.sh_analysis(vols, out=out)
    e1.record()
    torch.cuda.synchronize()
    print(f"dbg={dbg}: sh_analysis {e0.elapsed_time(e1) / 10:.3f} ms for {B} particles", flush=True)
