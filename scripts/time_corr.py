"""Time stage 2 (matcha_corr_coeffs) alone on c2-shaped inputs under several MATCHA_CORR_DBG values."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15285_b200 as mt  # noqa: E402

N, L, B = 64, 32, 1000
h = mt.Handle(N=N, L_max=L, quad_oversample=2, max_batch=B)
F = torch.randn(B, mt.ncoef(L), N // 2, dtype=torch.complex64, device="cuda")
H = torch.randn(mt.ncoef(L), N // 2, dtype=torch.complex64, device="cuda")
for dbg in (sys.argv[1:] or ["0"]):
    os.environ["MATCHA_CORR_DBG"] = dbg
    for _ in range(3):
        M = h.corr_coeffs(F, H, L)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        h.corr_coeffs(F, H, L, out=M)
    e1.record()
    torch.cuda.synchronize()
    print(f"dbg={dbg}: corr_coeffs {e0.elapsed_time(e1) / 10:.3f} ms for {B} particles", flush=True)
