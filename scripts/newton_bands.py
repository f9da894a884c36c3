"""Time the evaluation kernel per band (derivs / value-only) on c2-shaped M: where stage 4's time goes."""
import numpy as np, torch, time
import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15285_b200 as mt
torch.manual_seed(0)
B, L = 1000, 32
h = mt.Handle(N=64, L_max=L, max_batch=B)
M = (torch.randn(B, mt.corr_count(L), dtype=torch.complex64, device="cuda") * 100)
eul = torch.rand(B, 10, 3, device="cuda") * torch.tensor([6.28, 3.14, 6.28], device="cuda")
for Lb in (8, 12, 16, 24, 32):
    for derivs in (True, False):
        for _ in range(2): h.eval_corr(M, L, Lb, eul, derivs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): h.eval_corr(M, L, Lb, eul, derivs)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        el = mt.corr_count(Lb)
        fl = el * 10 * (28 if derivs else 8) * B
        print(f"L={Lb:2d} derivs={derivs!s:5} {ms:.3f} ms  {fl/ms/1e9:.1f} TFLOP/s(alg)")
params = mt.Params(bands=(8, 12, 16, 24, 32), n_cand=10)
for _ in range(2): h.newton_refine(M, L, eul, params)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(10): h.newton_refine(M, L, eul, params)
torch.cuda.synchronize(); print("newton_refine full schedule", (time.perf_counter() - t) / 10 * 1e3, "ms")
