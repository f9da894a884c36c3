import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen, oracle as O, paper_2603_15285_b200 as mt
dev=torch.device('cuda',0)
N,L,B=int(sys.argv[1]),int(sys.argv[2]),40
b=gen.particles(N,B,0.1,seed=26)
h=mt.Handle(N=N,L_max=L,max_batch=B)
r=np.random.default_rng(3)
sh=r.uniform(-3,3,(B,3))
F=h.sh_analysis(torch.from_numpy(b.vols).to(dev), torch.from_numpy(sh).float().to(dev)).cpu().numpy()
try: h.status(); print("status ok")
except Exception as e: print("status", e)
Fo=O.sh_analysis_batch(b.vols,L,2,sh.astype(np.float32).astype(np.float64))
bad=[]
for p in range(B):
    err=np.abs(F[p]-Fo[p]); sc=np.abs(Fo[p]).max()
    if err.max()/sc>2e-5:
        i=np.unravel_index(err.argmax(),err.shape); bad.append((p,err.max()/sc,i,sh[p].round(3).tolist()))
print(N,L,"bad",len(bad)); [print(x) for x in bad[:8]]
del h
