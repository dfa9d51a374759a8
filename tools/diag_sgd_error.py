import sys; sys.path.insert(0,'.')
import numpy as np, torch, synth
import paper_2008_00325_b200 as U
from oracle import oracle as O
A_, B_ = 1.5769434603, 0.8950608779
X = synth.lowrank(1900, 24, seed=7); Xtr, Xq = X[:1200], X[1200:]
Ytr = O.fit(Xtr, k=15, n_epochs=40, a=A_, b=B_, seed=1)
idx, dist = O.knn(Xq, Xtr, 15); rho, sigma = O.smooth_knn(dist); w = O.membership(dist, rho, sigma)
Nt=67; Y = O.transform_init(idx, w, Ytr)
cu=lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
errs=[]
for e in range(1, Nt):
    ref = O.transform_optimize(idx, w, Ytr, Y, A_, B_, Nt, seed=9, e_begin=e, e_end=e+1)
    Yg = cu(Y); U.transform_optimize(cu(idx), cu(w), cu(Ytr), Yg, Nt, e_begin=e, e_end=e+1, a=A_, b=B_, seed=9)
    d = np.abs(Yg.cpu().numpy()-ref).max(1); errs.append(d); Y = ref
E=np.array(errs); print('max per epoch', np.round(E.max(1)*1e6).astype(int)[:20]); print('p99.9', np.quantile(E,0.999), 'max', E.max(), 'frac>1e-4', (E>1e-4).mean(), 'frac>1e-5', (E>1e-5).mean())
# fit det mode per-epoch error distribution
_,_,_,_,_,(indptr,col,val)=O.fuzzy_graph(synth.lowrank(1500,32,seed=5),15)
Y=synth.uniform_embedding(1500,2,seed=1); errs=[]
for e in range(1,200,7):
    ref=O.optimize(indptr,col,val,Y,A_,B_,200,e_begin=e,e_end=e+1,m=5,seed=11)
    Yg=cu(Y); U.optimize(cu(indptr),cu(col),cu(val),Yg,e_begin=e,e_end=e+1,n_epochs=200,a=A_,b=B_,seed=11)
    errs.append(np.abs(Yg.cpu().numpy()-ref).max()); Y=ref
print('fit det max per epoch', max(errs), np.round(np.array(errs)*1e6).astype(int))
