"""Where does the e2e (host buffers) time go?  H2D copy alone, fit on device X, fit on host X."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2008_00325_b200 as U
c = synth.CONFIGS["C2"]
Xh = torch.from_numpy(synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"])).pin_memory()
X = Xh.cuda(); torch.cuda.synchronize()
Yh = torch.empty((c["n"], 2), pin_memory=True)
kw = dict(n_neighbors=15, n_epochs=500, knn_mode="tensor", trust_k=15)
for name, fn in [("h2d", lambda: X.copy_(Xh, non_blocking=True)),
                 ("fit dev", lambda: U.fit(X, **kw)), ("fit host", lambda: U.fit(Xh, out=Yh, **kw))]:
    for i in range(4):
        torch.cuda.synchronize(); t = time.perf_counter(); r = fn(); torch.cuda.synchronize()
        dt = (time.perf_counter() - t) * 1e3
        st = r[1] if isinstance(r, tuple) else {}
        print(f"{name}: {dt:.1f} ms  " + " ".join(f"{k}={v:.2f}" for k, v in st.items() if k.startswith("ms_")), flush=True)
