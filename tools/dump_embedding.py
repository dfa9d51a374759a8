import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2008_00325_b200 as U
c = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
X = torch.from_numpy(synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"])).cuda()
Y, st = U.fit(X, n_neighbors=c["k"], n_epochs=c["n_epochs"], knn_mode="tensor")
os.makedirs("gpurun_out", exist_ok=True)
np.save("gpurun_out/Y_%s.npy" % (sys.argv[1] if len(sys.argv) > 1 else "C2"), Y.cpu().numpy())
print(st)
