"""Measurement only: dump a config's fuzzy graph (CSR of B) to gpurun_out/graph_<cfg>.npz so the
SGD's per-epoch due-edge statistics can be studied on the CPU.   python tools/dump_graph.py [C2]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2008_00325_b200 as U  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
c = synth.CONFIGS[cfg]
X = torch.from_numpy(synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"])).cuda()
idx, dist = U.knn(X, X, c["k"], exclude_self=True, mode="tensor")
_, _, w, cs = U.smooth_knn(dist, idx, sort_by_col=True)
indptr, col, val = U.fuzzy_union(cs, w)
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed("gpurun_out/graph_%s.npz" % cfg, indptr=indptr.cpu().numpy(), col=col.cpu().numpy(),
                    val=val.cpu().numpy())
print(cfg, "n", c["n"], "nnz", int(indptr[-1]))
