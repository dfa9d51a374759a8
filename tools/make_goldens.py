"""Writes the end-to-end goldens tests/golden/e2e_<case>.json from the ORACLE ONLY (task rule ③:
a stored expected value is written by a committed script that calls only oracle/ and synth/).

Cases (the BASELINE.json configs' recipes):
  C2   the full MNIST-shaped config, 70,000 x 784, k = 15, 500 epochs: the oracle's deterministic
       (buffered, R13) and Hogwild (sequential in place, R14) fits and their trustworthiness T(15);
  C3s  Fashion/CIFAR-shaped rows (d = 3072, 20 blobs, seed 2) at n = 6,000, 200 epochs, T(5);
  C4s  scRNA-shaped rows (d = 50, 30 blobs, seed 3) at n = 20,000, 200 epochs, T(15);
  C5s  the distributed-inference recipe (mixture of seed 4): fit on 10,000 training rows
       (seed 40), transform 20,000 rows (seed 41) in two partitions with global query ids,
       T(15) of the transformed rows.
The full-size C3/C4/C5 oracle runs take hours to days single-node (C4: 1e12 distance pairs), so
those configs are checked end to end at these sizes and stage-wise at full size.

    python tools/make_goldens.py [case ...]      (OMP_NUM_THREADS = cores used)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from oracle import oracle as O  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
A_, B_ = 1.5769434603, 0.8950608779  # R8 fit of (min_dist 0.1, spread 1); pinned in test_oracle


def emit(name, d):
    d["written_by"] = "tools/make_goldens.py (oracle/ + synth/ only)"
    d["oracle_threads"] = O.get_threads()
    with open(os.path.join(GOLD, f"e2e_{name}.json"), "w") as f:
        json.dump(d, f, indent=1)
    print(name, d, flush=True)


def fit_case(name, X, k, n_epochs, trust_k, modes=("deterministic",), seed=0):
    t0 = time.time()
    idx, dist, rho, sigma, w, (indptr, col, val) = O.fuzzy_graph(X, k)
    t_graph = time.time() - t0
    out = {"n": int(X.shape[0]), "d": int(X.shape[1]), "k": k, "n_epochs": n_epochs, "trust_k": trust_k,
           "seed": seed, "nnz": int(indptr[-1]), "s_graph": round(t_graph, 1)}
    Y0 = O.random_init(X.shape[0], 2, seed)
    for mode in modes:
        t1 = time.time()
        Y = O.optimize(indptr, col, val, Y0, np.float32(A_), np.float32(B_), n_epochs, m=5, seed=seed, mode=mode)
        t2 = time.time()
        S, _ = O.trust_penalty(X, Y, trust_k)
        T = O.trust_from_penalty(S, X.shape[0], trust_k)
        out[mode] = {"T": T, "S": int(S), "s_sgd": round(t2 - t1, 1), "s_trust": round(time.time() - t2, 1)}
    emit(name, out)


def case_C2():
    c = synth.CONFIGS["C2"]
    X = synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"])
    fit_case("C2", X, c["k"], c["n_epochs"], 15, modes=("deterministic", "hogwild"))


def case_C3s():
    X = synth.lowrank(6000, 3072, 20, 2)
    fit_case("C3s", X, 15, 200, 5)


def case_C4s():
    X = synth.lowrank(20000, 50, 30, 3)
    fit_case("C4s", X, 15, 200, 15)


def case_C5s():
    model = synth.lowrank_model(784, 10, 4)
    Xtr = synth.lowrank_sample(model, 10000, 40)
    Xq = synth.lowrank_sample(model, 20000, 41)
    t0 = time.time()
    Ytr = O.fit(Xtr, k=15, n_epochs=200, a=A_, b=B_, seed=0, mode="deterministic")
    parts = [O.transform(Xtr, Ytr, Xq[lo:lo + 10000], k=15, n_epochs=200, a=A_, b=B_, seed=0, q_offset=lo)
             for lo in (0, 10000)]
    Yq = np.concatenate(parts)
    S, _ = O.trust_penalty(Xq, Yq, 15)
    emit("C5s", {"n_train": 10000, "n_transform": 20000, "d": 784, "k": 15, "n_epochs": 200,
                 "transform_epochs": 67, "partitions": 2, "seed": 0, "trust_k": 15,
                 "T_train": O.trustworthiness(Xtr, Ytr, 15),
                 "T": O.trust_from_penalty(S, 20000, 15), "S": int(S), "s_total": round(time.time() - t0, 1)})


if __name__ == "__main__":
    cases = sys.argv[1:] or ["C4s", "C3s", "C5s", "C2"]
    for cs in cases:
        globals()["case_" + cs]()
