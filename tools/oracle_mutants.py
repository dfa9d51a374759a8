"""Mutation check of the oracle pins: build deliberately broken copies of oracle/umap_oracle.c
(one plausible mistake each) and show that the `-m "not gpu"` pins fail on every one of them.

    python tools/oracle_mutants.py [> profiles/oracle_mutants_r02.txt]

Each mutant is compiled to /tmp and loaded through UMAP_ORACLE_LIB (test infrastructure only);
the pins run in a subprocess with that override.  A mutant "survives" if all its pins pass.
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "umap_oracle.c")

FIT_ALPHA = "float alpha = alpha0 * (1.0f - (float)e / (float)n_epochs);"
TR_ALPHA = "float alpha = alpha0 * (1.0f - (float)e / (float)n_epochs_t);"
MUTANTS = [
    ("fit alpha lags one epoch (R10)", FIT_ALPHA,
     "float alpha = alpha0 * (1.0f - (float)(e - 1) / (float)n_epochs);"),
    ("fit alpha never decays (R10)", FIT_ALPHA, "float alpha = alpha0;"),
    ("transform alpha lags one epoch (R10/R15)", TR_ALPHA,
     "float alpha = alpha0 * (1.0f - (float)(e - 1) / (float)n_epochs_t);"),
    ("transform alpha never decays", TR_ALPHA, "float alpha = alpha0;"),
    ("repulsion also pushes the sampled vertex (deterministic)",
     "for (int c = 0; c < dim; ++c) buf[h * dim + c] += g[c];\n                    } else {",
     "for (int c = 0; c < dim; ++c) { buf[h * dim + c] += g[c]; buf[v * dim + c] -= g[c]; }\n                    } else {"),
    ("repulsion also pushes the sampled vertex (hogwild)",
     "for (int c = 0; c < dim; ++c) yh[c] = (float)((double)yh[c] + g[c]);\n                    }\n                }",
     "for (int c = 0; c < dim; ++c) { yh[c] = (float)((double)yh[c] + g[c]); Y[v * dim + c] = (float)((double)Y[v * dim + c] - g[c]); }\n                    }\n                }"),
    ("transform negatives over n_train - 1 rows",
     "int64_t v = (int64_t)(((uint64_t)u * (uint64_t)ntr) >> 32);",
     "int64_t v = (int64_t)(((uint64_t)u * (uint64_t)(ntr - 1)) >> 32);"),
    ("transform negatives skip v == 0 like the fit's v == head",
     "const float* yv = Ytr + v * dim;",
     "if (v == 0) continue; const float* yv = Ytr + v * dim;"),
    ("transform RNG keyed by the local query id",
     "uint32_t head = (uint32_t)(q + q_offset);", "uint32_t head = (uint32_t)q;"),
]
PINS = ["tests/test_oracle_sgd_pins.py", "tests/test_oracle.py"]


def main():
    src = open(SRC).read()
    tmp = tempfile.mkdtemp()
    survived = 0
    for i, (name, old, new) in enumerate(MUTANTS):
        assert src.count(old) >= 1, name
        mut = src.replace(old, new, 1)
        c = os.path.join(tmp, f"m{i}.c")
        so = os.path.join(tmp, f"m{i}.so")
        open(c, "w").write(mut)
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-o", so, c, "-lm"])
        env = dict(os.environ, UMAP_ORACLE_LIB=so)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "not gpu", "-p", "no:cacheprovider", *PINS],
                           cwd=ROOT, env=env, capture_output=True, text=True)
        failed = [ln.split(" ")[1] for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
        status = "KILLED" if r.returncode != 0 else "SURVIVED"
        survived += r.returncode == 0
        print(f"{status:8s} {name}: {len(failed)} failing pins")
        for f in failed[:6]:
            print(f"           {f}")
    print(f"{len(MUTANTS) - survived}/{len(MUTANTS)} mutants killed")
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
