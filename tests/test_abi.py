"""CPU-side checks of the boundary: the C-ABI library loads and exports every symbol
include/umap_b200.h declares; the ctypes structs match the header layout; host-only
entry points work without a GPU; compute calls fail loudly without one."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2008_00325_b200 import build
    build.build()
    from paper_2008_00325_b200 import _lib
    return _lib


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "umap_b200.h")).read()
    return sorted(set(re.findall(r"UMAP_API\s+[\w\s\*]+?\b(umap_\w+)\s*\(", src)))


def test_header_declares_entry_points():
    names = _declared_symbols()
    for must in ("umap_fit", "umap_transform", "umap_trustworthiness", "umap_knn", "umap_topk_merge",
                 "umap_smooth_knn", "umap_fuzzy_union", "umap_optimize", "umap_random_init"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    L = lib.load()
    for name in _declared_symbols():
        assert hasattr(L, name), name
        assert name in lib.SIGNATURES, f"binding lacks {name}"
    assert set(lib.SIGNATURES) == set(_declared_symbols())


def _c_layout(struct, fields):
    """sizeof/offsetof of a header struct as gcc lays it out (the C side of the ABI)."""
    import subprocess
    import tempfile
    body = "".join(f'printf("%zu\\n", offsetof({struct}, {f}));' for f in fields)
    src = (f'#include <stdio.h>\n#include <stddef.h>\n#include "umap_b200.h"\n'
           f'int main(void){{printf("%zu\\n", sizeof({struct}));{body}return 0;}}\n')
    with tempfile.TemporaryDirectory() as td:
        c, exe = os.path.join(td, "probe.c"), os.path.join(td, "probe")
        open(c, "w").write(src)
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        vals = [int(x) for x in subprocess.check_output([exe]).split()]
    return vals[0], dict(zip(fields, vals[1:]))


@pytest.mark.parametrize("cname,pyname", [("umap_params", "UmapParams"), ("umap_fit_stats", "UmapFitStats")])
def test_struct_layout_matches_header(lib, cname, pyname):
    cls = getattr(lib, pyname)
    fields = [f for f, _ in cls._fields_]
    size, offs = _c_layout(cname, fields)
    assert ctypes.sizeof(cls) == size
    for f in fields:
        assert getattr(cls, f).offset == offs[f], f


def test_params_defaults(lib):
    p = lib.UmapParams()
    lib.load().umap_params_default(ctypes.byref(p))
    assert p.struct_size == ctypes.sizeof(lib.UmapParams) and p.n_neighbors == 15 and p.n_components == 2
    assert p.negative_sample_rate == 5 and p.trust_k == 0
    assert p.sgd_mode == lib.SGD_DETERMINISTIC and p.knn_candidates == 32


def test_fit_ab_host_only_matches_published(lib):
    a, b = ctypes.c_float(), ctypes.c_float()
    assert lib.load().umap_fit_ab(0.1, 1.0, ctypes.byref(a), ctypes.byref(b)) == 0
    assert abs(a.value - 1.5769434603) < 1e-6 and abs(b.value - 0.8950608779) < 1e-6
    assert lib.load().umap_fit_ab(0.1, 0.0, ctypes.byref(a), ctypes.byref(b)) == 1  # INVALID_ARGUMENT


def test_status_strings(lib):
    L = lib.load()
    for code, name in lib.STATUS.items():
        assert L.umap_status_string(code).decode() == name


def test_compute_without_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    L = lib.load()
    p = lib.UmapParams()
    L.umap_params_default(ctypes.byref(p))
    buf = (ctypes.c_float * 64)()
    out = (ctypes.c_float * 32)()
    st = L.umap_fit(ctypes.cast(buf, ctypes.c_void_p), 16, 4, ctypes.byref(p), ctypes.cast(out, ctypes.c_void_p),
                    None, None)
    assert st == 8  # UMAP_ERR_CUDA: no CPU fallback
    assert "no CPU fallback" in L.umap_last_error().decode()


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2008_00325_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace("oracle/", ""), f
