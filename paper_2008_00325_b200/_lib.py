"""ctypes declarations of the C ABI in include/umap_b200.h (argument marshalling only).

Loading fails loudly if libumapb200.so has not been built: there is no Python or
CPU fallback for any step of the hot path.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libumapb200.so")

c_int32, c_int64, c_uint32, c_uint64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64
c_float, c_double, c_void_p = ctypes.c_float, ctypes.c_double, ctypes.c_void_p
P = ctypes.POINTER

UMAP_OK = 0
STATUS = {0: "UMAP_OK", 1: "UMAP_ERR_INVALID_ARGUMENT", 2: "UMAP_ERR_NOT_DEVICE_POINTER", 3: "UMAP_ERR_TOO_FEW_ROWS",
          4: "UMAP_ERR_K_OUT_OF_RANGE", 5: "UMAP_ERR_NONFINITE_INPUT", 6: "UMAP_ERR_NONFINITE_EMBEDDING",
          7: "UMAP_ERR_FIT_AB_NO_CONVERGENCE", 8: "UMAP_ERR_CUDA", 9: "UMAP_ERR_OUT_OF_MEMORY",
          10: "UMAP_ERR_UNSUPPORTED"}
SGD_HOGWILD, SGD_DETERMINISTIC = 0, 1
KNN_EXACT_FP32, KNN_TENSOR_BF16 = 0, 1


class UmapParams(ctypes.Structure):
    _fields_ = [("struct_size", c_uint32), ("n_neighbors", c_int32), ("n_components", c_int32),
                ("n_epochs", c_int32), ("min_dist", c_float), ("spread", c_float),
                ("negative_sample_rate", c_int32), ("learning_rate", c_float), ("repulsion_strength", c_float),
                ("a", c_float), ("b", c_float), ("seed", c_uint64), ("sgd_mode", c_int32), ("knn_mode", c_int32),
                ("knn_candidates", c_int32), ("transform_epochs", c_int32), ("trust_k", c_int32),
                ("far_dist", c_float), ("unknown_dist", c_float), ("init", c_int32), ("spectral_iters", c_int32),
                ("transform_precision", c_int32)]


class UmapFitStats(ctypes.Structure):
    _fields_ = [("ms_knn", c_double), ("ms_smooth", c_double), ("ms_union", c_double), ("ms_init", c_double),
                ("ms_sgd", c_double), ("ms_total", c_double), ("nnz", c_int64), ("positives", c_int64),
                ("w_max", c_float), ("a", c_float), ("b", c_float), ("n_epochs", c_int32),
                ("gpu_launches", c_int32), ("ms_trust", c_double), ("trustworthiness", c_double),
                ("trust_penalty", c_int64)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


# name -> (restype, argtypes); must mirror include/umap_b200.h
SIGNATURES = {
    "umap_params_default": (None, [P(UmapParams)]),
    "umap_fit_ab": (c_int32, [c_float, c_float, P(c_float), P(c_float)]),
    "umap_fit": (c_int32, [c_void_p, c_int64, c_int32, P(UmapParams), c_void_p, P(UmapFitStats), c_void_p]),
    "umap_fit_supervised": (c_int32, [c_void_p, c_int64, c_int32, c_void_p, P(UmapParams), c_void_p,
                                      P(UmapFitStats), c_void_p]),
    "umap_supervised_adjust": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_float, c_float,
                                         c_void_p, c_void_p, c_void_p, c_int64, P(c_int64), c_void_p]),
    "umap_spectral_init": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_int32, c_uint64, c_int32, c_void_p,
                                     c_void_p]),
    "umap_fit_knn": (c_int32, [c_void_p, c_void_p, c_int64, P(UmapParams), c_void_p, P(UmapFitStats), c_void_p]),
    "umap_transform": (c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_int64, c_int64, P(UmapParams),
                                 c_void_p, c_void_p]),
    "umap_trustworthiness": (c_int32, [c_void_p, c_int32, c_void_p, c_int32, c_int64, c_int32, c_int32, P(c_double),
                                       P(c_int64), c_void_p]),
    "umap_knn": (c_int32, [c_void_p, c_int64, c_void_p, c_int64, c_int32, c_int32, c_int64, c_int64, c_int32, c_int32,
                           c_int32, c_void_p, c_void_p, c_void_p]),
    "umap_topk_merge": (c_int32, [c_void_p, c_void_p, c_int32, c_int64, c_int32, c_int32, c_int32, c_void_p, c_void_p,
                                  c_void_p]),
    "umap_smooth_knn": (c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                                  c_void_p]),
    "umap_fuzzy_union": (c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_int64,
                                   P(c_int64), c_void_p]),
    "umap_random_init": (c_int32, [c_int64, c_int32, c_uint64, c_void_p, c_void_p]),
    "umap_optimize": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, P(UmapParams), c_int32, c_int32,
                                P(c_int64), c_void_p]),
    "umap_transform_optimize": (c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_int64, c_void_p,
                                          P(UmapParams), c_int32, c_int32, c_int32, c_int64, c_int32, c_void_p]),
    "umap_trust_penalty": (c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_int32, c_int64, c_int64, c_int32,
                                     c_void_p, c_int32, c_void_p, P(c_int64), c_void_p]),
    "umap_trust_from_penalty": (c_double, [c_int64, c_int64, c_int32]),
    "umap_transform_epoch_count": (c_int32, [c_int32, c_int32, c_int64]),
    "umap_status_string": (ctypes.c_char_p, [c_int32]),
    "umap_last_error": (ctypes.c_char_p, []),
    "umap_kernel_launch_count": (c_int64, []),
    "umap_version": (ctypes.c_char_p, []),
    "umap_trust_ambiguous_count": (c_int64, []),
    "umap_trust_fine_fraction": (c_double, []),
    "umap_profile_begin": (None, []),
    "umap_profile_end": (ctypes.c_int32, [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(c_int64), ctypes.c_int32]),
    "umap_profile_slot_name": (ctypes.c_char_p, [ctypes.c_int32]),
}

_lib = None


def load():
    """Load libumapb200.so (raises if it is missing: build it with __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class UmapError(RuntimeError):
    def __init__(self, status, where):
        L = load()
        super().__init__(f"{where}: {STATUS.get(status, status)}: {L.umap_last_error().decode()}")
        self.status = status


def check(status, where):
    if status != UMAP_OK:
        raise UmapError(status, where)
