"""B200-native GPU-UMAP hot path (arXiv 2008.00325) behind a C ABI (include/umap_b200.h).

The compute lives in libumapb200.so (hand-written CUDA for sm_100a); this package
only marshals torch tensors into that ABI (api.py) and orchestrates multi-GPU runs
over torch.distributed (dist.py).  There is no CPU fallback.
"""
from .api import (fit, fit_ab, fit_knn, fuzzy_union, kernel_launch_count, knn, optimize, params, random_init, smooth_knn,
                  topk_merge, transform, transform_optimize, trust_from_penalty, trust_penalty, trustworthiness,
                  version, default_transform_epochs, trust_ambiguous_count,
                  profile_begin, profile_end, trust_fine_fraction,
                  supervised_adjust, spectral_init)

__all__ = ["fit", "fit_ab", "fit_knn", "fuzzy_union", "kernel_launch_count", "knn", "optimize", "params", "random_init",
           "smooth_knn", "topk_merge", "transform", "transform_optimize", "trust_from_penalty", "trust_penalty",
           "trustworthiness", "version", "default_transform_epochs", "trust_ambiguous_count", "profile_begin", "profile_end", "trust_fine_fraction",
           "supervised_adjust", "spectral_init"]
