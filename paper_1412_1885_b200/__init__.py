"""B200-native (sm_100a) randomized Tucker decomposition hot path of arXiv 1412.1885.

The compute (multi-mode TTM sketches, tall-skinny pivoted QR, core projection) runs in
hand-written CUDA kernels behind the C-ABI of include/tenkit_b200.h
(paper_1412_1885_b200/lib/libtenkit_b200.so); `tenkit` mirrors the reference's API.
"""
from .tenkit import (SeedSpec, DenseTensor, TuckerModel, StopRule, ConstraintSpec, ConstraintKind,  # noqa: F401
                     Context, rand_tucker_2i, rand_tucker, ttm, ttm_all, unfold_times, orthonormal_basis,
                     gram_orthonormalize, gram_ortho_transform,
                     gaussian_matrix, ffcp, CpModel, model_fit, TenkitError)

__version__ = "0.1.0"
