"""paper_1207_4684_b200 -- B200-native (sm_100a) hot path of the Fast Cauchy Transform l1-conditioning
pipeline (Clarkson et al., arXiv 1207.4684): FCT1 sketch, conditioning, l1 row-norm estimation and
l1 row sampling, behind the C ABI in include/fct.h (libfct.so, built from csrc/ by build.py).

The Python layer only marshals torch tensors into that ABI; there is no CPU fallback.
"""
from ._lib import FctError, load  # noqa: F401
from .api import (  # noqa: F401
    HostPipeline,
    Pipeline,
    fct_condition,
    fct2_sketch,
    fct_sketch,
    l1_coreset_gather,
    l1_coreset_regression,
    l1_lad_solve,
    l1_probs,
    l1_probs_sample,
    l1_rownorm,
    l1_rownorm_exact,
    l1_rownorm_probs,
    l1_sample,
    l1_sample_multinomial,
    l1_sample_u,
    trim,
)

__version__ = "0.1.0"
