"""ctypes loader for libfct.so (the C ABI declared in include/fct.h).  No compute happens here."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfct.so")
_lib = None

_i64, _i32, _u64, _vp, _sz, _int = (ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_void_p,
                                    ctypes.c_size_t, ctypes.c_int)

# name -> (restype, argtypes); mirrors include/fct.h one to one
SIGNATURES = {
    "fct_last_error": (ctypes.c_char_p, []),
    "fct_version": (ctypes.c_char_p, []),
    "fct_launch_count": (_u64, []),
    "fct_last_instance": (ctypes.c_int, [ctypes.c_int32, ctypes.c_char_p, ctypes.c_size_t]),
    "fct_sketch_workspace_bytes": (_sz, [_i64, _i64, _i32, _i32]),
    "fct_sketch": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _i32, _i32, _vp, _int, _vp, _sz, _vp]),
    "fct_condition_workspace_bytes": (_sz, [_i32, _i64]),
    "fct_condition": (_int, [_vp, _i32, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "l1_rownorm_workspace_bytes": (_sz, [_i64, _i64, _i32]),
    "l1_rownorm": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _i32, _vp, _vp, _vp, _sz, _vp]),
    "l1_rownorm_exact_workspace_bytes": (_sz, [_i64, _i64]),
    "l1_rownorm_exact": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "l1_probs": (_int, [_vp, _i64, _vp, _vp, _vp]),
    "l1_rownorm_probs": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "l1_sample_workspace_bytes": (_sz, [_i64]),
    "l1_sample": (_int, [_vp, _i64, _i64, _i64, _u64, _vp, _vp, _i64, _vp, _vp, _sz, _vp]),
    "l1_sample_u": (_int, [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _sz, _vp]),
    "l1_sample_multinomial_workspace_bytes": (_sz, [_i64]),
    "l1_sample_multinomial": (_int, [_vp, _i64, _i64, _u64, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "l1_coreset_gather": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _i64, _i64, _vp, _i64, _vp]),
    "l1_lad_workspace_bytes": (_sz, [_i64, _i64]),
    "l1_lad_solve": (_int, [_vp, _vp, _i64, _i64, _i64, _i32, ctypes.c_double, _vp, _vp, _vp, _sz, _vp]),
    "fct2_workspace_bytes": (_sz, [_i64, _i64, _i32, _i32, _i32]),
    "fct2_sketch": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _sz, _vp]),
    "l1_probs_sample_workspace_bytes": (_sz, [_i64]),
    "l1_probs_sample": (_int, [_vp, _i64, _vp, _i64, _i64, _u64, _vp, _vp, _vp, _i64, _vp, _vp, _sz, _vp]),
    "fct_pipeline_workspace_bytes": (_sz, [_i64, _i64, _i32, _i32, _i32]),
    "fct_pipeline": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _i32, _i32, _vp, _i32, _i64, _u64,
                            _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "fct_pipeline_aux_bytes": (_sz, [_i64, _i64, _i32, _i32]),
    "fct_pipeline_host_workspace_bytes": (_sz, [_i64, _i64, _i32, _i32, _i32, _i64]),
    "fct_pipeline_host": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _i32, _i32, _vp, _i32, _i64, _u64,
                                 _vp, _vp, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
}

STATUS = {0: "FCT_OK", -1: "FCT_ERR_ARG", -2: "FCT_ERR_SHAPE", -3: "FCT_ERR_CUDA", -4: "FCT_ERR_CAPACITY",
          -5: "FCT_ERR_SINGULAR", -6: "FCT_ERR_UNSUPPORTED", -7: "FCT_ERR_WORKSPACE"}


class FctError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


def load(path: str | None = None):
    """Load libfct.so; raises (loudly) if the CUDA library has not been built."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(f"libfct.so not found at {p}: run `python -m paper_1207_4684_b200.build` "
                           "(there is no CPU fallback)")
    lib = ctypes.CDLL(p)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(code: int):
    if code != 0:
        raise FctError(code, load().fct_last_error().decode())
