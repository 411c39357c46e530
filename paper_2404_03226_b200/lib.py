"""Loader of the in-tree CUDA extension libtbsim_b200.so (no fallback).

Importing this module never touches a GPU; ``load()`` dlopens the library and
declares every entry point of include/tbsim_b200.h.  If the library is
missing the product fails loudly -- there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import os

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
# TBSIM_LIB: another in-tree build of the same library (A/B timing of kernel variants)
LIB_PATH = os.path.join(HERE, os.environ.get("TBSIM_LIB", "libtbsim_b200.so"))

# Every symbol the header declares (tests check the .so exports all of them).
EXPORTS = [
    "tbsim_last_error", "tbsim_abi_version",
    "tbsim_ctx_create", "tbsim_ctx_destroy", "tbsim_ctx_set_stream", "tbsim_ctx_set_upload_stream", "tbsim_ctx_synchronize",
    "tbsim_ctx_launch_count", "tbsim_ctx_set_timing", "tbsim_ctx_last_kernel_ms",
    "tbsim_ctx_set_large_graph_threshold",
    "tbsim_ctx_set_sweep_tile",
    "tbsim_ctx_set_async_results",
    "tbsim_attributes_shard_partial",
    "tbsim_attributes_shard_finish",
    "tbsim_ctx_last_sweep_relaxations",
    "tbsim_ctx_last_sim_shape",
    "tbsim_probe_sweep_peak",
    "tbsim_batch_upload", "tbsim_batch_free", "tbsim_batch_h2d_bytes", "tbsim_batch_generate_layered",
    "tbsim_batch_generate_tiled",
    "tbsim_batch_sizes", "tbsim_batch_download",
    "tbsim_attributes", "tbsim_simulate", "tbsim_schedule", "tbsim_default_regulator_config",
    "tbsim_hostbatch_new", "tbsim_hostbatch_free", "tbsim_hostbatch_add_layered",
    "tbsim_hostbatch_add_cholesky", "tbsim_hostbatch_add_lu", "tbsim_hostbatch_add_qr",
    "tbsim_hostbatch_add_csr", "tbsim_hostbatch_desc", "tbsim_hostbatch_save", "tbsim_hostbatch_load", "tbsim_hostbatch_set_type_names",
    "tbsim_batch_desc_save",
    "tbsim_type_count", "tbsim_type_name",
    "tbsim_default_costs",
]

_lib = None


class ExtensionMissing(RuntimeError):
    pass


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ExtensionMissing(
            f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    P = C.POINTER
    L.tbsim_last_error.restype = C.c_char_p
    L.tbsim_ctx_create.argtypes = [C.c_int, P(vp)]
    L.tbsim_ctx_destroy.argtypes = [vp]
    L.tbsim_ctx_set_stream.argtypes = [vp, vp]
    L.tbsim_ctx_set_upload_stream.argtypes = [vp, vp]
    L.tbsim_ctx_synchronize.argtypes = [vp]
    L.tbsim_ctx_launch_count.argtypes = [vp]
    L.tbsim_ctx_launch_count.restype = i64
    L.tbsim_ctx_set_timing.argtypes = [vp, C.c_int]
    L.tbsim_ctx_set_large_graph_threshold.argtypes = [vp, i64]
    L.tbsim_ctx_set_sweep_tile.argtypes = [vp, i32]
    L.tbsim_ctx_set_async_results.argtypes = [vp, C.c_int]
    L.tbsim_attributes_shard_partial.argtypes = [vp, vp, P(abi.Costs), i32, i32, P(i64), P(i64), i64, P(i64)]
    L.tbsim_attributes_shard_finish.argtypes = [vp, vp, P(i64), i64, i32, P(abi.AttrOut)]
    L.tbsim_ctx_last_sweep_relaxations.argtypes = [vp, P(i64), P(i64)]
    L.tbsim_ctx_last_sim_shape.argtypes = [vp, P(i32), P(i32), P(i32)]
    L.tbsim_probe_sweep_peak.argtypes = [vp, i32, P(dbl), P(dbl)]
    L.tbsim_ctx_last_kernel_ms.argtypes = [vp, C.c_char_p, P(dbl)]
    L.tbsim_batch_upload.argtypes = [vp, P(abi.BatchDesc), P(vp)]
    L.tbsim_batch_free.argtypes = [vp, vp]
    L.tbsim_batch_h2d_bytes.argtypes = [vp]
    L.tbsim_batch_h2d_bytes.restype = i64
    L.tbsim_batch_generate_layered.argtypes = [vp, i32, i32, dbl, P(C.c_uint64), i64, P(vp)]
    L.tbsim_batch_generate_tiled.argtypes = [vp, i32, i32, i64, i64, P(vp)]
    L.tbsim_batch_sizes.argtypes = [vp, P(i64)]
    L.tbsim_batch_download.argtypes = [vp, vp, P(abi.BatchDesc)]
    L.tbsim_attributes.argtypes = [vp, vp, P(abi.Costs), i32, i32, P(abi.AttrOut)]
    L.tbsim_simulate.argtypes = [vp, vp, P(abi.PlatformDesc), i32, P(i32), i32,
                                 P(abi.RegulatorCfg), P(abi.AttrIn), P(abi.SimOut)]
    L.tbsim_schedule.argtypes = [vp, vp, P(abi.PlatformDesc), i32, P(i32), i32, i32,
                                 P(abi.AttrOut), P(abi.SimOut)]
    L.tbsim_default_regulator_config.argtypes = [i32, dbl, P(abi.RegulatorCfg)]
    L.tbsim_hostbatch_new.argtypes = [P(vp)]
    L.tbsim_hostbatch_free.argtypes = [vp]
    L.tbsim_hostbatch_add_layered.argtypes = [vp, i32, i32, dbl, P(C.c_uint64), i64, i32]
    L.tbsim_hostbatch_add_cholesky.argtypes = [vp, i32, i64]
    L.tbsim_hostbatch_add_lu.argtypes = [vp, i32, i64]
    L.tbsim_hostbatch_add_qr.argtypes = [vp, i32, i64]
    L.tbsim_hostbatch_add_csr.argtypes = [vp, i32, P(i32), P(i32), P(i32), P(i32), P(i32), P(i32),
                                          P(i32), i32, P(i64), P(i64)]
    L.tbsim_hostbatch_desc.argtypes = [vp, P(abi.BatchDesc)]
    L.tbsim_hostbatch_save.argtypes = [vp, C.c_char_p]
    L.tbsim_hostbatch_set_type_names.argtypes = [vp, i32, P(C.c_char_p)]
    L.tbsim_hostbatch_load.argtypes = [C.c_char_p, P(vp)]
    L.tbsim_batch_desc_save.argtypes = [P(abi.BatchDesc), C.c_char_p]
    L.tbsim_type_name.restype = C.c_char_p
    L.tbsim_default_costs.argtypes = [P(dbl), P(dbl)]
    _lib = L
    return L
