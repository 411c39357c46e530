"""ctypes mirror of include/tbsim_b200.h (the C-ABI boundary).

Only layouts and constants live here -- no behaviour.  The product library
(libtbsim_b200.so) is loaded by :mod:`paper_2404_03226_b200.lib`; the test
oracles in ``oracle/`` reuse these struct definitions so that every
implementation is fed byte-identical CSR batches.
"""
from __future__ import annotations

import ctypes as C

TBSIM_OK = 0
TBSIM_E_INVALID_ARGUMENT = 1
TBSIM_E_RUNTIME = 2
TBSIM_E_LOGIC = 3
TBSIM_E_OUT_OF_RANGE = 4
TBSIM_E_CUDA = 5

ATTR_ABILITY = 1 << 0
ATTR_EFFICIENCY = 1 << 1
ATTR_CALIBRATE = 1 << 2
ATTR_RANK = 1 << 3
ATTR_DEPTH = 1 << 4
ATTR_LAYERS = 1 << 5
ATTR_ALL = 1 << 6

PRIO_UPWARD_RANK, PRIO_DEPTH, PRIO_ZERO = 0, 1, 2
POLICIES = ("fifo", "dm", "dmda", "dmdap", "inspirit")
POLICY_ID = {n: i for i, n in enumerate(POLICIES)}
MODE_ABILITY, MODE_EFFICIENCY, MODE_LOCALITY = 0, 1, 2
PHASE_INC, PHASE_DEC = 0, 1
MAX_SLOPE_SAMPLES = 64

_p64 = C.POINTER(C.c_int64)
_p32 = C.POINTER(C.c_int32)
_pd = C.POINTER(C.c_double)


class BatchDesc(C.Structure):
    _fields_ = [
        ("n_graphs", C.c_int64),
        ("task_base", _p64), ("edge_base", _p64), ("handle_base", _p64),
        ("in_base", _p64), ("out_base", _p64),
        ("dep_off", _p32), ("dep", _p32),
        ("in_off", _p32), ("in_", _p32),
        ("out_off", _p32), ("out", _p32),
        ("type", _p32), ("handle_bytes", _p64), ("task_id", _p64),
        ("n_type_names", C.c_int32), ("type_names", C.POINTER(C.c_char_p)),
    ]


class Costs(C.Structure):
    _fields_ = [("n_types", C.c_int32), ("cpu_ms", _pd), ("gpu_ms", _pd)]


class PlatformDesc(C.Structure):
    _fields_ = [
        ("n_workers", C.c_int32), ("kind", _p32), ("memory_node", _p32),
        ("n_nodes", C.c_int32), ("latency_ms", C.c_double), ("bandwidth", _pd),
        ("costs", Costs),
    ]


class AttrOut(C.Structure):
    _fields_ = [
        ("ability", _p64), ("efficiency", _p64), ("static_priority", _p64),
        ("depth", _p64), ("layer", _p32), ("unit_time_ms", _pd),
        ("w0_ms", _pd), ("best_score", _p64), ("w0_score", _p64),
        ("evaluations", _p32), ("on_device", C.c_int32),
    ]


class RegulatorCfg(C.Structure):
    _fields_ = [
        ("task_window", C.c_int64), ("s_inc", C.c_int64), ("k_inc", C.c_double),
        ("s_dec", C.c_int64), ("c", C.c_int64), ("dec_step", C.c_int64),
        ("slope_samples", C.c_int32), ("_pad", C.c_int32),
    ]


class RegulatorState(C.Structure):
    _fields_ = [
        ("mode", C.c_int32), ("phase", C.c_int32),
        ("peak", C.c_int64), ("prev_nready", C.c_int64),
        ("last_trigger_nready", C.c_int64), ("s_dec_count", C.c_int64),
        ("cur_k", C.c_double), ("n_samples", C.c_int32), ("_pad", C.c_int32),
        ("sample_time", C.c_double * MAX_SLOPE_SAMPLES),
        ("sample_nready", C.c_int64 * MAX_SLOPE_SAMPLES),
    ]


class AttrIn(C.Structure):
    _fields_ = [("ability", _p64), ("efficiency", _p64),
                ("static_priority", _p64), ("on_device", C.c_int32)]


class SimOut(C.Structure):
    _fields_ = [
        ("worker", _p32), ("start_ms", _pd), ("end_ms", _pd),
        ("makespan_ms", _pd), ("completed", _p64), ("pop_mode_counts", _p64),
        ("reg_state", C.POINTER(RegulatorState)),
        ("push_time", _pd), ("push_task", _p32),
        ("pop_time", _pd), ("pop_task", _p32), ("pop_worker", _p32),
        ("sample_time", _pd), ("sample_nready", _p64),
        ("on_device", C.c_int32),
    ]


def fresh_regulator_state() -> RegulatorState:
    """RegulatorState{} defaults (policies.hpp:89-98): HighEfficiency, Inc,
    s_dec_count = 1, everything else zero."""
    s = RegulatorState()
    s.mode = MODE_EFFICIENCY
    s.phase = PHASE_INC
    s.s_dec_count = 1
    return s
