"""Host output buffers for the C-ABI result structs (tbsim_attr_out /
tbsim_sim_out), shared by the product binding and the test oracles so every
implementation writes into identically shaped numpy arrays."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi


def _p(a, ct):
    return None if a is None else a.ctypes.data_as(C.POINTER(ct))


def attr_out(T: int, G: int, unit_time=None):
    out = {"ability": np.zeros(T, np.int64), "efficiency": np.zeros(T, np.int64),
           "static_priority": np.zeros(T, np.int64), "depth": np.zeros(T, np.int64),
           "layer": np.zeros(T, np.int32),
           "unit_time_ms": (np.ascontiguousarray(unit_time, np.float64).copy()
                            if unit_time is not None else np.zeros(G, np.float64)),
           "w0_ms": np.zeros(G), "best_score": np.zeros(G, np.int64),
           "w0_score": np.zeros(G, np.int64), "evaluations": np.zeros(G, np.int32)}
    o = abi.AttrOut(_p(out["ability"], C.c_int64), _p(out["efficiency"], C.c_int64),
                    _p(out["static_priority"], C.c_int64), _p(out["depth"], C.c_int64),
                    _p(out["layer"], C.c_int32), _p(out["unit_time_ms"], C.c_double),
                    _p(out["w0_ms"], C.c_double), _p(out["best_score"], C.c_int64),
                    _p(out["w0_score"], C.c_int64), _p(out["evaluations"], C.c_int32), 0)
    return out, o


def sim_out(T: int, G: int, record: bool, states=None, want_states=True, arrays=None):
    """arrays: optional dict of preallocated (ideally pinned) numpy outputs."""
    if arrays is not None:
        out = dict(arrays)
    else:
        out = {"worker": np.zeros(T, np.int32), "start_ms": np.zeros(T), "end_ms": np.zeros(T),
               "makespan_ms": np.zeros(G), "completed": np.zeros(G, np.int64),
               "pop_mode_counts": np.zeros(3 * G, np.int64)}
    if states is None and want_states:
        states = (abi.RegulatorState * max(G, 1))()
        fresh = abi.fresh_regulator_state()
        for i in range(G):
            states[i] = fresh
    o = abi.SimOut()
    o.worker = _p(out["worker"], C.c_int32)
    o.start_ms = _p(out["start_ms"], C.c_double)
    o.end_ms = _p(out["end_ms"], C.c_double)
    o.makespan_ms = _p(out["makespan_ms"], C.c_double)
    o.completed = _p(out["completed"], C.c_int64)
    o.pop_mode_counts = _p(out.get("pop_mode_counts"), C.c_int64)
    o.reg_state = states
    if record:
        out.update(push_time=np.zeros(T), push_task=np.zeros(T, np.int32),
                   pop_time=np.zeros(T), pop_task=np.zeros(T, np.int32),
                   pop_worker=np.zeros(T, np.int32), sample_time=np.zeros(2 * T),
                   sample_nready=np.zeros(2 * T, np.int64))
        o.push_time = _p(out["push_time"], C.c_double)
        o.push_task = _p(out["push_task"], C.c_int32)
        o.pop_time = _p(out["pop_time"], C.c_double)
        o.pop_task = _p(out["pop_task"], C.c_int32)
        o.pop_worker = _p(out["pop_worker"], C.c_int32)
        o.sample_time = _p(out["sample_time"], C.c_double)
        o.sample_nready = _p(out["sample_nready"], C.c_int64)
    out["reg_state"] = states
    return out, o


def attr_in(attrs):
    """tbsim_attr_in over a dict of ability/efficiency/static_priority."""
    if attrs is None:
        return None, []
    ai = abi.AttrIn()
    keep = []
    for k in ("ability", "efficiency", "static_priority"):
        if attrs.get(k) is not None:
            a = np.ascontiguousarray(attrs[k], np.int64)
            keep.append(a)
            setattr(ai, k, _p(a, C.c_int64))
    return ai, keep


def costs_struct(costs, type_names):
    cpu, gpu = costs.arrays(type_names)
    c = abi.Costs(len(type_names), _p(cpu, C.c_double), _p(gpu, C.c_double))
    return c, (cpu, gpu)


def state_dict(s: abi.RegulatorState) -> dict:
    n = s.n_samples
    return {"mode": s.mode, "phase": s.phase, "peak": s.peak, "prev_nready": s.prev_nready,
            "last_trigger_nready": s.last_trigger_nready, "s_dec_count": s.s_dec_count,
            "cur_k": s.cur_k, "samples": [(s.sample_time[i], s.sample_nready[i]) for i in range(n)]}
