"""TEST INFRASTRUCTURE: ctypes driver of the C restatement oracle/oracle.c.

The checker the CUDA product is compared against in tests/, in
__graft_entry__.smoke() and in bench.py's cpu_baseline leg -- never the
thing measured or shipped.  Same call shapes as oracle/pyref.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2404_03226_b200 import abi, outbuf
from paper_2404_03226_b200.batch import GraphBatch
from paper_2404_03226_b200.platform import TYPE_NAMES, platform_array

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
_lib = None


class OracleError(Exception):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


class OrcGraph(C.Structure):
    _fields_ = [("n", C.c_int32), ("n_dep", C.c_int32), ("n_in", C.c_int32),
                ("n_out", C.c_int32), ("n_handles", C.c_int32),
                ("dep_off", C.POINTER(C.c_int32)), ("dep", C.POINTER(C.c_int32)),
                ("in_off", C.POINTER(C.c_int32)), ("in_", C.POINTER(C.c_int32)),
                ("out_off", C.POINTER(C.c_int32)), ("out", C.POINTER(C.c_int32)),
                ("type", C.POINTER(C.c_int32)), ("handle_bytes", C.POINTER(C.c_int64))]


def build():
    subprocess.check_call(["make", "-s", "-C", HERE])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        L.orc_calculate_k.restype = C.c_double
        L.orc_calculate_k.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int]
        L.orc_regulator_step.argtypes = [C.POINTER(abi.RegulatorState),
                                         C.POINTER(abi.RegulatorCfg), C.c_int64, C.c_double]
        L.orc_gen_layered.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_uint64,
                                      C.POINTER(OrcGraph)]
        L.orc_gen_cholesky.argtypes = [C.c_int32, C.c_int64, C.POINTER(OrcGraph)]
        L.orc_gen_lu.argtypes = [C.c_int32, C.c_int64, C.POINTER(OrcGraph)]
        _lib = L
    return _lib


def _check(status):
    if status:
        raise OracleError(status, lib().orc_last_error().decode())


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def attributes(batch: GraphBatch, costs, request, prio=abi.PRIO_UPWARD_RANK, unit_time=None):
    out, o = outbuf.attr_out(batch.n_tasks, batch.n_graphs, unit_time)
    c, _keep = outbuf.costs_struct(costs, batch.type_names)
    _check(lib().orc_attributes(C.byref(batch.desc()), C.byref(c), request, prio, C.byref(o)))
    return out


def simulate(batch: GraphBatch, platforms, policy, platform_of=None, reg=None, attrs=None,
             record=True, states=None):
    G = batch.n_graphs
    parr = platform_array(platforms, batch.type_names)
    pof = None if platform_of is None else np.ascontiguousarray(platform_of, np.int32)
    regarr = None if reg is None else (abi.RegulatorCfg * G)(*reg)
    ai, _keep = outbuf.attr_in(attrs)
    out, o = outbuf.sim_out(batch.n_tasks, G, record, states)
    _check(lib().orc_simulate(C.byref(batch.desc()), parr,
                              None if pof is None else _p(pof, C.c_int32),
                              abi.POLICY_ID[policy], regarr,
                              None if ai is None else C.byref(ai), C.byref(o)))
    return out


def default_regulator_config(batch: GraphBatch, g: int, platform) -> abi.RegulatorCfg:
    parr = platform_array([platform], batch.type_names)
    cfg = abi.RegulatorCfg()
    _check(lib().orc_default_regulator_config(C.byref(batch.desc()), C.c_int64(g), parr,
                                              C.byref(cfg)))
    return cfg


def calculate_k(samples):
    t = np.array([x for x, _ in samples] or [0.0], np.float64)
    y = np.array([v for _, v in samples] or [0], np.int64)
    return lib().orc_calculate_k(_p(t, C.c_double), _p(y, C.c_int64), len(samples))


def regulator_step(state: abi.RegulatorState, cfg: abi.RegulatorCfg, cur: int, now: float):
    lib().orc_regulator_step(C.byref(state), C.byref(cfg), cur, now)


def _graph_to_batch(g: OrcGraph) -> GraphBatch:
    n = g.n
    arr = lambda p, k, dt: np.ctypeslib.as_array(p, (k,)).astype(dt) if k > 0 else np.zeros(0, dt)
    b = GraphBatch([0, n], [0, g.n_dep], [0, g.n_handles], [0, g.n_in], [0, g.n_out],
                   arr(g.dep_off, n + 1, np.int32), arr(g.dep, g.n_dep, np.int32),
                   arr(g.in_off, n + 1, np.int32), arr(g.in_, g.n_in, np.int32),
                   arr(g.out_off, n + 1, np.int32), arr(g.out, g.n_out, np.int32),
                   arr(g.type, n, np.int32), arr(g.handle_bytes, g.n_handles, np.int64),
                   TYPE_NAMES, np.arange(n, dtype=np.int64))
    lib().orc_graph_free(C.byref(g))
    return b


def gen_layered(n, layers, p, seed) -> GraphBatch:
    g = OrcGraph()
    _check(lib().orc_gen_layered(n, layers, p, seed, C.byref(g)))
    return _graph_to_batch(g)


def gen_cholesky(nb, block_bytes) -> GraphBatch:
    g = OrcGraph()
    _check(lib().orc_gen_cholesky(nb, block_bytes, C.byref(g)))
    return _graph_to_batch(g)


def gen_lu(nb, block_bytes) -> GraphBatch:
    g = OrcGraph()
    _check(lib().orc_gen_lu(nb, block_bytes, C.byref(g)))
    return _graph_to_batch(g)
