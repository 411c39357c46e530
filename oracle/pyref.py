"""TEST INFRASTRUCTURE: ctypes driver of the real reference (oracle/_ref).

oracle/_ref/libtbsim_ref.so is the reference's own sources
(/root/reference/proj/src/*.cpp + tests/oracles.cpp), compiled unmodified by
oracle/Makefile, plus oracle/ref_shim.cpp (my extern "C" adapter).  Used to
(1) pin the C restatement oracle/oracle.c, (2) generate the committed golden
fixtures under tests/golden/, (3) time the reference CPU path for bench.py's
cpu_baseline / --impl reference.  Never imported by the product.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2404_03226_b200 import abi, outbuf
from paper_2404_03226_b200.batch import GraphBatch
from paper_2404_03226_b200.platform import TYPE_NAMES, platform_array

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libtbsim_ref.so")
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference library missing: {LIB_PATH} (make -C oracle ref)")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        for f in ("ref_gen_layered", "ref_gen_cholesky", "ref_gen_lu", "ref_gen_random",
                  "ref_gen_file", "ref_bench_prepare_layered"):
            getattr(L, f).restype = vp
        L.ref_gen_layered.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint64]
        L.ref_gen_cholesky.argtypes = [C.c_int, C.c_int64]
        L.ref_gen_lu.argtypes = [C.c_int, C.c_int64]
        L.ref_gen_random.argtypes = [C.c_uint64, C.c_int, C.c_double,
                                     C.POINTER(C.c_char_p), C.c_int, C.c_int]
        L.ref_gen_file.argtypes = [C.c_char_p]
        L.ref_exported_sizes.argtypes = [vp, C.POINTER(C.c_int64)]
        L.ref_exported_type_name.argtypes = [vp, C.c_int]
        L.ref_exported_type_name.restype = C.c_char_p
        L.ref_exported_free.argtypes = [vp]
        L.ref_last_error.restype = C.c_char_p
        L.ref_bench_prepare_layered.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_double,
                                                C.POINTER(C.c_uint64), C.POINTER(C.c_int32),
                                                C.POINTER(C.c_int32), C.c_int]
        L.ref_bench_free.argtypes = [vp]
        L.ref_bench_run.argtypes = [vp, C.c_int, C.c_int, C.POINTER(C.c_double),
                                    C.POINTER(C.c_double)]
        _lib = L
    return _lib


class RefError(Exception):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


def _check(status):
    if status:
        raise RefError(status, lib().ref_last_error().decode())


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _exported_to_batch(h) -> GraphBatch:
    L = lib()
    if not h:
        raise RefError(abi.TBSIM_E_INVALID_ARGUMENT, L.ref_last_error().decode())
    try:
        s = (C.c_int64 * 6)()
        L.ref_exported_sizes(h, s)
        n, ne, ni, no, nh, nt = list(s)
        local_names = [L.ref_exported_type_name(h, i).decode() for i in range(nt)]
        doff = np.zeros(n + 1, np.int32); dep = np.zeros(ne, np.int32)
        ioff = np.zeros(n + 1, np.int32); inn = np.zeros(ni, np.int32)
        ooff = np.zeros(n + 1, np.int32); out = np.zeros(no, np.int32)
        ty = np.zeros(n, np.int32); hb = np.zeros(nh, np.int64); tid = np.zeros(n, np.int64)
        L.ref_exported_copy(C.c_void_p(h), _p(doff, C.c_int32), _p(dep, C.c_int32),
                            _p(ioff, C.c_int32), _p(inn, C.c_int32), _p(ooff, C.c_int32),
                            _p(out, C.c_int32), _p(ty, C.c_int32), _p(hb, C.c_int64),
                            _p(tid, C.c_int64))
    finally:
        L.ref_exported_free(C.c_void_p(h))
    names = list(TYPE_NAMES)
    remap = []
    for nm in local_names:
        if nm not in names:
            names.append(nm)
        remap.append(names.index(nm))
    ty = np.array(remap, np.int32)[ty] if n else ty
    return GraphBatch([0, n], [0, ne], [0, nh], [0, ni], [0, no], doff, dep, ioff, inn,
                      ooff, out, ty, hb, names, tid)


def gen_layered(n, layers, p, seed) -> GraphBatch:
    return _exported_to_batch(lib().ref_gen_layered(n, layers, p, seed))


def gen_cholesky(nb, block_bytes) -> GraphBatch:
    return _exported_to_batch(lib().ref_gen_cholesky(nb, block_bytes))


def gen_lu(nb, block_bytes) -> GraphBatch:
    return _exported_to_batch(lib().ref_gen_lu(nb, block_bytes))


def gen_random(seed, n, p, types, with_handles) -> GraphBatch:
    arr = (C.c_char_p * len(types))(*[t.encode() for t in types])
    return _exported_to_batch(lib().ref_gen_random(seed, n, p, arr, len(types), int(with_handles)))


def gen_file(path) -> GraphBatch:
    return _exported_to_batch(lib().ref_gen_file(path.encode()))


def _names(batch):
    arr = (C.c_char_p * len(batch.type_names))(*[t.encode() for t in batch.type_names])
    return arr


def attributes(batch: GraphBatch, costs, request, prio=abi.PRIO_UPWARD_RANK,
               unit_time=None, threads=0):
    """costs: CostTable.  Returns dict of numpy arrays."""
    out, o = outbuf.attr_out(batch.n_tasks, batch.n_graphs, unit_time)
    c, _keep = outbuf.costs_struct(costs, batch.type_names)
    _check(lib().ref_attributes(C.byref(batch.desc()), _names(batch), C.byref(c),
                                request, prio, C.byref(o), threads))
    return out


def simulate(batch: GraphBatch, platforms, policy, platform_of=None, reg=None,
             attrs=None, record=True, threads=0):
    """platforms: list of Platform; policy: name; reg: list of RegulatorCfg or None;
    attrs: dict with ability/efficiency/static_priority arrays (or None)."""
    G = batch.n_graphs
    parr = platform_array(platforms, batch.type_names)
    pof = None if platform_of is None else np.ascontiguousarray(platform_of, np.int32)
    regarr = None if reg is None else (abi.RegulatorCfg * G)(*reg)
    ai, _keep = outbuf.attr_in(attrs)
    out, o = outbuf.sim_out(batch.n_tasks, G, record)
    _check(lib().ref_simulate(C.byref(batch.desc()), _names(batch), parr,
                              None if pof is None else _p(pof, C.c_int32),
                              abi.POLICY_ID[policy], regarr,
                              None if ai is None else C.byref(ai), C.byref(o), threads))
    return out


class BenchSet:
    """Reference-generated layered DAGs + platforms, for CPU timing."""

    def __init__(self, n_dags, n, layers, p, seeds, n_cpus, n_gpus, threads=0):
        L = lib()
        seeds = np.ascontiguousarray(seeds, np.uint64)
        nc = np.ascontiguousarray(np.broadcast_to(n_cpus, (n_dags,)), np.int32)
        ng = np.ascontiguousarray(np.broadcast_to(n_gpus, (n_dags,)), np.int32)
        self.n = n_dags
        self.h = L.ref_bench_prepare_layered(n_dags, n, layers, p, _p(seeds, C.c_uint64),
                                             _p(nc, C.c_int32), _p(ng, C.c_int32), threads)
        if not self.h:
            raise RefError(2, L.ref_last_error().decode())

    def run(self, policy="inspirit", threads=0):
        ms = np.zeros(self.n)
        secs = C.c_double()
        _check(lib().ref_bench_run(C.c_void_p(self.h), abi.POLICY_ID[policy], threads,
                                   _p(ms, C.c_double), C.byref(secs)))
        return secs.value, ms

    def __del__(self):
        try:
            if self.h:
                lib().ref_bench_free(C.c_void_p(self.h))
        except Exception:
            pass


def max_threads() -> int:
    return lib().ref_max_threads()


# ---- C4 scale (oracle/ref_c4.cpp -> _ref/libtbsim_ref_c4.so) --------------

C4_LIB_PATH = os.path.join(HERE, "_ref", "libtbsim_ref_c4.so")
_lib_c4 = None


def lib_c4():
    global _lib_c4
    if _lib_c4 is None:
        if not os.path.exists(C4_LIB_PATH):
            raise RuntimeError(f"reference library missing: {C4_LIB_PATH} (make -C oracle ref)")
        L = C.CDLL(C4_LIB_PATH)
        vp = C.c_void_p
        L.ref_c4_last_error.restype = C.c_char_p
        L.ref_c4_load.restype = vp
        L.ref_c4_load.argtypes = [vp, vp, vp]
        L.ref_c4_free.argtypes = [vp]
        L.ref_c4_structure.argtypes = [vp, C.c_int, vp, vp, vp, vp, vp, vp]
        L.ref_c4_efficiency_sample.argtypes = [vp, vp, C.c_int64, vp, C.c_int, C.c_int, vp, vp]
        _lib_c4 = L
    return _lib_c4


class C4Ref:
    """One large graph (graph 0 of `batch`) held by the reference as a
    TaskGraph: its public attribute API in full, and its internal per-source
    efficiency_of (src/attributes.cpp:110-137) on sampled sources."""

    def __init__(self, batch: GraphBatch, costs):
        L = lib_c4()
        c, self._keep = outbuf.costs_struct(costs, batch.type_names)
        self._names = _names(batch)
        self.n = batch.sizes(0)
        self.h = L.ref_c4_load(C.addressof(batch.desc()), C.addressof(self._names), C.addressof(c))
        if not self.h:
            raise RefError(abi.TBSIM_E_RUNTIME, L.ref_c4_last_error().decode())

    def _chk(self, status):
        if status:
            raise RefError(status, lib_c4().ref_c4_last_error().decode())

    def structure(self, threads=0, ability=True, rank=True, depth=True, layers=True):
        n = self.n
        out = {"ability": np.zeros(n, np.int64) if ability else None,
               "static_priority": np.zeros(n, np.int64) if rank else None,
               "depth": np.zeros(n, np.int64) if depth else None,
               "layer": np.zeros(n, np.int32) if layers else None}
        w0 = C.c_double()
        sec = np.zeros(4)
        ptr = lambda a: None if a is None else a.ctypes.data
        self._chk(lib_c4().ref_c4_structure(self.h, threads, ptr(out["ability"]), ptr(out["static_priority"]),
                                            ptr(out["depth"]), ptr(out["layer"]), C.addressof(w0), sec.ctypes.data))
        out["w0_ms"] = w0.value
        out["seconds"] = dict(zip(("ability", "rank", "depth", "layers"), sec.tolist()))
        return out

    def efficiency_sample(self, sources, windows, threads=0):
        """out[i, k] = efficiency_of(sources[i], windows[k]); (out, setup_s, calls_s)."""
        src = np.ascontiguousarray(sources, np.int64)
        w = np.ascontiguousarray(windows, np.float64)
        out = np.zeros((len(src), len(w)), np.int64)
        sec = np.zeros(2)
        self._chk(lib_c4().ref_c4_efficiency_sample(self.h, src.ctypes.data, len(src), w.ctypes.data, len(w),
                                                    threads, out.ctypes.data, sec.ctypes.data))
        return out, float(sec[0]), float(sec[1])

    def __del__(self):
        try:
            if self.h:
                lib_c4().ref_c4_free(C.c_void_p(self.h))
        except Exception:
            pass
