"""Python host API over the C-ABI: the reference's operator surface
(compute_attributes, simulate, the bench-cell "schedule" pipeline) for whole
batches of DAGs on one B200.

Errors carry the reference's exception type (``TbsimError.kind`` is
``invalid_argument`` / ``runtime_error`` / ``logic_error`` /
``out_of_range``) and its message text.
"""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from . import abi, outbuf
from .batch import GraphBatch
from .lib import load
from .platform import TYPE_NAMES, CostTable, Platform, platform_array

_KIND = {abi.TBSIM_E_INVALID_ARGUMENT: "invalid_argument", abi.TBSIM_E_RUNTIME: "runtime_error",
         abi.TBSIM_E_LOGIC: "logic_error", abi.TBSIM_E_OUT_OF_RANGE: "out_of_range",
         abi.TBSIM_E_CUDA: "cuda"}


class TbsimError(Exception):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status
        self.kind = _KIND.get(status, "unknown")


class TbsimInvalidArgument(TbsimError, ValueError):
    pass


class TbsimRuntimeError(TbsimError, RuntimeError):
    pass


def _check(status: int):
    if status:
        msg = load().tbsim_last_error().decode()
        cls = TbsimInvalidArgument if status == abi.TBSIM_E_INVALID_ARGUMENT else \
            TbsimRuntimeError if status in (abi.TBSIM_E_RUNTIME, abi.TBSIM_E_CUDA) else TbsimError
        raise cls(status, msg)


def _p(a, ct):
    return None if a is None else a.ctypes.data_as(C.POINTER(ct))


# ------------------------------------------------------------ host batches

class HostBatch:
    """Packed host batch produced by the C++ generators (pinned memory when a
    CUDA runtime is present).  ``view()`` exposes it as a GraphBatch of numpy
    arrays sharing the same memory (for the oracle / tests)."""

    def __init__(self):
        self._h = C.c_void_p()
        _check(load().tbsim_hostbatch_new(C.byref(self._h)))
        self._desc = None

    def add_layered(self, n_tasks, n_layers, edge_prob, seeds, threads=0):
        seeds = np.ascontiguousarray(seeds, np.uint64)
        _check(load().tbsim_hostbatch_add_layered(self._h, n_tasks, n_layers, edge_prob,
                                                  _p(seeds, C.c_uint64), len(seeds), threads))
        return self

    def add_cholesky(self, nblocks, block_bytes):
        _check(load().tbsim_hostbatch_add_cholesky(self._h, nblocks, block_bytes))
        return self

    def add_lu(self, nblocks, block_bytes):
        _check(load().tbsim_hostbatch_add_lu(self._h, nblocks, block_bytes))
        return self

    def add_qr(self, nblocks, block_bytes):
        _check(load().tbsim_hostbatch_add_qr(self._h, nblocks, block_bytes))
        return self

    def add_batch(self, gb: GraphBatch):
        if list(gb.type_names) != list(TYPE_NAMES):
            names = (C.c_char_p * len(gb.type_names))(*[t.encode() for t in gb.type_names])
            _check(load().tbsim_hostbatch_set_type_names(self._h, len(gb.type_names), names))
        for g in range(gb.n_graphs):
            one = gb._one(g)
            n = one.n_tasks
            _check(load().tbsim_hostbatch_add_csr(
                self._h, n, _p(one.dep_off, C.c_int32), _p(one.dep, C.c_int32),
                _p(one.in_off, C.c_int32), _p(one.in_, C.c_int32), _p(one.out_off, C.c_int32),
                _p(one.out, C.c_int32), _p(one.type, C.c_int32), len(one.handle_bytes),
                _p(one.handle_bytes, C.c_int64), _p(one.task_id, C.c_int64)))
        return self

    def save(self, path: str) -> "HostBatch":
        """Binary CSR cache of this batch (tbsim_hostbatch_save)."""
        _check(load().tbsim_hostbatch_save(self._h, str(path).encode()))
        return self

    @classmethod
    def load(cls, path: str) -> "HostBatch":
        """A batch from a binary CSR cache (tbsim_hostbatch_load): sections
        read straight into pinned memory, ready for Context.upload."""
        hb = cls.__new__(cls)
        hb._h = C.c_void_p()
        hb._desc = None
        _check(load().tbsim_hostbatch_load(str(path).encode(), C.byref(hb._h)))
        return hb

    def desc(self) -> abi.BatchDesc:
        if self._desc is None:
            d = abi.BatchDesc()
            _check(load().tbsim_hostbatch_desc(self._h, C.byref(d)))
            self._desc = d
        return self._desc

    def view(self) -> GraphBatch:
        d = self.desc()
        G = d.n_graphs
        arr = lambda p, n, dt: np.ctypeslib.as_array(p, (n,)).view(dt) if n > 0 else np.zeros(0, dt)
        tb = arr(d.task_base, G + 1, np.int64)
        eb = arr(d.edge_base, G + 1, np.int64)
        hb = arr(d.handle_base, G + 1, np.int64)
        ib = arr(d.in_base, G + 1, np.int64)
        ob = arr(d.out_base, G + 1, np.int64)
        T = int(tb[-1])
        gb = GraphBatch(tb, eb, hb, ib, ob, arr(d.dep_off, T + G, np.int32), arr(d.dep, int(eb[-1]), np.int32),
                        arr(d.in_off, T + G, np.int32), arr(d.in_, int(ib[-1]), np.int32),
                        arr(d.out_off, T + G, np.int32), arr(d.out, int(ob[-1]), np.int32),
                        arr(d.type, T, np.int32), arr(d.handle_bytes, int(hb[-1]), np.int64),
                        [d.type_names[i].decode() for i in range(d.n_type_names)] if d.type_names else TYPE_NAMES,
                        None if not d.task_id else arr(d.task_id, T, np.int64))
        gb._owner = self
        return gb

    def __del__(self):
        try:
            if self._h:
                load().tbsim_hostbatch_free(self._h)
                self._h = C.c_void_p()
        except Exception:
            pass


# ----------------------------------------------------------------- context

class DeviceBatch:
    def __init__(self, ctx: "Context", handle, n_tasks, n_graphs, type_names):
        self.ctx, self.h = ctx, handle
        self.n_tasks, self.n_graphs, self.type_names = n_tasks, n_graphs, type_names

    @property
    def h2d_bytes(self) -> int:
        return load().tbsim_batch_h2d_bytes(self.h)

    def download(self) -> GraphBatch:
        """Copy the device CSR back to host numpy arrays (tests, debugging)."""
        sz = (C.c_int64 * 6)()
        _check(load().tbsim_batch_sizes(self.h, sz))
        G, T, E, H, I, O = list(sz)
        z = lambda k, dt: np.zeros(k, dt)
        gb = GraphBatch(z(G + 1, np.int64), z(G + 1, np.int64), z(G + 1, np.int64), z(G + 1, np.int64),
                        z(G + 1, np.int64), z(T + G, np.int32), z(E, np.int32), z(T + G, np.int32), z(I, np.int32),
                        z(T + G, np.int32), z(O, np.int32), z(T, np.int32), z(H, np.int64), self.type_names)
        _check(load().tbsim_batch_download(self.ctx.h, self.h, C.byref(gb.desc())))
        return gb

    def free(self):
        if self.h:
            _check(load().tbsim_batch_free(self.ctx.h, self.h))
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Context:
    """One CUDA device + stream (tbsim_ctx)."""

    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        _check(load().tbsim_ctx_create(device, C.byref(self.h)))

    def close(self):
        if self.h:
            load().tbsim_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def set_stream(self, stream_ptr: int | None):
        _check(load().tbsim_ctx_set_stream(self.h, C.c_void_p(stream_ptr or 0)))

    def set_upload_stream(self, stream_ptr: int | None):
        """Run batch uploads on this stream (overlapping the compute stream's
        kernels); compute calls wait for a batch's copies on the device."""
        _check(load().tbsim_ctx_set_upload_stream(self.h, C.c_void_p(stream_ptr or 0)))

    def synchronize(self):
        _check(load().tbsim_ctx_synchronize(self.h))

    @property
    def launch_count(self) -> int:
        return load().tbsim_ctx_launch_count(self.h)

    def set_large_graph_threshold(self, n_tasks: int):
        _check(load().tbsim_ctx_set_large_graph_threshold(self.h, n_tasks))

    def last_sim_shape(self) -> dict:
        """Launch shape of the last simulation (DAGs in flight per SM, ...)."""
        a, b, c = C.c_int32(0), C.c_int32(0), C.c_int32(0)
        _check(load().tbsim_ctx_last_sim_shape(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return {"warps_per_sm": a.value, "state_in_smem": bool(b.value), "queue_capacity": c.value}

    def last_sweep_relaxations(self) -> tuple[int, int]:
        """Relaxations executed by the last timed efficiency sweep:
        (in FP64 windows, in FP32-exact windows)."""
        a, b = C.c_int64(0), C.c_int64(0)
        _check(load().tbsim_ctx_last_sweep_relaxations(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def probe_sweep_peak(self, repeats: int = 3) -> tuple[float, float]:
        """Relaxations/s of the sweep's inner loop alone (its roofline):
        (FP64 windows, FP32-exact windows)."""
        a, b = C.c_double(0.0), C.c_double(0.0)
        _check(load().tbsim_probe_sweep_peak(self.h, repeats, C.byref(a), C.byref(b)))
        return a.value, b.value

    def set_async_results(self, on: bool):
        """schedule() with host outputs returns once their D2H copies are
        queued (overlapping the next call); read them after synchronize()."""
        _check(load().tbsim_ctx_set_async_results(self.h, int(on)))

    def set_sweep_tile(self, sources: int):
        """Force the efficiency sweep's sources per tile (0: automatic)."""
        _check(load().tbsim_ctx_set_sweep_tile(self.h, sources))

    def set_timing(self, on: bool):
        _check(load().tbsim_ctx_set_timing(self.h, int(on)))

    def last_kernel_ms(self, name: str) -> float:
        v = C.c_double()
        _check(load().tbsim_ctx_last_kernel_ms(self.h, name.encode(), C.byref(v)))
        return v.value

    # -------------------------------------------------------------- upload
    def upload(self, batch) -> DeviceBatch:
        """batch: GraphBatch (numpy) or HostBatch (pinned)."""
        desc = batch.desc()
        names = batch.type_names if isinstance(batch, GraphBatch) else TYPE_NAMES
        h = C.c_void_p()
        _check(load().tbsim_batch_upload(self.h, C.byref(desc), C.byref(h)))
        T = int(desc.task_base[desc.n_graphs])
        return DeviceBatch(self, h, T, int(desc.n_graphs), names)

    def generate_layered(self, n_tasks, n_layers, edge_prob, seeds) -> DeviceBatch:
        """generate_layered_dag for every seed, built directly in HBM."""
        seeds = np.ascontiguousarray(seeds, np.uint64)
        h = C.c_void_p()
        _check(load().tbsim_batch_generate_layered(self.h, n_tasks, n_layers, edge_prob,
                                                   _p(seeds, C.c_uint64), len(seeds), C.byref(h)))
        return DeviceBatch(self, h, n_tasks * len(seeds), len(seeds), TYPE_NAMES)

    def generate_tiled(self, kind: str, nblocks: int, block_bytes: int, count: int = 1) -> DeviceBatch:
        """`count` copies of a tiled Cholesky / LU / QR DAG built directly in
        HBM (bit-identical to HostBatch.add_cholesky / add_lu / add_qr)."""
        k = {"cholesky": 0, "lu": 1, "qr": 2}[kind]
        h = C.c_void_p()
        _check(load().tbsim_batch_generate_tiled(self.h, k, nblocks, block_bytes, count, C.byref(h)))
        n = api_tiled_tasks(kind, nblocks)
        return DeviceBatch(self, h, n * count, count, TYPE_NAMES)

    # ---------------------------------------------------------- attributes
    def attributes(self, db: DeviceBatch, costs: CostTable, request: int,
                   prio: int = abi.PRIO_UPWARD_RANK, unit_time=None) -> dict:
        out, o = outbuf.attr_out(db.n_tasks, db.n_graphs, unit_time)
        c, _keep = outbuf.costs_struct(costs, db.type_names)
        _check(load().tbsim_attributes(self.h, db.h, C.byref(c), request, prio, C.byref(o)))
        return out

    def attributes_shard_partial(self, db: DeviceBatch, costs: CostTable, rank: int, world: int):
        """Rank `rank` of `world`: partial ability [T] and per-class window
        sums of one large graph (tbsim_attributes_shard_partial); the caller
        sums both over the ranks, then calls attributes_shard_finish."""
        T = db.n_tasks
        ab = np.zeros(T, np.int64)
        sums = np.zeros(max(12 * T, 12), np.int64)
        nw = C.c_int64(0)
        c, _keep = outbuf.costs_struct(costs, db.type_names)
        _check(load().tbsim_attributes_shard_partial(self.h, db.h, C.byref(c), rank, world, _p(ab, C.c_int64),
                                                     _p(sums, C.c_int64), sums.size, C.byref(nw)))
        return ab, sums[:nw.value].copy()

    def attributes_shard_finish(self, db: DeviceBatch, class_sums, prio: int = abi.PRIO_UPWARD_RANK) -> dict:
        """This rank's sources' efficiency (zero elsewhere), the static
        priority and the calibration, from the class sums of all ranks."""
        sums = np.ascontiguousarray(class_sums, np.int64)
        out, o = outbuf.attr_out(db.n_tasks, db.n_graphs)
        _check(load().tbsim_attributes_shard_finish(self.h, db.h, _p(sums, C.c_int64), sums.size, prio, C.byref(o)))
        for k in ("ability", "depth", "layer"):
            out.pop(k)
        return out

    def attributes_sharded(self, db: DeviceBatch, costs: CostTable, rank: int, world: int, allreduce_sum,
                           prio: int = abi.PRIO_UPWARD_RANK) -> dict:
        """compute_attributes of one large graph over `world` ranks; `allreduce_sum`
        sums an int64 numpy array over the ranks (e.g. NCCL all-reduce)."""
        ab, sums = self.attributes_shard_partial(db, costs, rank, world)
        ab = allreduce_sum(ab)
        sums = allreduce_sum(sums)
        out = self.attributes_shard_finish(db, sums, prio)
        out["efficiency"] = allreduce_sum(out["efficiency"])
        out["ability"] = ab
        return out

    # ------------------------------------------------------------ simulate
    def simulate(self, db: DeviceBatch, platforms: Sequence[Platform], policy: str,
                 reg, platform_of=None, attrs=None, record=True, states=None) -> dict:
        G = db.n_graphs
        parr = platform_array(platforms, db.type_names)
        pof = None if platform_of is None else np.ascontiguousarray(platform_of, np.int32)
        regarr = (abi.RegulatorCfg * max(G, 1))(*reg)
        ai, _keep = outbuf.attr_in(attrs)
        out, o = outbuf.sim_out(db.n_tasks, G, record, states)
        _check(load().tbsim_simulate(self.h, db.h, parr, len(platforms), _p(pof, C.c_int32),
                                     abi.POLICY_ID[policy], regarr,
                                     None if ai is None else C.byref(ai), C.byref(o)))
        return out

    # ------------------------------------------------------------ schedule
    def schedule(self, db: DeviceBatch, platforms: Sequence[Platform], policy: str = "inspirit",
                 platform_of=None, prio: int = abi.PRIO_UPWARD_RANK, want_attrs=True,
                 record=False, out_arrays=None, want_states=True) -> dict:
        """compute_attributes + default_regulator_config + simulate per graph.
        out_arrays: preallocated (pinned) host arrays worker/start_ms/end_ms/
        makespan_ms/completed/pop_mode_counts to receive the results."""
        G = db.n_graphs
        parr = platform_array(platforms, db.type_names)
        pof = None if platform_of is None else np.ascontiguousarray(platform_of, np.int32)
        aout, ao = outbuf.attr_out(db.n_tasks, G) if want_attrs else ({}, None)
        out, o = outbuf.sim_out(db.n_tasks, G, False, want_states=want_states, arrays=out_arrays)
        _check(load().tbsim_schedule(self.h, db.h, parr, len(platforms), _p(pof, C.c_int32),
                                     abi.POLICY_ID[policy], prio,
                                     None if ao is None else C.byref(ao), C.byref(o)))
        out.update({"attr_" + k: v for k, v in aout.items()})
        return out

    def schedule_device(self, db: DeviceBatch, platforms: Sequence[Platform], policy: str,
                        ptrs: dict, platform_of=None, prio: int = abi.PRIO_UPWARD_RANK):
        """tbsim_schedule writing straight into device buffers (e.g. torch
        tensors' data_ptr()): keys worker/start_ms/end_ms [T], makespan_ms [G]."""
        parr = platform_array(platforms, db.type_names)
        pof = None if platform_of is None else np.ascontiguousarray(platform_of, np.int32)
        o = abi.SimOut()
        o.on_device = 1
        for k, ct in (("worker", C.c_int32), ("start_ms", C.c_double), ("end_ms", C.c_double),
                      ("makespan_ms", C.c_double)):
            if ptrs.get(k):
                setattr(o, k, C.cast(C.c_void_p(ptrs[k]), C.POINTER(ct)))
        _check(load().tbsim_schedule(self.h, db.h, parr, len(platforms), _p(pof, C.c_int32),
                                     abi.POLICY_ID[policy], prio, None, C.byref(o)))

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def api_tiled_tasks(kind: str, nb: int) -> int:
    """Tasks of a tiled DAG: sum over steps of its roles (generators.cpp)."""
    total = 0
    for k in range(nb):
        m = nb - k - 1
        total += 1 + 2 * m + (m * (m - 1) // 2 if kind == "cholesky" else m * m)
    return total


def default_regulator_config(n_workers: int, median_gpu_ms: float) -> abi.RegulatorCfg:
    cfg = abi.RegulatorCfg()
    _check(load().tbsim_default_regulator_config(n_workers, median_gpu_ms, C.byref(cfg)))
    return cfg


def median_gpu_times(batch: GraphBatch, costs: CostTable) -> np.ndarray:
    """Lower-median GPU time per graph (platform.cpp:233-240), host helper for
    default regulator configs of tbsim_simulate calls."""
    _cpu, gpu = costs.arrays(batch.type_names)
    t = gpu[batch.type]
    out = np.zeros(batch.n_graphs)
    for g in range(batch.n_graphs):
        seg = np.sort(t[batch.task_base[g]:batch.task_base[g + 1]])
        out[g] = seg[(len(seg) - 1) // 2] if len(seg) else np.nan
    return out
