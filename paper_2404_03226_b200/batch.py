"""Host-side graph batches in the CSR layout of include/tbsim_b200.h.

A :class:`GraphBatch` is the Python twin of ``tbsim_batch_desc``: numpy
arrays for every CSR section plus the type-name table their ids index.  The
reference's ``TaskGraph`` (include/tbsim/taskgraph.hpp:36-42) converts into a
one-graph batch with :meth:`GraphBatch.from_taskgraphs`; id resolution raises
the reference's ``build_index`` errors (src/taskgraph.cpp:11-33).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from . import abi


@dataclass
class TaskNode:
    """TaskNode (taskgraph.hpp:25-33)."""
    id: int
    type: str
    deps: list = field(default_factory=list)
    inputs: list = field(default_factory=list)
    outputs: list = field(default_factory=list)


@dataclass
class TaskGraph:
    """TaskGraph (taskgraph.hpp:36-42): tasks in submission order."""
    name: str = ""
    tasks: list = field(default_factory=list)
    handles: list = field(default_factory=list)  # (id, bytes) pairs


def _ptr(a, ct):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ct))


class GraphBatch:
    """G graphs in batched CSR form (see tbsim_batch_desc)."""

    def __init__(self, task_base, edge_base, handle_base, in_base, out_base,
                 dep_off, dep, in_off, in_, out_off, out, type_, handle_bytes,
                 type_names: Sequence[str], task_id=None, names=None):
        i64 = lambda a: np.ascontiguousarray(a, dtype=np.int64)
        i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)
        self.task_base, self.edge_base = i64(task_base), i64(edge_base)
        self.handle_base, self.in_base, self.out_base = i64(handle_base), i64(in_base), i64(out_base)
        self.dep_off, self.dep = i32(dep_off), i32(dep)
        self.in_off, self.in_ = i32(in_off), i32(in_)
        self.out_off, self.out = i32(out_off), i32(out)
        self.type = i32(type_)
        self.handle_bytes = i64(handle_bytes)
        self.task_id = None if task_id is None else i64(task_id)
        self.type_names = list(type_names)
        self.names = names
        self._desc = None

    # ------------------------------------------------------------------ shape
    @property
    def n_graphs(self) -> int:
        return len(self.task_base) - 1

    @property
    def n_tasks(self) -> int:
        return int(self.task_base[-1])

    @property
    def n_edges(self) -> int:
        return int(self.edge_base[-1])

    def sizes(self, g: int) -> int:
        return int(self.task_base[g + 1] - self.task_base[g])

    def nbytes(self) -> int:
        arrs = [self.task_base, self.edge_base, self.handle_base, self.in_base, self.out_base,
                self.dep_off, self.dep, self.in_off, self.in_, self.out_off, self.out,
                self.type, self.handle_bytes]
        if self.task_id is not None:
            arrs.append(self.task_id)
        return int(sum(a.nbytes for a in arrs))

    # ------------------------------------------------------------- ctypes view
    def desc(self) -> abi.BatchDesc:
        if self._desc is None:
            d = abi.BatchDesc()
            d.n_graphs = self.n_graphs
            d.task_base = _ptr(self.task_base, C.c_int64)
            d.edge_base = _ptr(self.edge_base, C.c_int64)
            d.handle_base = _ptr(self.handle_base, C.c_int64)
            d.in_base = _ptr(self.in_base, C.c_int64)
            d.out_base = _ptr(self.out_base, C.c_int64)
            d.dep_off = _ptr(self.dep_off, C.c_int32)
            d.dep = _ptr(self.dep, C.c_int32)
            d.in_off = _ptr(self.in_off, C.c_int32)
            d.in_ = _ptr(self.in_, C.c_int32)
            d.out_off = _ptr(self.out_off, C.c_int32)
            d.out = _ptr(self.out, C.c_int32)
            d.type = _ptr(self.type, C.c_int32)
            d.handle_bytes = _ptr(self.handle_bytes, C.c_int64)
            d.task_id = _ptr(self.task_id, C.c_int64)
            self._names_c = (C.c_char_p * max(1, len(self.type_names)))(
                *[n.encode() for n in self.type_names])
            d.n_type_names = len(self.type_names)
            d.type_names = self._names_c
            self._desc = d
        return self._desc

    # ------------------------------------------------------------ per graph
    def graph_deps(self, g: int):
        """(dep_off, dep) of graph g as local arrays."""
        t0, t1 = self.task_base[g], self.task_base[g + 1]
        off = self.dep_off[t0 + g:t1 + g + 1]
        e0 = self.edge_base[g]
        return off, self.dep[e0:e0 + off[-1]]

    def slice(self, graphs: Iterable[int]) -> "GraphBatch":
        return GraphBatch.concat([self._one(g) for g in graphs])

    def _one(self, g: int) -> "GraphBatch":
        t0, t1 = int(self.task_base[g]), int(self.task_base[g + 1])
        n = t1 - t0
        sec = lambda base, off_arr, data: (
            off_arr[t0 + g:t1 + g + 1].copy(),
            data[int(base[g]):int(base[g]) + int(off_arr[t1 + g])].copy())
        doff, dep = sec(self.edge_base, self.dep_off, self.dep)
        ioff, inn = sec(self.in_base, self.in_off, self.in_)
        ooff, out = sec(self.out_base, self.out_off, self.out)
        h0, h1 = int(self.handle_base[g]), int(self.handle_base[g + 1])
        return GraphBatch([0, n], [0, len(dep)], [0, h1 - h0], [0, len(inn)], [0, len(out)],
                          doff, dep, ioff, inn, ooff, out, self.type[t0:t1].copy(),
                          self.handle_bytes[h0:h1].copy(), self.type_names,
                          None if self.task_id is None else self.task_id[t0:t1].copy())

    # ---------------------------------------------------------- constructors
    @staticmethod
    def concat(batches: Sequence["GraphBatch"]) -> "GraphBatch":
        if len(batches) == 1:
            return batches[0]
        names = list(batches[0].type_names)
        for b in batches[1:]:
            if list(b.type_names) != names:
                raise ValueError("concat needs a shared type-name table")

        def bases(attr):
            out = [0]
            for b in batches:
                arr = getattr(b, attr)
                out.extend((arr[1:] + out[-1]).tolist())
            return out

        cat = lambda attr: np.concatenate([getattr(b, attr) for b in batches])
        has_ids = all(b.task_id is not None for b in batches)
        return GraphBatch(bases("task_base"), bases("edge_base"), bases("handle_base"),
                          bases("in_base"), bases("out_base"), cat("dep_off"), cat("dep"),
                          cat("in_off"), cat("in_"), cat("out_off"), cat("out"), cat("type"),
                          cat("handle_bytes"), names, cat("task_id") if has_ids else None)

    @staticmethod
    def from_taskgraphs(graphs: Sequence[TaskGraph], type_names: Sequence[str] | None = None):
        """Resolve ids to positions (build_index, src/taskgraph.cpp:11-43)."""
        names = list(type_names) if type_names is not None else []
        name_id = {n: i for i, n in enumerate(names)}
        parts = []
        for tg in graphs:
            pos = {}
            for i, t in enumerate(tg.tasks):
                if t.id in pos:
                    raise ValueError(f"duplicate task id {t.id}")
                pos[t.id] = i
            hpos = {}
            for i, (hid, _b) in enumerate(tg.handles):
                if hid in hpos:
                    raise ValueError(f"duplicate handle id {hid}")
                hpos[hid] = i
            doff, dep, ioff, inn, ooff, out, ty = [0], [], [0], [], [0], [], []
            for t in tg.tasks:
                for d in t.deps:
                    if d not in pos:
                        raise ValueError(f"task {t.id} depends on unknown task {d}")
                    dep.append(pos[d])
                for h in t.inputs:
                    if h not in hpos:
                        raise KeyError(f"unknown handle {h}")
                    inn.append(hpos[h])
                for h in t.outputs:
                    if h not in hpos:
                        raise KeyError(f"unknown handle {h}")
                    out.append(hpos[h])
                doff.append(len(dep)); ioff.append(len(inn)); ooff.append(len(out))
                if t.type not in name_id:
                    name_id[t.type] = len(names)
                    names.append(t.type)
                ty.append(name_id[t.type])
            n = len(tg.tasks)
            parts.append((n, doff, dep, ioff, inn, ooff, out, ty,
                          [b for _h, b in tg.handles], [t.id for t in tg.tasks]))
        batches = [GraphBatch([0, p[0]], [0, len(p[2])], [0, len(p[8])], [0, len(p[4])],
                              [0, len(p[6])], p[1], p[2], p[3], p[4], p[5], p[6], p[7], p[8],
                              names, p[9]) for p in parts]
        for b in batches:
            b.type_names = names
        return GraphBatch.concat(batches)
