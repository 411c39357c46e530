"""Machine model: cost table, workers, memory nodes, bandwidth.

Python twin of include/tbsim/platform.hpp for building the
``tbsim_platform_desc`` the device simulator consumes.  Values restate the
reference's synthetic model (src/platform.cpp:80-129).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import abi

CPU, GPU = 0, 1

# Canonical type-name table of the generators (ids index it).  Must equal the
# C++ host library's table (csrc/host_graph.cpp, tbsim_type_name()).
TYPE_NAMES = ["GEMM", "SYRK", "TRSM", "POTRF", "GETRF", "STENCIL",
              "LAYERK0", "LAYERK1", "LAYERK2", "LAYERK3", "UNIT",
              "GEQRT", "UNMQR", "TSQRT", "TSMQR"]
TYPE_ID = {n: i for i, n in enumerate(TYPE_NAMES)}

# (GPU ms, CPU/GPU ratio) -- default_cost_table, src/platform.cpp:93-98.
_DEFAULT_ROWS = {
    "GEMM": (0.4, 10.0), "SYRK": (1.0, 10.0), "TRSM": (1.2, 10.0),
    "POTRF": (2.0, 3.0), "GETRF": (2.0, 3.0), "STENCIL": (0.8, 5.0),
    "LAYERK0": (0.5, 5.0), "LAYERK1": (1.0, 8.0), "LAYERK2": (2.0, 3.0),
    "LAYERK3": (4.0, 6.0), "UNIT": (1.0, 1.0),
}
# Tiled-QR kernels have no reference cost rows; these are
# builder-chosen, GEQRT/TSQRT panel-like (latency bound, 3x), UNMQR/TSMQR
# update-like (BLAS-3, 10x), scaled like the LU rows.
_QR_ROWS = {"GEQRT": (2.0, 3.0), "TSQRT": (2.4, 3.0), "UNMQR": (0.8, 10.0),
            "TSMQR": (0.8, 10.0)}

HOST_GPU_BW = 12e6   # bytes/ms, src/platform.cpp:108
GPU_GPU_BW = 24e6    # src/platform.cpp:109
LATENCY_MS = 0.01    # src/platform.cpp:110


class CostTable:
    """CostTable (platform.hpp:23-47)."""

    def __init__(self):
        self.entries: dict[tuple[str, int], float] = {}

    def set(self, type_: str, kind: int, ms: float):
        if not (ms > 0.0):
            raise ValueError(f"cost for {type_} must be positive")
        self.entries[(type_, kind)] = float(ms)

    def find(self, type_: str, kind: int):
        return self.entries.get((type_, kind))

    def gpu_ms(self, type_: str) -> float:
        v = self.find(type_, GPU)
        if v is None:
            raise RuntimeError(f"no gpu cost entry for task type {type_}")
        return v

    def arrays(self, type_names):
        cpu = np.zeros(len(type_names), np.float64)
        gpu = np.zeros(len(type_names), np.float64)
        for i, n in enumerate(type_names):
            cpu[i] = self.entries.get((n, CPU), 0.0)
            gpu[i] = self.entries.get((n, GPU), 0.0)
        return cpu, gpu


def default_cost_table(with_qr: bool = False) -> CostTable:
    t = CostTable()
    rows = dict(_DEFAULT_ROWS)
    if with_qr:
        rows.update(_QR_ROWS)
    for name, (gpu, ratio) in rows.items():
        t.set(name, GPU, gpu)
        t.set(name, CPU, gpu * ratio)  # FP64 product, exact for these rows
    return t


@dataclass
class Platform:
    """Platform (platform.hpp:51-63).  workers: list of (kind, memory_node);
    worker ids are the list positions."""
    name: str = ""
    workers: list = field(default_factory=list)
    costs: CostTable = field(default_factory=CostTable)
    num_nodes: int = 1
    latency_ms: float = 0.0
    bandwidth: list = field(default_factory=list)

    @property
    def n_workers(self) -> int:
        return len(self.workers)

    def desc(self, type_names) -> abi.PlatformDesc:
        """ctypes view; the numpy buffers are kept alive on the returned object."""
        d = abi.PlatformDesc()
        kind = np.array([k for k, _ in self.workers], np.int32)
        node = np.array([m for _, m in self.workers], np.int32)
        bw = np.zeros((self.num_nodes, self.num_nodes), np.float64)
        for a in range(self.num_nodes):
            for b in range(self.num_nodes):
                bw[a, b] = self.bandwidth[a][b]
        cpu, gpu = self.costs.arrays(type_names)
        d.n_workers = len(self.workers)
        d.kind = kind.ctypes.data_as(C.POINTER(C.c_int32))
        d.memory_node = node.ctypes.data_as(C.POINTER(C.c_int32))
        d.n_nodes = self.num_nodes
        d.latency_ms = self.latency_ms
        d.bandwidth = bw.ctypes.data_as(C.POINTER(C.c_double))
        d.costs.n_types = len(type_names)
        d.costs.cpu_ms = cpu.ctypes.data_as(C.POINTER(C.c_double))
        d.costs.gpu_ms = gpu.ctypes.data_as(C.POINTER(C.c_double))
        d._keep = (kind, node, bw, cpu, gpu)
        return d


def assemble(name: str, n_cpus: int, n_gpus: int, with_qr: bool = False) -> Platform:
    """CPUs on node 0, GPU i on node 1+i (src/platform.cpp:112-129)."""
    p = Platform(name=name, costs=default_cost_table(with_qr))
    p.workers = [(CPU, 0)] * n_cpus + [(GPU, 1 + i) for i in range(n_gpus)]
    p.num_nodes = 1 + n_gpus
    p.latency_ms = LATENCY_MS
    p.bandwidth = [[0.0 if a == b else (GPU_GPU_BW if a > 0 and b > 0 else HOST_GPU_BW)
                    for b in range(p.num_nodes)] for a in range(p.num_nodes)]
    return p


_PRESETS = {"2gpu": (0, 2), "26cpu_2gpu": (26, 2), "26cpu_1gpu": (26, 1), "homog2": (2, 0)}


def make_preset(name: str) -> Platform:
    """make_preset (src/platform.cpp:169-183)."""
    if name not in _PRESETS:
        raise RuntimeError(f'unknown platform preset "{name}"')
    return assemble(name, *_PRESETS[name])


def preset_names():
    return list(_PRESETS)


def platform_array(platforms, type_names):
    """Contiguous tbsim_platform_desc[] for a list of Platforms."""
    arr = (abi.PlatformDesc * len(platforms))()
    keep = []
    for i, p in enumerate(platforms):
        d = p.desc(type_names)
        keep.append(d._keep)
        arr[i] = d
    arr._keep = keep
    return arr
