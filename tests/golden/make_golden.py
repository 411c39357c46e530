"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Run in the build container (needs /root/reference and oracle/_ref built):

    make -C oracle ref && python tests/golden/make_golden.py

Every fixture is one .npz holding a batch in the C-ABI CSR layout, its cost
table, and the reference's outputs: compute_attributes (UpwardRank), the
calibration record, depth, layers, and for each platform x policy the full
SimTrace (per-task worker/start/end, makespan, push/pop/nready ledger,
pop-mode counts, final regulator state).  Graph sources: the reference's own
generators, its tests' oracle::random_dag (non-contiguous ids, handles), its
hand graphs (tests/test_attributes.cpp chain3/diamond) and its committed
fixture tests/data/chain_wave.dag.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import pyref  # noqa: E402
from paper_2404_03226_b200 import abi  # noqa: E402
from paper_2404_03226_b200 import platform as P  # noqa: E402
from paper_2404_03226_b200.batch import GraphBatch, TaskGraph, TaskNode  # noqa: E402

MIXED = ["LAYERK0", "LAYERK1", "LAYERK2", "LAYERK3", "UNIT"]
PLATFORMS = {
    "homog2": P.make_preset("homog2"),
    "26cpu_2gpu": P.make_preset("26cpu_2gpu"),
    "2gpu": P.make_preset("2gpu"),
    "4c1g": P.assemble("4c1g", 4, 1),
    "8c2g": P.assemble("8c2g", 8, 2),
    "32c4g": P.assemble("32c4g", 32, 4),
}


def save(name, batch: GraphBatch, costs: P.CostTable, platforms, policies=abi.POLICIES, prio=abi.PRIO_UPWARD_RANK,
         sim=True):
    cpu, gpu = costs.arrays(batch.type_names)
    rec = {"task_base": batch.task_base, "edge_base": batch.edge_base, "handle_base": batch.handle_base,
           "in_base": batch.in_base, "out_base": batch.out_base, "dep_off": batch.dep_off, "dep": batch.dep,
           "in_off": batch.in_off, "in_": batch.in_, "out_off": batch.out_off, "out": batch.out,
           "type": batch.type, "handle_bytes": batch.handle_bytes,
           "task_id": batch.task_id if batch.task_id is not None else np.arange(batch.n_tasks),
           "type_names": np.array(batch.type_names), "cost_cpu": cpu, "cost_gpu": gpu,
           "prio_kind": np.array(prio)}
    a = pyref.attributes(batch, costs, abi.ATTR_ALL, prio)
    for k in ("ability", "efficiency", "static_priority", "unit_time_ms"):
        rec["attr_" + k] = a[k]
    c = pyref.attributes(batch, costs, abi.ATTR_CALIBRATE)
    for k in ("w0_ms", "best_score", "w0_score", "evaluations"):
        rec["calib_" + k] = c[k]
    rec["depth"] = pyref.attributes(batch, costs, abi.ATTR_DEPTH)["depth"]
    rec["layer"] = pyref.attributes(batch, costs, abi.ATTR_LAYERS)["layer"]
    rec["rank"] = pyref.attributes(batch, costs, abi.ATTR_RANK)["static_priority"]
    for w in (0.5, 1.0, 4.0, 16.0):
        rec[f"eff_w{w}"] = pyref.attributes(batch, costs, abi.ATTR_EFFICIENCY,
                                            unit_time=np.full(batch.n_graphs, w))["efficiency"]
    if sim:
        rec["platforms"] = np.array(list(platforms))
        for pname in platforms:
            pl = PLATFORMS[pname]
            if costs is not None:
                pl = P.Platform(pl.name, pl.workers, costs, pl.num_nodes, pl.latency_ms, pl.bandwidth)
            for pol in policies:
                r = pyref.simulate(batch, [pl], pol, attrs=a, record=True)
                key = f"sim_{pname}_{pol}_"
                for k in ("worker", "start_ms", "end_ms", "makespan_ms", "pop_mode_counts", "push_time",
                          "push_task", "pop_time", "pop_task", "pop_worker", "sample_time", "sample_nready"):
                    rec[key + k] = r[k]
                st = r["reg_state"]
                rec[key + "reg"] = np.array([[s.mode, s.phase, s.peak, s.prev_nready, s.last_trigger_nready,
                                              s.s_dec_count] for s in st[:batch.n_graphs]], np.int64)
                rec[key + "reg_cur_k"] = np.array([s.cur_k for s in st[:batch.n_graphs]])
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **rec)
    print("wrote", name, batch.n_graphs, "graphs", batch.n_tasks, "tasks")


def hand_graphs():
    chain = TaskGraph("chain3", [TaskNode(0, "UNIT"), TaskNode(1, "UNIT", [0]), TaskNode(2, "UNIT", [1])])
    diamond = TaskGraph("diamond", [TaskNode(0, "A"), TaskNode(1, "B", [0]), TaskNode(2, "C", [0]),
                                    TaskNode(3, "D", [1, 2])])
    return chain, diamond


def _fmt_ms(v):
    s = "%.6f" % v
    if "." in s:
        s = s.rstrip("0")
        if s.endswith("."):
            s = s[:-1]
    return "0" if s == "-0" else s


def grid_csv():
    """The acceptance gate's INSPIRIT-vs-DMDA grid (tests/acceptance.cpp:430-480)
    as the reference's bench CSV (src/bench.cpp:149-159), cells computed by
    the reference itself."""
    pl = P.make_preset("26cpu_2gpu")
    costs = pl.costs
    rows = []
    cells = [("autogen", n, lambda n: pyref.gen_layered(n, 10, 0.05, 7)) for n in (1000, 5000)]
    cells += [("cholesky", n, lambda n: pyref.gen_cholesky(n, 960 * 960 * 4)) for n in (8, 12, 16, 20, 24)]
    cells += [("lu", n, lambda n: pyref.gen_lu(n, 160 * 160 * 4)) for n in (8, 12, 16)]
    for app, n, gen in cells:
        b = gen(n)
        a = pyref.attributes(b, costs, abi.ATTR_ALL)
        ms = {pol: pyref.simulate(b, [pl], pol, attrs=a, record=False)["makespan_ms"][0] for pol in ("dmda", "inspirit")}
        for pol in ("dmda", "inspirit"):
            sp = 1.0 if pol == "dmda" else ms["dmda"] / ms[pol]
            rows.append((app, n, pol, f"{app},{n},26cpu_2gpu,{pol},{_fmt_ms(ms[pol])},{sp:.3f},ok"))
    rows.sort(key=lambda r: (r[0], r[1], r[2]))
    with open(os.path.join(HERE, "grid_bench.csv"), "w") as f:
        f.write("app,size,platform,policy,makespan_ms,speedup_vs_baseline,status\n")
        for r in rows:
            f.write(r[3] + "\n")
    print("wrote grid_bench.csv", len(rows), "rows")


def main():
    default = P.default_cost_table()
    # hand graphs of tests/test_attributes.cpp
    chain, diamond = hand_graphs()
    save("hand_chain3", GraphBatch.from_taskgraphs([chain]), default, ["homog2", "26cpu_2gpu"])
    dcost = P.CostTable()
    for t, ms in (("A", 1.0), ("B", 2.0), ("C", 3.0), ("D", 1.0)):
        dcost.set(t, P.GPU, ms)
        dcost.set(t, P.CPU, 2 * ms)
    save("hand_diamond", GraphBatch.from_taskgraphs([diamond]), dcost, ["homog2", "2gpu"])
    # committed fixture of the reference tests
    save("chain_wave", pyref.gen_file("/root/reference/proj/tests/data/chain_wave.dag"), default,
         ["homog2", "26cpu_2gpu"], prio=abi.PRIO_UPWARD_RANK)
    save("chain_wave_depth", pyref.gen_file("/root/reference/proj/tests/data/chain_wave.dag"), default,
         ["homog2"], prio=abi.PRIO_DEPTH)
    # tiled factorizations (C1 = cholesky 10 on 4c1g; README goldens: cholesky 8/12 on 26cpu_2gpu)
    save("cholesky", GraphBatch.concat([pyref.gen_cholesky(n, 960 * 960 * 4) for n in (4, 6, 8, 10, 12)]),
         default, ["4c1g", "26cpu_2gpu", "2gpu"])
    save("lu", GraphBatch.concat([pyref.gen_lu(n, 160 * 160 * 4) for n in (3, 6, 10)]), default,
         ["26cpu_2gpu", "32c4g"])
    # layered synthesized DAGs (C2 shape and small ones)
    save("layered_1k", GraphBatch.concat([pyref.gen_layered(1000, 10, 0.05, s) for s in (0, 1)]), default,
         ["8c2g"])
    save("layered_small", GraphBatch.concat([pyref.gen_layered(30 + 17 * s, 3 + s % 7, 0.03 + 0.01 * (s % 5), s)
                                             for s in range(12)]), default, ["26cpu_2gpu", "2gpu", "homog2"])
    # oracle::random_dag of the reference tests (non-contiguous ids, handles)
    rnd = [pyref.gen_random(seed * 101, 60, 0.08, MIXED, True) for seed in range(1, 5)]
    rnd += [pyref.gen_random(100 + i, 20 + (i * 13) % 181, 0.04 + 0.02 * (i % 4), MIXED, False) for i in range(6)]
    # type tables must agree to concatenate: remap onto one name list
    names = list(P.TYPE_NAMES)
    for b in rnd:
        assert b.type_names[:len(P.TYPE_NAMES)] == P.TYPE_NAMES
    save("random_dag", GraphBatch.concat(rnd), default, ["homog2", "26cpu_2gpu", "2gpu"])
    grid_csv()
    # README goldens (proj/README.md:81-88,117-125): cholesky 8/12 dmda/inspirit
    # are inside "cholesky" on 26cpu_2gpu; a quick self-check:
    z = np.load(os.path.join(HERE, "cholesky.npz"))
    ms = z["sim_26cpu_2gpu_inspirit_makespan_ms"]
    print("README check: cholesky8 inspirit", ms[2], "dmda", z["sim_26cpu_2gpu_dmda_makespan_ms"][2],
          "cholesky12 inspirit", ms[4])


if __name__ == "__main__":
    main()
