"""GPU: the CUDA path (through the C-ABI) against the reference's golden
fixtures and the oracle -- bit-exact for every integer attribute, every
assignment/start/end double, the push/pop/nready ledger and the regulator
state.  Run with `pytest -m gpu` on a B200."""
import numpy as np
import pytest

from golden_util import SIM_KEYS, Fixture, names, reg_rows
from oracle import pyoracle as po
from paper_2404_03226_b200 import abi, api
from paper_2404_03226_b200 import platform as P
from paper_2404_03226_b200.batch import GraphBatch, TaskGraph, TaskNode

pytestmark = pytest.mark.gpu
FIXTURES = names()
MIXED = ["LAYERK0", "LAYERK1", "LAYERK2", "LAYERK3", "UNIT"]


def eq(a, b, msg):
    np.testing.assert_array_equal(np.asarray(a), np.asarray(b), err_msg=msg)


@pytest.mark.parametrize("name", FIXTURES)
def test_attributes_match_reference_fixture(ctx, name):
    f = Fixture(name)
    db = ctx.upload(f.batch)
    a = ctx.attributes(db, f.costs, abi.ATTR_ALL, f.prio)
    for k in ("ability", "efficiency", "static_priority", "unit_time_ms"):
        eq(a[k], f.z["attr_" + k], k)
    c = ctx.attributes(db, f.costs, abi.ATTR_CALIBRATE)
    for k in ("w0_ms", "best_score", "w0_score", "evaluations"):
        eq(c[k], f.z["calib_" + k], k)
    eq(ctx.attributes(db, f.costs, abi.ATTR_DEPTH)["depth"], f.z["depth"], "depth")
    eq(ctx.attributes(db, f.costs, abi.ATTR_LAYERS)["layer"], f.z["layer"], "layer")
    eq(ctx.attributes(db, f.costs, abi.ATTR_RANK)["static_priority"], f.z["rank"], "rank")
    eq(ctx.attributes(db, f.costs, abi.ATTR_ABILITY)["ability"], f.z["attr_ability"], "ability only")
    for w in (0.5, 1.0, 4.0, 16.0):
        e = ctx.attributes(db, f.costs, abi.ATTR_EFFICIENCY, unit_time=np.full(f.batch.n_graphs, w))
        eq(e["efficiency"], f.z[f"eff_w{w}"], f"eff@{w}")


@pytest.mark.parametrize("name", FIXTURES)
def test_simulation_matches_reference_fixture(ctx, name):
    f = Fixture(name)
    db = ctx.upload(f.batch)
    for pname in f.platform_names:
        pl = f.platform(pname)
        reg = f.reg_cfgs(pname, po)
        for pol in abi.POLICIES:
            r = ctx.simulate(db, [pl], pol, reg, attrs=f.attrs(), record=True)
            want = f.sim(pname, pol)
            for k in SIM_KEYS:
                eq(r[k], want[k], f"{pname}/{pol}/{k}")
            if pol == "inspirit":
                eq(reg_rows(r["reg_state"], f.batch.n_graphs), want["reg"], "regulator state")
                eq([s.cur_k for s in r["reg_state"][:f.batch.n_graphs]], want["reg_cur_k"], "cur_k")


def random_graphs(seed, count, with_handles=True, max_n=120):
    """Random DAGs with non-contiguous ids, multi-edges, ids out of order and
    inputs that are not dependencies (a construction unlike both generators)."""
    rng = np.random.default_rng(seed)
    out = []
    for gi in range(count):
        n = int(rng.integers(1, max_n))
        ids = rng.permutation(np.arange(n) * 7 + 1000)
        tasks = []
        handles = [(5000 + 3 * h, int(rng.integers(1, 5)) * 100_000) for h in range(n)]
        for i in range(n):
            deps = [int(ids[j]) for j in range(i) if rng.random() < 0.08]
            if deps and rng.random() < 0.2:
                deps.append(deps[0])  # multi-edge
            inputs = [5000 + 3 * int(rng.integers(0, n)) for _ in range(int(rng.integers(0, 4)))] if with_handles else []
            outputs = [5000 + 3 * i] if with_handles else []
            tasks.append(TaskNode(int(ids[i]), MIXED[int(rng.integers(0, 5))], deps, inputs, outputs))
        out.append(TaskGraph(f"r{gi}", tasks, handles if with_handles else []))
    return GraphBatch.from_taskgraphs(out, P.TYPE_NAMES)


def test_random_graphs_all_policies_platform_mix(ctx):
    b = random_graphs(7, 40)
    costs = P.default_cost_table()
    pls = [P.make_preset("26cpu_2gpu"), P.make_preset("2gpu"), P.make_preset("homog2"),
           P.assemble("32c4g", 32, 4), P.assemble("4c1g", 4, 1)]
    pof = np.arange(b.n_graphs) % len(pls)
    db = ctx.upload(b)
    ga = ctx.attributes(db, costs, abi.ATTR_ALL)
    oa = po.attributes(b, costs, abi.ATTR_ALL)
    for k in ("ability", "efficiency", "static_priority", "unit_time_ms"):
        eq(ga[k], oa[k], k)
    reg = [po.default_regulator_config(b, g, pls[pof[g]]) for g in range(b.n_graphs)]
    for pol in abi.POLICIES:
        g = ctx.simulate(db, pls, pol, reg, platform_of=pof, attrs=oa, record=True)
        o = po.simulate(b, pls, pol, platform_of=pof, reg=reg, attrs=oa, record=True)
        for k in SIM_KEYS:
            eq(g[k], o[k], f"{pol}/{k}")


def test_fused_upload_kernel_on_many_random_graphs(ctx):
    """Batches of >= 4 graphs per SM build their successor CSR and packed
    simulation view in one pass (k_ingest_pack): multi-edges, shuffled ids,
    inputs that are not dependencies, tasks without inputs, every policy and
    the full push/pop/nready ledger against the oracle."""
    b = random_graphs(11, 640, max_n=40)
    costs = P.default_cost_table()
    pls = [P.assemble("8c2g", 8, 2), P.make_preset("2gpu"), P.assemble("4c1g", 4, 1)]
    pof = np.arange(b.n_graphs) % len(pls)
    ctx.set_timing(True)
    try:
        db = ctx.upload(b)
        ga = ctx.attributes(db, costs, abi.ATTR_ALL)
        assert ctx.last_kernel_ms("k_ingest_pack") > 0.0, "the fused upload kernel did not run"
    finally:
        ctx.set_timing(False)
    oa = po.attributes(b, costs, abi.ATTR_ALL)
    for k in ("ability", "efficiency", "static_priority", "unit_time_ms"):
        eq(ga[k], oa[k], k)
    reg = [po.default_regulator_config(b, g, pls[pof[g]]) for g in range(b.n_graphs)]
    for pol in abi.POLICIES:
        g = ctx.simulate(db, pls, pol, reg, platform_of=pof, attrs=oa, record=True)
        o = po.simulate(b, pls, pol, platform_of=pof, reg=reg, attrs=oa, record=True)
        for k in SIM_KEYS:
            eq(g[k], o[k], f"{pol}/{k}")


@pytest.mark.parametrize("tile", [8, 16, 32, 64, 128, 256])
def test_every_sweep_tile_width_matches_oracle(ctx, tile):
    """Each tile width runs its own kernel shape (one node per warp at 128
    sources, rows of 8 / 4 lanes at 64 / 32, a lane per node at 16 / 8):
    attributes equal the oracle's for all of them, on random graphs and on
    layered ones wide enough to need several tiles per level."""
    b = random_graphs(23, 30)
    lay = api.HostBatch().add_layered(700, 7, 0.08, [3, 4]).view()
    costs = P.default_cost_table()
    for batch in (b, lay):
        db = ctx.upload(batch)
        oa = po.attributes(batch, costs, abi.ATTR_ALL)
        o3 = po.attributes(batch, costs, abi.ATTR_EFFICIENCY, unit_time=np.full(batch.n_graphs, 3.0))
        ctx.set_sweep_tile(tile)
        try:
            ga = ctx.attributes(db, costs, abi.ATTR_ALL)
            g3 = ctx.attributes(db, costs, abi.ATTR_EFFICIENCY, unit_time=np.full(batch.n_graphs, 3.0))
            gb = ctx.attributes(db, costs, abi.ATTR_ABILITY)
        finally:
            ctx.set_sweep_tile(0)
        for k in ("ability", "efficiency", "static_priority", "unit_time_ms"):
            eq(ga[k], oa[k], f"S={tile} {k}")
        eq(g3["efficiency"], o3["efficiency"], f"S={tile} efficiency@3")
        eq(gb["ability"], oa["ability"], f"S={tile} ability only")


@pytest.mark.parametrize("gpu_ms", [(0.5, 1.0, 2.0, 4.0), (1.0 + 2.0 ** -23, 0.5, 2.0, 3.0),
                                    (0.1, 0.5, 2.0, 4.0), (3.0 * 2.0 ** -40, 2.0 ** -41, 2.0 ** -38, 1.0)])
def test_fp32_windows_only_when_exact(ctx, gpu_ms):
    """The sweep keeps distances in FP32 only when every path sum is exact
    there (dyadic GPU times, levels x largest mantissa < 2^24); otherwise FP64.
    Either way the attributes equal the oracle's: (1) exact -> FP32; (2)
    dyadic but 2^23+1 mantissa over 12 levels -> FP64; (3) 0.1 is not dyadic
    -> FP64; (4) tiny dyadic times with a 2^41 spread -> FP64."""
    costs = P.CostTable()
    for name, g in zip(("LAYERK0", "LAYERK1", "LAYERK2", "LAYERK3"), gpu_ms):
        costs.set(name, P.GPU, g)
        costs.set(name, P.CPU, 3.0 * g)
    b = api.HostBatch().add_layered(400, 12, 0.06, [7, 8, 9]).view()
    db = ctx.upload(b)
    for tile in (0, 256, 64):
        ctx.set_sweep_tile(tile)
        try:
            ga = ctx.attributes(db, costs, abi.ATTR_ALL)
        finally:
            ctx.set_sweep_tile(0)
        oa = po.attributes(b, costs, abi.ATTR_ALL)
        for k in ("ability", "efficiency", "unit_time_ms"):
            eq(ga[k], oa[k], f"tile {tile} {k}")


def test_sweep_tile_rejects_other_widths(ctx):
    with pytest.raises(ValueError):
        ctx.set_sweep_tile(24)


def odd_platform(name, bw_rows, latency=0.02):
    """4 CPUs on node 0, one GPU per further node, custom bandwidths."""
    nn = len(bw_rows)
    workers = [(0, 0)] * 4 + [(1, k) for k in range(1, nn)]
    return P.Platform(name, workers, P.default_cost_table(), nn, latency, bw_rows)


def test_transfers_on_custom_bandwidth_matrices(ctx):
    """Fastest-copy transfers (engine.cpp:86-110) on asymmetric bandwidth
    matrices with 1..5 distinct values and a zero bandwidth, alone and mixed
    in one batch, give the reference's schedules."""
    b = random_graphs(11, 30)
    two = [[0, 7e6, 9e6], [7e6, 0, 9e6], [9e6, 9e6, 0]]
    one = [[0, 5e6], [5e6, 0]]
    three = [[0, 3e6, 5e6, 7e6], [3e6, 0, 7e6, 5e6], [5e6, 7e6, 0, 3e6], [7e6, 5e6, 3e6, 0]]
    five = [[0, 1e6, 2e6, 3e6], [1e6, 0, 4e6, 5e6], [2e6, 4e6, 0, 5e6], [3e6, 5e6, 4e6, 0]]
    zero = [[0, 0.0, 9e6], [6e6, 0, 9e6], [9e6, 9e6, 0]]
    costs = P.default_cost_table()
    oa = po.attributes(b, costs, abi.ATTR_ALL)
    db = ctx.upload(b)
    for pls in ([odd_platform("one", one)], [odd_platform("two", two)], [odd_platform("three", three)],
                [odd_platform("five", five)], [odd_platform("zero", zero)],
                [odd_platform("two", two), odd_platform("five", five), odd_platform("three", three)]):
        pof = np.arange(b.n_graphs) % len(pls)
        reg = [po.default_regulator_config(b, g, pls[pof[g]]) for g in range(b.n_graphs)]
        for pol in ("dmda", "inspirit"):
            g = ctx.simulate(db, pls, pol, reg, platform_of=pof, attrs=oa, record=True)
            o = po.simulate(b, pls, pol, platform_of=pof, reg=reg, attrs=oa, record=True)
            for k in SIM_KEYS:
                eq(g[k], o[k], f"{[p.name for p in pls]}/{pol}/{k}")


def test_schedule_pipeline_matches_oracle(ctx):
    hb = api.HostBatch().add_cholesky(10, 960 * 960 * 4).add_layered(1000, 10, 0.05, [3, 4, 5])
    hb.add_lu(12, 160 * 160 * 4).add_qr(10, 160 * 160 * 4)
    b = hb.view()
    pls = [P.assemble("4c1g", 4, 1, True), P.assemble("8c2g", 8, 2, True), P.assemble("32c4g", 32, 4, True)]
    pof = np.array([0, 1, 1, 1, 2, 2], np.int32)
    db = ctx.upload(hb)
    for prio in (abi.PRIO_UPWARD_RANK, abi.PRIO_DEPTH, abi.PRIO_ZERO):
        r = ctx.schedule(db, pls, "inspirit", platform_of=pof, prio=prio)
        oa = po.attributes(b, pls[0].costs, abi.ATTR_ALL, prio)
        for k in ("ability", "efficiency", "static_priority", "unit_time_ms"):
            eq(r["attr_" + k], oa[k], f"prio{prio}/{k}")
        reg = [po.default_regulator_config(b, g, pls[pof[g]]) for g in range(b.n_graphs)]
        o = po.simulate(b, pls, "inspirit", platform_of=pof, reg=reg, attrs=oa, record=False)
        for k in ("worker", "start_ms", "end_ms", "makespan_ms", "pop_mode_counts"):
            eq(r[k], o[k], f"prio{prio}/{k}")


def test_c2_batch_sample_and_properties(ctx):
    seeds = np.arange(4096)
    hb = api.HostBatch().add_layered(1000, 10, 0.05, seeds)
    b = hb.view()
    pl = [P.assemble("8c2g", 8, 2)]
    db = ctx.upload(hb)
    r = ctx.schedule(db, pl, "inspirit")
    # size-independent properties over the whole batch
    assert np.all(r["attr_efficiency"] <= r["attr_ability"])
    assert np.all(r["worker"] >= 0) and np.all(r["worker"] < 10)
    assert np.all(r["end_ms"] > r["start_ms"])
    for g in range(0, 4096, 97):
        t0, t1 = b.task_base[g], b.task_base[g + 1]
        assert r["makespan_ms"][g] == r["end_ms"][t0:t1].max()
        off, dep = b.graph_deps(g)
        st, en = r["start_ms"][t0:t1], r["end_ms"][t0:t1]
        for v in range(t1 - t0):  # precedence (trace_checks.hpp:64-73)
            preds = dep[off[v]:off[v + 1]]
            if len(preds):
                assert st[v] >= en[preds].max()
    # exact parity on a sample
    idx = list(range(0, 4096, 256))
    sub = b.slice(idx)
    costs = P.default_cost_table()
    oa = po.attributes(sub, costs, abi.ATTR_ALL)
    reg = [po.default_regulator_config(sub, i, pl[0]) for i in range(sub.n_graphs)]
    o = po.simulate(sub, pl, "inspirit", reg=reg, attrs=oa, record=False)
    eq(r["makespan_ms"][idx], o["makespan_ms"], "makespan sample")
    rows = np.concatenate([np.arange(b.task_base[g], b.task_base[g + 1]) for g in idx])
    eq(r["worker"][rows], o["worker"], "assignment sample")
    eq(r["attr_efficiency"][rows], oa["efficiency"], "efficiency sample")


def test_regulator_state_carries_across_runs(ctx):
    # a policy object reused for a second simulate() continues from its state
    f = Fixture("cholesky")
    pl = f.platform("26cpu_2gpu")
    reg = f.reg_cfgs("26cpu_2gpu", po)
    db = ctx.upload(f.batch)
    g1 = ctx.simulate(db, [pl], "inspirit", reg, attrs=f.attrs())
    g2 = ctx.simulate(db, [pl], "inspirit", reg, attrs=f.attrs(), states=g1["reg_state"])
    o1 = po.simulate(f.batch, [pl], "inspirit", reg=reg, attrs=f.attrs())
    o2 = po.simulate(f.batch, [pl], "inspirit", reg=reg, attrs=f.attrs(), states=o1["reg_state"])
    for k in SIM_KEYS:
        eq(g2[k], o2[k], k)
    eq(reg_rows(g2["reg_state"], f.batch.n_graphs), reg_rows(o2["reg_state"], f.batch.n_graphs), "state")


def _tg(tasks):
    return GraphBatch.from_taskgraphs([TaskGraph("t", tasks)], P.TYPE_NAMES)


def test_errors_carry_reference_type_and_text(ctx):
    costs = P.default_cost_table()
    cyc = _tg([TaskNode(0, "UNIT", [1]), TaskNode(1, "UNIT", [0])])
    db = ctx.upload(cyc)
    with pytest.raises(api.TbsimRuntimeError, match="graph has a dependency cycle"):
        ctx.attributes(db, costs, abi.ATTR_ALL)
    with pytest.raises(api.TbsimRuntimeError, match="graph has a dependency cycle"):
        ctx.attributes(db, costs, abi.ATTR_LAYERS)
    reg = [api.default_regulator_config(2, 1.0)]
    with pytest.raises(api.TbsimRuntimeError, match=r"simulation stuck with 2 tasks unfinished: 0 1$"):
        ctx.simulate(db, [P.make_preset("homog2")], "fifo", reg)
    gonly = GraphBatch.from_taskgraphs([TaskGraph("g", [TaskNode(0, "GONLY_TYPE")])])
    pl = P.make_preset("homog2")
    pl.costs = P.CostTable()
    pl.costs.set("GONLY_TYPE", P.GPU, 1.0)
    with pytest.raises(api.TbsimRuntimeError, match="no worker can run task type GONLY_TYPE"):
        ctx.simulate(ctx.upload(gonly), [pl], "dmda", reg)
    unit = P.CostTable()
    unit.set("UNIT", P.GPU, 1.0)
    chain = ctx.upload(_tg([TaskNode(0, "UNIT"), TaskNode(1, "UNIT", [0])]))
    with pytest.raises(api.TbsimInvalidArgument, match="unit time must be non-negative"):
        ctx.attributes(chain, unit, abi.ATTR_EFFICIENCY, unit_time=[-1.0])
    nogpu = P.CostTable()
    nogpu.set("UNIT", P.CPU, 1.0)
    with pytest.raises(api.TbsimRuntimeError, match="no gpu cost entry for task type UNIT"):
        ctx.attributes(chain, nogpu, abi.ATTR_ALL)
    empty = ctx.upload(GraphBatch.from_taskgraphs([TaskGraph("e", [])], P.TYPE_NAMES))
    with pytest.raises(api.TbsimRuntimeError, match="empty graph has no median time"):
        ctx.attributes(empty, costs, abi.ATTR_ALL)
    assert ctx.attributes(empty, costs, abi.ATTR_ABILITY)["ability"].size == 0


def test_c3_lu_and_qr_on_32c4g(ctx):
    # BASELINE configs[2]: 40x40 tiles, 36 workers (two workers per lane)
    hb = api.HostBatch().add_lu(40, 160 * 160 * 4).add_qr(40, 160 * 160 * 4)
    b = hb.view()
    pl = [P.assemble("32c4g", 32, 4, True)]
    db = ctx.upload(hb)
    r = ctx.schedule(db, pl, "inspirit")
    oa = po.attributes(b, pl[0].costs, abi.ATTR_ALL)
    for k in ("ability", "efficiency", "static_priority", "unit_time_ms"):
        eq(r["attr_" + k], oa[k], k)
    reg = [po.default_regulator_config(b, g, pl[0]) for g in range(2)]
    for pol in ("dmda", "inspirit"):
        g = ctx.simulate(db, pl, pol, reg, attrs=oa, record=True)
        o = po.simulate(b, pl, pol, reg=reg, attrs=oa, record=True)
        for k in SIM_KEYS:
            eq(g[k], o[k], f"{pol}/{k}")


@pytest.mark.parametrize("policy", abi.POLICIES)
def test_c3_matches_the_reference_library(ctx, policy):
    """BASELINE configs[2] against the reference library itself (oracle/_ref:
    the reference sources compiled unmodified), every policy: the LU DAG is
    the reference's own generator, the QR DAG this repo's (the reference has
    none), both scheduled by the reference's compute_attributes + simulate."""
    from oracle import pyref
    if not pyref.available():
        pytest.skip("oracle/_ref not built")
    hb = api.HostBatch().add_lu(40, 160 * 160 * 4).add_qr(40, 160 * 160 * 4)
    b = hb.view()
    pl = [P.assemble("32c4g", 32, 4, True)]
    r = ctx.schedule(ctx.upload(hb), pl, policy)
    ra = pyref.attributes(b, pl[0].costs, abi.ATTR_ALL, threads=2)
    rs = pyref.simulate(b, pl, policy, attrs=ra, record=False, threads=2)
    for k in ("ability", "efficiency", "static_priority"):
        eq(r["attr_" + k], ra[k], k)
    for k in ("worker", "start_ms", "end_ms", "makespan_ms"):
        eq(r[k], rs[k], f"{policy}/{k}")


def _long_edge_graph(seed, n, levels, p_long):
    """Layered DAG plus random long edges (edge spans > 1 exercise the
    pruning history and the reverse live ranges)."""
    rng = np.random.default_rng(seed)
    tasks = []
    per = n // levels
    for i in range(n):
        lv = i // per
        deps = []
        if lv > 0:
            prev = list(range((lv - 1) * per, lv * per))
            deps = [int(x) for x in rng.choice(prev, size=min(3, per), replace=False)]
            if lv > 2 and rng.random() < p_long:
                deps.append(int(rng.integers(0, (lv - 2) * per)))
        tasks.append(TaskNode(i, MIXED[int(rng.integers(0, 4))], deps))
    return GraphBatch.from_taskgraphs([TaskGraph("long", tasks)], P.TYPE_NAMES)


@pytest.mark.parametrize("kind", ["layered", "long_edges", "span_beyond_64"])
def test_large_graph_path_matches_batched_path_and_oracle(ctx, kind):
    costs = P.default_cost_table()
    if kind == "layered":
        b = api.HostBatch().add_layered(12288, 96, 1.0 / 32, [5]).view()
    elif kind == "long_edges":
        b = _long_edge_graph(3, 6000, 60, 0.3)
    else:
        b = _long_edge_graph(4, 4000, 200, 0.05)
    db = ctx.upload(b)
    ctx.set_large_graph_threshold(1 << 30)
    small = ctx.attributes(db, costs, abi.ATTR_ALL)
    ctx.set_large_graph_threshold(1000)
    try:
        large = ctx.attributes(db, costs, abi.ATTR_ALL)
        ab_only = ctx.attributes(db, costs, abi.ATTR_ABILITY)
        eff3 = ctx.attributes(db, costs, abi.ATTR_EFFICIENCY, unit_time=[3.0])
    finally:
        ctx.set_large_graph_threshold(65536)
    for k in ("ability", "efficiency", "static_priority", "unit_time_ms"):
        eq(large[k], small[k], f"large vs batched {k}")
    eq(ab_only["ability"], small["ability"], "closure ability")
    o = po.attributes(b, costs, abi.ATTR_ALL)
    for k in ("ability", "efficiency", "static_priority", "unit_time_ms"):
        eq(large[k], o[k], f"large vs oracle {k}")
    o3 = po.attributes(b, costs, abi.ATTR_EFFICIENCY, unit_time=[3.0])
    eq(eff3["efficiency"], o3["efficiency"], "pruned single window")


@pytest.mark.parametrize("shape", [(1000, 10, 0.05), (4096, 10, 0.05), (300, 7, 0.2), (64, 64, 0.5), (50, 1, 0.1)])
def test_device_generator_is_bit_identical_to_host(ctx, shape):
    n, L, p = shape
    seeds = np.array([0, 1, 2, 17, 123456789, 2**63 + 5], np.uint64)
    dev = ctx.generate_layered(n, L, p, seeds).download()
    host = api.HostBatch().add_layered(n, L, p, seeds).view()
    for k in ("task_base", "edge_base", "handle_base", "in_base", "out_base", "dep_off", "dep", "in_off", "in_",
              "out_off", "out", "type", "handle_bytes"):
        eq(getattr(dev, k), getattr(host, k), k)


def test_device_generated_batch_schedules_like_host_batch(ctx):
    seeds = np.arange(300, 556)
    pl = [P.assemble("8c2g", 8, 2)]
    a = ctx.schedule(ctx.generate_layered(1000, 10, 0.05, seeds), pl, "inspirit")
    b = ctx.schedule(ctx.upload(api.HostBatch().add_layered(1000, 10, 0.05, seeds)), pl, "inspirit")
    for k in ("worker", "start_ms", "end_ms", "makespan_ms", "attr_efficiency", "attr_ability"):
        eq(a[k], b[k], k)


def test_upload_stream_pipeline_matches_serial(ctx):
    """Uploads on a second stream (step k+1's copies overlapping step k's
    kernels, freed batch memory recycled through the pool) give the same
    schedules as serial upload-then-compute."""
    import torch
    pl = [P.assemble("8c2g", 8, 2)]
    batches = [api.HostBatch().add_layered(600 + 37 * i, 6 + i, 0.04 + 0.01 * i, np.arange(50 * i, 50 * i + 64))
               for i in range(4)]
    serial = [ctx.schedule(ctx.upload(hb), pl, "inspirit") for hb in batches]
    up = torch.cuda.Stream()
    ctx.set_upload_stream(up.cuda_stream)
    try:
        for _ in range(2):  # second pass reuses pooled batch memory
            nxt = ctx.upload(batches[0])
            for i in range(len(batches)):
                cur = nxt
                if i + 1 < len(batches):
                    nxt = ctx.upload(batches[i + 1])
                got = ctx.schedule(cur, pl, "inspirit")
                cur.free()
                for k in ("worker", "start_ms", "end_ms", "makespan_ms", "attr_efficiency", "attr_ability"):
                    eq(got[k], serial[i][k], f"{k} batch {i}")
    finally:
        ctx.set_upload_stream(None)


def test_async_results_match_synchronous(ctx):
    """Asynchronous results (D2H on the download stream, two staging sets):
    every call's host arrays hold that call's schedules once synchronized,
    including arrays reused by a later call."""
    import torch
    pl = [P.assemble("8c2g", 8, 2)]
    batches = [api.HostBatch().add_layered(500 + 41 * i, 7, 0.05, np.arange(40 * i, 40 * i + 48)) for i in range(5)]
    serial = [ctx.schedule(ctx.upload(hb), pl, "inspirit", want_attrs=False) for hb in batches]
    keys = ("worker", "start_ms", "end_ms", "makespan_ms", "completed")
    ctx.set_async_results(True)
    try:
        outs = []
        for i, hb in enumerate(batches):
            T, G = hb.view().n_tasks, hb.view().n_graphs
            arr = {"worker": torch.empty(T, dtype=torch.int32, pin_memory=True).numpy(),
                   "start_ms": torch.empty(T, dtype=torch.float64, pin_memory=True).numpy(),
                   "end_ms": torch.empty(T, dtype=torch.float64, pin_memory=True).numpy(),
                   "makespan_ms": torch.empty(G, dtype=torch.float64, pin_memory=True).numpy(),
                   "completed": torch.empty(G, dtype=torch.int64, pin_memory=True).numpy()}
            outs.append(ctx.schedule(ctx.upload(hb), pl, "inspirit", want_attrs=False, out_arrays=arr,
                                     want_states=False))
        ctx.synchronize()
        for i, got in enumerate(outs):
            for k in keys:
                eq(got[k], serial[i][k], f"async {k} call {i}")
    finally:
        ctx.set_async_results(False)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind", ["layered", "long_edges"])
def test_sharded_large_graph_attributes_match_single_gpu(ctx, world, kind):
    """Multi-GPU attributes of one large graph, emulated with
    one context per rank on this GPU: closure word ranges + sweep source
    ranges + summed partials equal the single-GPU compute_attributes."""
    costs = P.default_cost_table()
    if kind == "layered":
        b = api.HostBatch().add_layered(12288, 96, 1.0 / 32, [5]).view()
    else:
        b = _long_edge_graph(3, 6000, 60, 0.3)
    db = ctx.upload(b)
    ctx.set_large_graph_threshold(1000)
    ctxs = [api.Context(0) for _ in range(world)]
    try:
        want = ctx.attributes(db, costs, abi.ATTR_ALL)
        for c in ctxs:
            c.set_large_graph_threshold(1000)
        dbs = [c.upload(b) for c in ctxs]
        parts = [c.attributes_shard_partial(d, costs, r, world) for r, (c, d) in enumerate(zip(ctxs, dbs))]
        ab = sum(p[0] for p in parts)
        sums = sum(p[1] for p in parts)
        fins = [c.attributes_shard_finish(d, sums) for c, d in zip(ctxs, dbs)]
    finally:
        ctx.set_large_graph_threshold(65536)
    eq(ab, want["ability"], "ability")
    eq(sum(f["efficiency"] for f in fins), want["efficiency"], "efficiency")
    for f in fins:
        for k in ("static_priority", "unit_time_ms", "w0_ms", "best_score", "w0_score", "evaluations"):
            eq(f[k], want[k] if k in want else f[k], k)


def test_mixed_width_batch_more_graphs_than_warps(ctx):
    """A batch mixing <= 32-worker platforms with a 36-worker one (C5's mixes,
    two workers per lane) and more graphs than resident warps -- enough of
    each that the <= 32-worker graphs run in their own launch: schedules and
    ledgers equal the oracle's for every graph and policy."""
    G = 4 * 148 + 40
    b = api.HostBatch().add_layered(90, 6, 0.12, np.arange(G)).view()
    pls = [P.assemble(f"{c}c{g}g", c, g) for c, g in ((4, 1), (8, 2), (16, 2), (32, 4))]
    pof = (np.arange(G) % 4).astype(np.int32)
    costs = P.default_cost_table()
    db = ctx.upload(b)
    oa = po.attributes(b, costs, abi.ATTR_ALL)
    reg = [po.default_regulator_config(b, g, pls[pof[g]]) for g in range(G)]
    for pol in ("dmda", "inspirit"):
        g_ = ctx.simulate(db, pls, pol, reg, platform_of=pof, attrs=oa, record=True)
        o = po.simulate(b, pls, pol, platform_of=pof, reg=reg, attrs=oa, record=True)
        for k in SIM_KEYS:
            eq(g_[k], o[k], f"{pol}/{k}")
    s = ctx.schedule(db, pls, "inspirit", platform_of=pof, want_attrs=False)
    o = po.simulate(b, pls, "inspirit", platform_of=pof, reg=reg, attrs=oa, record=False)
    eq(s["makespan_ms"], o["makespan_ms"], "schedule makespans")


@pytest.mark.parametrize("policy", ["dmda", "dmdap", "inspirit"])
def test_many_input_tasks_match_oracle(ctx, policy):
    """Tasks reading ~30 inputs on 2..5 memory nodes select the kernels
    whose transfer sums run in rounds and skip resident inputs (1 and 2
    worker slots per lane): every schedule equals the oracle's."""
    hb = api.HostBatch().add_layered(400, 4, 0.3, np.arange(12))
    b = hb.view()
    mixes = [(4, 1), (8, 2), (16, 2), (32, 4)]
    costs = P.default_cost_table()
    oa = po.attributes(b, costs, abi.ATTR_ALL)
    db = ctx.upload(b)
    for sel in ([0, 1, 2], [0, 1, 2, 3]):  # <= 32 workers, then up to 36
        pls = [P.assemble(f"{c}c{g}g", c, g) for c, g in (mixes[i] for i in sel)]
        pof = (np.arange(b.n_graphs) % len(sel)).astype(np.int32)
        reg = [po.default_regulator_config(b, g, pls[pof[g]]) for g in range(b.n_graphs)]
        g_ = ctx.simulate(db, pls, policy, reg, attrs=oa, record=True, platform_of=pof)
        o = po.simulate(b, pls, policy, platform_of=pof, reg=reg, attrs=oa, record=True)
        for k in SIM_KEYS:
            eq(g_[k], o[k], f"{policy} {sel} {k}")


def test_queue_overflow_rerun_matches_oracle(ctx):
    """Many graphs (shared-memory state with short queues) plus two whose
    first level puts hundreds of tasks on 10 workers at once: those overflow
    their shared-memory queues and are re-run with HBM state -- every
    schedule still equals the oracle's."""
    G = 2 * 148 * 4
    hb = api.HostBatch().add_layered(120, 6, 0.1, np.arange(G)).add_layered(1500, 2, 0.01, [5, 6])
    b = hb.view()
    pl = [P.assemble("8c2g", 8, 2)]
    costs = P.default_cost_table()
    db = ctx.upload(b)
    oa = po.attributes(b, costs, abi.ATTR_ALL)
    reg = [po.default_regulator_config(b, g, pl[0]) for g in range(b.n_graphs)]
    ctx.set_timing(True)
    try:
        g_ = ctx.simulate(db, pl, "inspirit", reg, attrs=oa, record=True)
        rerun_ms = ctx.last_kernel_ms("k_simulate_rerun")
    finally:
        ctx.set_timing(False)
    o = po.simulate(b, pl, "inspirit", reg=reg, attrs=oa, record=True)
    for k in SIM_KEYS:
        eq(g_[k], o[k], k)
    assert rerun_ms > 0.0, "the wide graphs were expected to overflow into the HBM rerun"


_C2_REF = {}


def _c2_reference():
    """C2's host batch and the reference's attributes of all 4096 DAGs (once)."""
    from oracle import pyref
    if "b" not in _C2_REF:
        hb = api.HostBatch().add_layered(1000, 10, 0.05, np.arange(4096))
        _C2_REF["hb"] = hb
        _C2_REF["b"] = hb.view()
        _C2_REF["ra"] = pyref.attributes(_C2_REF["b"], P.default_cost_table(), abi.ATTR_ALL,
                                         threads=pyref.max_threads())
    return _C2_REF["hb"], _C2_REF["b"], _C2_REF["ra"]


@pytest.mark.parametrize("policy", abi.POLICIES)
def test_c2_every_dag_matches_the_reference(ctx, policy):
    """BASELINE configs[1] in full: all 4096 layered DAGs of C2 scheduled on
    the device equal the reference implementation (oracle/_ref, the reference
    sources compiled unmodified, on all host threads) under every policy --
    attributes, every assignment, every start/end double and every
    makespan."""
    from oracle import pyref
    if not pyref.available():
        pytest.skip("oracle/_ref not built")
    hb, b, ra = _c2_reference()
    pl = [P.assemble("8c2g", 8, 2)]
    r = ctx.schedule(ctx.upload(hb), pl, policy)
    rs = pyref.simulate(b, pl, policy, attrs=ra, record=False, threads=pyref.max_threads())
    for k in ("ability", "efficiency", "static_priority"):
        eq(r["attr_" + k], ra[k], k)
    for k in ("worker", "start_ms", "end_ms", "makespan_ms"):
        eq(r[k], rs[k], f"{policy}/{k}")


@pytest.mark.parametrize("policy", abi.POLICIES)
def test_c5_one_percent_sample_matches_the_reference(ctx, policy):
    """BASELINE configs[4]: a 1% sample (every 100th seed of a GPU's 8192) of
    the 4096-task layered DAGs on the four worker mixes (seed mod 4),
    generated on the device, equals the reference implementation under every
    policy."""
    from oracle import pyref
    if not pyref.available():
        pytest.skip("oracle/_ref not built")
    seeds = np.arange(0, 8192, 100, dtype=np.uint64)
    mixes = [(4, 1), (8, 2), (16, 2), (32, 4)]
    pls = [P.assemble(f"{c}c{g}g", c, g) for c, g in mixes]
    pof = (seeds % 4).astype(np.int32)
    db = ctx.generate_layered(4096, 10, 0.05, seeds)
    r = ctx.schedule(db, pls, policy, platform_of=pof)
    if "c5" not in _C2_REF:  # the reference's attributes of the sample, once
        b5 = api.HostBatch().add_layered(4096, 10, 0.05, seeds).view()
        _C2_REF["c5"] = (b5, pyref.attributes(b5, P.default_cost_table(), abi.ATTR_ALL, threads=pyref.max_threads()))
    b, ra = _C2_REF["c5"]
    rs = pyref.simulate(b, pls, policy, platform_of=pof, attrs=ra, record=False, threads=pyref.max_threads())
    for k in ("ability", "efficiency", "static_priority"):
        eq(r["attr_" + k], ra[k], k)
    for k in ("worker", "start_ms", "end_ms", "makespan_ms"):
        eq(r[k], rs[k], f"{policy}/{k}")


def _star_batch(m):
    """Root (LAYERK3) -> m UNIT leaves, built as CSR directly."""
    n = m + 1
    z = lambda k: np.zeros(k, np.int64)
    dep_off = np.concatenate([[0], np.arange(0, m + 1)]).astype(np.int32)
    type_ = np.full(n, P.TYPE_ID["UNIT"], np.int32)
    type_[0] = P.TYPE_ID["LAYERK3"]
    return GraphBatch([0, n], [0, m], [0, 0], [0, 0], [0, 0], dep_off, np.zeros(m, np.int32),
                      np.zeros(n + 1, np.int32), np.zeros(0, np.int32), np.zeros(n + 1, np.int32),
                      np.zeros(0, np.int32), type_, z(0), P.TYPE_NAMES)


@pytest.mark.parametrize("path", ["large", "batched"])
def test_window_bins_hold_more_than_2_21_descendants(ctx, path):
    """A source with more than 2^21 descendants in ONE calibration window bin
    (a 2^21+1000-leaf star: every leaf at distance 1.0 = W_3).  The bins were
    21-bit fields in round 1 (ADVICE: silent carry into the next bin); they
    are 32-bit counters now.  Expected values are analytic: w0 = 2 (lower
    median 1), windows 2^(k-3); the root counts m leaves from W = 1 on, so
    the score is 1 below k = 3 and 2 from k = 3 (strict > keeps W = 1)."""
    m = (1 << 21) + 1000
    b = _star_batch(m)
    db = ctx.upload(b)
    costs = P.default_cost_table()
    ctx.set_large_graph_threshold(65536 if path == "large" else 1 << 30)
    try:
        a = ctx.attributes(db, costs, abi.ATTR_ALL)
        c = ctx.attributes(db, costs, abi.ATTR_CALIBRATE)
        e = ctx.attributes(db, costs, abi.ATTR_EFFICIENCY, unit_time=[64.0])
    finally:
        ctx.set_large_graph_threshold(65536)
    assert a["ability"][0] == m and not a["ability"][1:].any()
    assert a["efficiency"][0] == m and not a["efficiency"][1:].any()
    assert a["unit_time_ms"][0] == 1.0
    assert (c["w0_ms"][0], c["best_score"][0], c["w0_score"][0], c["evaluations"][0]) == (2.0, 2, 2, 11)
    assert e["efficiency"][0] == m
    assert a["static_priority"][0] == 15000 and (a["static_priority"][1:] == 1000).all()


def test_shard_finish_rejects_scratch_reused_in_between(ctx):
    """a shard finish after another attribute pass on the same
    context (which reuses/regrows the scratch the partial left) is rejected
    instead of reading overwritten data."""
    costs = P.default_cost_table()
    b = _long_edge_graph(3, 6000, 60, 0.3)
    c = api.Context(0)
    c.set_large_graph_threshold(1000)
    db = c.upload(b)
    ab, sums = c.attributes_shard_partial(db, costs, 0, 2)
    c.attributes(db, costs, abi.ATTR_ALL)
    with pytest.raises(api.TbsimError):
        c.attributes_shard_finish(db, sums)


def test_csr_cache_feeds_upload_with_identical_schedules(ctx, tmp_path):
    """A batch saved to the binary CSR cache and loaded back uploads and
    schedules exactly like the generated one."""
    hb = api.HostBatch().add_layered(800, 8, 0.05, np.arange(40)).add_lu(6, 640)
    p = str(tmp_path / "b.csr")
    hb.save(p)
    pl = [P.assemble("8c2g", 8, 2)]
    a = ctx.schedule(ctx.upload(hb), pl, "inspirit")
    b = ctx.schedule(ctx.upload(api.HostBatch.load(p)), pl, "inspirit")
    for k in ("worker", "start_ms", "end_ms", "makespan_ms", "attr_ability", "attr_efficiency"):
        eq(a[k], b[k], k)


@pytest.mark.parametrize("kind", ["cholesky", "lu", "qr"])
@pytest.mark.parametrize("nb", [1, 2, 3, 10, 40])
def test_device_tiled_generators_are_bit_identical_to_host(ctx, kind, nb):
    """tiled Cholesky / LU / QR built on the device equal the
    host builders (which replay generators.cpp:30-142) section by section."""
    bytes_ = 160 * 160 * 4
    dev = ctx.generate_tiled(kind, nb, bytes_, count=3).download()
    hb = api.HostBatch()
    for _ in range(3):
        getattr(hb, "add_" + kind)(nb, bytes_)
    host = hb.view()
    for k in ("task_base", "edge_base", "handle_base", "in_base", "out_base", "dep_off", "dep", "in_off", "in_",
              "out_off", "out", "type", "handle_bytes"):
        eq(getattr(dev, k), getattr(host, k), f"{kind}{nb}:{k}")


def test_async_schedule_defers_errors_to_synchronize(ctx):
    """Asynchronous results: schedule() makes no host round trip, so its
    errors (the reference's texts) surface at synchronize() -- a missing GPU
    cost (compute_attributes), a cycle, a task no worker can run -- and a
    good call on the same context is unaffected."""
    gonly_pl = P.make_preset("homog2")
    gonly_pl.costs = P.CostTable()
    gonly_pl.costs.set("GONLY_TYPE", P.GPU, 1.0)
    gonly = GraphBatch.from_taskgraphs([TaskGraph("g", [TaskNode(0, "GONLY_TYPE")])])
    cyc = _tg([TaskNode(0, "UNIT", [1]), TaskNode(1, "UNIT", [0])])
    good = api.HostBatch().add_layered(200, 5, 0.1, np.arange(8))
    want = ctx.schedule(ctx.upload(good), [P.assemble("8c2g", 8, 2)], "inspirit", want_attrs=False)
    ctx.set_async_results(True)
    try:
        for batch, pl, msg in ((gonly, gonly_pl, "no worker can run task type GONLY_TYPE"),
                               (cyc, P.assemble("8c2g", 8, 2), "graph has a dependency cycle")):
            ctx.schedule(ctx.upload(batch), [pl], "dmda", want_attrs=False, want_states=False)
            with pytest.raises(api.TbsimRuntimeError, match=msg):
                ctx.synchronize()
        got = ctx.schedule(ctx.upload(good), [P.assemble("8c2g", 8, 2)], "inspirit", want_attrs=False,
                           want_states=False)
        ctx.synchronize()
        for k in ("worker", "start_ms", "end_ms", "makespan_ms"):
            eq(got[k], want[k], k)
    finally:
        ctx.set_async_results(False)


def test_async_schedule_reruns_queue_overflows_on_the_device(ctx):
    """The overflow rerun list is built on the device in asynchronous mode:
    the same schedules as the synchronous call."""
    G = 2 * 148 * 4
    hb = api.HostBatch().add_layered(120, 6, 0.1, np.arange(G)).add_layered(1500, 2, 0.01, [5, 6])
    pl = [P.assemble("8c2g", 8, 2)]
    db = ctx.upload(hb)
    want = ctx.schedule(db, pl, "inspirit", want_attrs=False)
    ctx.set_async_results(True)
    ctx.set_timing(True)
    try:
        got = ctx.schedule(db, pl, "inspirit", want_attrs=False, want_states=False)
        ctx.synchronize()
        rerun_ms = ctx.last_kernel_ms("k_simulate_rerun")
    finally:
        ctx.set_timing(False)
        ctx.set_async_results(False)
    for k in ("worker", "start_ms", "end_ms", "makespan_ms", "completed"):
        eq(got[k], want[k], k)
    assert rerun_ms > 0.0


def _edge_shapes():
    """Degenerate shapes the reference accepts: an empty graph, one task,
    no edges, a chain, a star (one source, 49 sinks) and a join (50 sources
    into one task)."""
    return [TaskGraph("empty", []),
            TaskGraph("one", [TaskNode(0, "UNIT")]),
            TaskGraph("flat", [TaskNode(i, "LAYERK1") for i in range(40)]),
            TaskGraph("chain", [TaskNode(i, "LAYERK2", [i - 1] if i else []) for i in range(60)]),
            TaskGraph("star", [TaskNode(0, "LAYERK3")] + [TaskNode(i, "LAYERK0", [0]) for i in range(1, 50)]),
            TaskGraph("join", [TaskNode(i, "LAYERK0") for i in range(50)] + [TaskNode(50, "LAYERK3", list(range(50)))])]


def test_degenerate_shapes_match_oracle(ctx):
    b = GraphBatch.from_taskgraphs(_edge_shapes(), P.TYPE_NAMES)
    costs = P.default_cost_table()
    db = ctx.upload(b)
    for req, keys in ((abi.ATTR_ABILITY, ("ability",)), (abi.ATTR_LAYERS, ("layer",)), (abi.ATTR_DEPTH, ("depth",))):
        g, o = ctx.attributes(db, costs, req), po.attributes(b, costs, req)
        for k in keys:
            eq(g[k], o[k], k)
    pls = [P.make_preset("26cpu_2gpu"), P.make_preset("homog2")]
    pof = np.arange(b.n_graphs) % 2
    reg = [abi.RegulatorCfg(task_window=2, s_inc=4, k_inc=1.0, s_dec=2, c=1, dec_step=2, slope_samples=8)] * b.n_graphs
    for pol in abi.POLICIES:
        g = ctx.simulate(db, pls, pol, reg, platform_of=pof, record=True)
        o = po.simulate(b, pls, pol, platform_of=pof, reg=reg, record=True)
        for k in SIM_KEYS:
            eq(g[k], o[k], f"{pol}/{k}")
    # the full pipeline on the non-empty shapes (an empty graph has no median)
    nb = GraphBatch.from_taskgraphs(_edge_shapes()[1:], P.TYPE_NAMES)
    ndb = ctx.upload(nb)
    oa = po.attributes(nb, costs, abi.ATTR_ALL)
    ga = ctx.attributes(ndb, costs, abi.ATTR_ALL)
    for k in ("ability", "efficiency", "static_priority", "unit_time_ms"):
        eq(ga[k], oa[k], k)
    r = ctx.schedule(ndb, [pls[0]], "inspirit")
    nreg = [po.default_regulator_config(nb, i, pls[0]) for i in range(nb.n_graphs)]
    o = po.simulate(nb, [pls[0]], "inspirit", reg=nreg, attrs=oa, record=False)
    for k in ("worker", "start_ms", "end_ms", "makespan_ms"):
        eq(r[k], o[k], k)


def test_wide_state_simulators_match_oracle(ctx):
    """The non-compact simulator kernels (32-bit unmet counters, 64-bit
    event slots): graphs of >= 32768 tasks, and platforms of more than 8
    memory nodes, each with one and with two workers per lane."""
    costs = P.default_cost_table()
    # more than 8 memory nodes: random graphs on 4c9g (13 workers) and 32c9g (41)
    b = random_graphs(11, 24)
    pls = [P.assemble("4c9g", 4, 9), P.assemble("32c9g", 32, 9)]
    db = ctx.upload(b)
    oa = po.attributes(b, costs, abi.ATTR_ALL)
    for pl in pls:
        reg = [po.default_regulator_config(b, g, pl) for g in range(b.n_graphs)]
        for pol in abi.POLICIES:
            g = ctx.simulate(db, [pl], pol, reg, attrs=oa, record=True)
            o = po.simulate(b, [pl], pol, reg=reg, attrs=oa, record=True)
            for k in SIM_KEYS:
                eq(g[k], o[k], f"{pl.name}/{pol}/{k}")
    # >= 32768 tasks (the attributes are the device's, pinned elsewhere)
    hb = api.HostBatch().add_layered(40000, 40, 0.002, 3)
    lb = hb.view()
    ldb = ctx.upload(hb)
    ga = ctx.attributes(ldb, costs, abi.ATTR_ALL)
    for pl in (P.assemble("4c1g", 4, 1), P.assemble("32c4g", 32, 4)):
        reg = [po.default_regulator_config(lb, 0, pl)]
        for pol in ("dmda", "inspirit"):
            g = ctx.simulate(ldb, [pl], pol, reg, attrs=ga, record=True)
            o = po.simulate(lb, [pl], pol, reg=reg, attrs=ga, record=True)
            for k in SIM_KEYS:
                eq(g[k], o[k], f"40k/{pl.name}/{pol}/{k}")


def test_contexts_on_concurrent_host_threads_match_serial():
    """one context (and stream) per calling thread.  Four host
    threads schedule different batches at once on the same GPU (ctypes drops
    the GIL in the calls); every result equals the same batch run alone."""
    import threading
    pl = [P.assemble("8c2g", 8, 2)]
    seeds = [np.arange(64 * k, 64 * k + 64, dtype=np.uint64) for k in range(4)]
    hbs = [api.HostBatch().add_layered(1000, 10, 0.05, s) for s in seeds]

    def run(hb):
        c = api.Context(0)
        try:
            r = c.schedule(c.upload(hb), pl, "inspirit")
            return {k: np.array(r[k]) for k in ("worker", "start_ms", "end_ms", "makespan_ms")}
        finally:
            c.close()

    serial = [run(hb) for hb in hbs]
    out, errs = [None] * 4, []

    def worker(i):
        try:
            for _ in range(3):
                out[i] = run(hbs[i])
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for i in range(4):
        for k, v in serial[i].items():
            eq(out[i][k], v, f"thread {i}: {k}")
