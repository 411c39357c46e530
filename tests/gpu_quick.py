"""Quick GPU parity probe (developer script; the real suite is pytest -m gpu)."""
import sys
import time
import traceback

import numpy as np

sys.path.insert(0, ".")
from oracle import pyoracle as po  # noqa: E402
from paper_2404_03226_b200 import abi, api  # noqa: E402
from paper_2404_03226_b200 import platform as P  # noqa: E402

costs = P.default_cost_table(with_qr=True)


def cmp(name, a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape or not np.array_equal(a, b):
        idx = np.nonzero(a != b)[0][:10] if a.shape == b.shape else []
        print(f"  MISMATCH {name}: shapes {a.shape} {b.shape} first idx {idx} got {a[idx] if len(idx) else ''} want {b[idx] if len(idx) else ''}")
        return False
    return True


def main():
    ctx = api.Context(0)
    hb = api.HostBatch().add_layered(1000, 10, 0.05, np.arange(4)).add_cholesky(10, 960 * 960 * 4).add_lu(8, 160 * 160 * 4)
    hb.add_qr(6, 160 * 160 * 4)
    gb = hb.view()
    db = ctx.upload(hb)
    print("uploaded", gb.n_graphs, gb.n_tasks, "h2d", db.h2d_bytes)
    ok = True
    t = time.time()
    ga = ctx.attributes(db, costs, abi.ATTR_ALL)
    print("gpu attrs", time.time() - t)
    oa = po.attributes(gb, costs, abi.ATTR_ALL)
    for k in ["ability", "efficiency", "static_priority", "unit_time_ms"]:
        ok &= cmp("attr " + k, ga[k], oa[k])
    for req, keys in [(abi.ATTR_LAYERS, ["layer"]), (abi.ATTR_DEPTH, ["depth"]), (abi.ATTR_ABILITY, ["ability"]),
                      (abi.ATTR_CALIBRATE, ["unit_time_ms", "w0_ms", "best_score", "w0_score", "evaluations"]),
                      (abi.ATTR_RANK, ["static_priority"])]:
        g2 = ctx.attributes(db, costs, req)
        o2 = po.attributes(gb, costs, req)
        for k in keys:
            ok &= cmp(f"req{req} {k}", g2[k], o2[k])
    ut = np.full(gb.n_graphs, 3.0)
    g3 = ctx.attributes(db, costs, abi.ATTR_EFFICIENCY, unit_time=ut)
    o3 = po.attributes(gb, costs, abi.ATTR_EFFICIENCY, unit_time=ut)
    ok &= cmp("eff@3", g3["efficiency"], o3["efficiency"])
    pl = [P.assemble("4c1g", 4, 1, True), P.assemble("8c2g", 8, 2, True), P.assemble("32c4g", 32, 4, True)]
    pof = np.array([1, 1, 1, 1, 0, 2, 0], np.int32)
    reg = [po.default_regulator_config(gb, g, pl[pof[g]]) for g in range(gb.n_graphs)]
    for pol in abi.POLICIES:
        try:
            t = time.time()
            gs = ctx.simulate(db, pl, pol, reg, platform_of=pof, attrs=oa, record=True)
            el = time.time() - t
            os_ = po.simulate(gb, pl, pol, platform_of=pof, reg=reg, attrs=oa, record=True)
            good = True
            for k in ["worker", "start_ms", "end_ms", "makespan_ms", "pop_mode_counts", "push_task", "pop_task",
                      "pop_worker", "push_time", "pop_time", "sample_time", "sample_nready"]:
                good &= cmp(f"{pol} {k}", gs[k], os_[k])
            print(pol, "ok" if good else "FAIL", f"{el:.3f}s", gs["makespan_ms"][:3], os_["makespan_ms"][:3])
            ok &= good
        except Exception:
            traceback.print_exc()
            ok = False
    try:
        t = time.time()
        sc = ctx.schedule(db, pl, "inspirit", platform_of=pof)
        el = time.time() - t
        # oracle pipeline: attrs on each graph's platform costs (all same table here)
        os_ = po.simulate(gb, pl, "inspirit", platform_of=pof, reg=reg, attrs=oa, record=False)
        good = cmp("schedule makespan", sc["makespan_ms"], os_["makespan_ms"]) and cmp("schedule worker", sc["worker"], os_["worker"])
        print("schedule", "ok" if good else "FAIL", f"{el:.3f}s")
        ok &= good
    except Exception:
        traceback.print_exc()
        ok = False
    # bigger batch timing
    hb2 = api.HostBatch().add_layered(1000, 10, 0.05, np.arange(4096), threads=0)
    db2 = ctx.upload(hb2)
    pl2 = [P.assemble("8c2g", 8, 2)]
    for it in range(3):
        ctx.synchronize()
        t = time.time()
        sc = ctx.schedule(db2, pl2, "inspirit", want_attrs=False)
        print("schedule 4096 x 1k:", f"{time.time() - t:.4f}s")
    ctx.set_timing(True)
    sc = ctx.schedule(db2, pl2, "inspirit", want_attrs=False)
    for k in ["k_structure", "k_sweep", "k_finalize", "k_simulate", "k_structure_out"]:
        print("  ", k, ctx.last_kernel_ms(k), "ms")
    # parity on a sample of the big batch
    sub = hb2.view().slice(range(0, 4096, 512))
    oa2 = po.attributes(sub, costs, abi.ATTR_ALL)
    reg2 = [po.default_regulator_config(sub, g, pl2[0]) for g in range(sub.n_graphs)]
    os2 = po.simulate(sub, pl2, "inspirit", reg=reg2, attrs=oa2, record=False)
    ok &= cmp("big sample makespan", sc["makespan_ms"][::512], os2["makespan_ms"])
    print("ALL OK" if ok else "SOME FAILURES")


if __name__ == "__main__":
    main()
