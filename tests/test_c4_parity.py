"""C4 (one 1M-task DAG, BASELINE configs[3]) against the reference itself at
the configuration's own scale (oracle/c4check.py, oracle/ref_c4.cpp):
ability / upward rank / depth / layers bit-exact in full, efficiency at all
11 calibration windows on sampled sources through the reference's own
efficiency_of, calibration re-scored from the device's per-window vectors.
The CPU tests pin the checker itself against the reference's public API."""
import numpy as np
import pytest

from oracle import c4check, pyref
from paper_2404_03226_b200 import abi, api
from paper_2404_03226_b200 import platform as P

needs_ref = pytest.mark.skipif(not pyref.available() or not __import__("os").path.exists(pyref.C4_LIB_PATH),
                               reason="oracle/_ref not built")


@needs_ref
def test_c4_adapter_matches_reference_public_api():
    """ref_c4's structure + per-source efficiency_of and the numpy score_of
    restatement reproduce ref_attributes (compute_attributes,
    calibrate_unit_time, compute_inspiring_efficiency) on a 3000-task DAG."""
    b = api.HostBatch().add_layered(3000, 30, 0.02, [7]).view()
    costs = P.default_cost_table()
    r = pyref.C4Ref(b, costs)
    s = r.structure(threads=4)
    full = pyref.attributes(b, costs, abi.ATTR_ALL)
    np.testing.assert_array_equal(s["ability"], full["ability"])
    np.testing.assert_array_equal(s["static_priority"], full["static_priority"])
    np.testing.assert_array_equal(s["depth"], pyref.attributes(b, costs, abi.ATTR_DEPTH)["depth"])
    np.testing.assert_array_equal(s["layer"], pyref.attributes(b, costs, abi.ATTR_LAYERS)["layer"])
    cal = pyref.attributes(b, costs, abi.ATTR_CALIBRATE)
    assert s["w0_ms"] == cal["w0_ms"][0]
    ws = [float(np.ldexp(s["w0_ms"], k - 4)) for k in range(11)]
    per_w = np.stack([pyref.attributes(b, costs, abi.ATTR_EFFICIENCY, unit_time=[w])["efficiency"] for w in ws])
    src = np.arange(b.n_tasks)
    e, _, _ = r.efficiency_sample(src, ws, threads=4)
    np.testing.assert_array_equal(e.T, per_w)
    sc = c4check.class_scores(per_w, s["layer"], b.type)
    best = int(np.argmax(sc))
    assert (sc[best], sc[4], ws[best]) == (cal["best_score"][0], cal["w0_score"][0], cal["unit_time_ms"][0])


@needs_ref
@pytest.mark.gpu
def test_c4_large_path_against_reference_full_sample(ctx):
    """The large-graph kernels (closure, cooperative structure/finalize,
    pruned sweep) on a 65536-task DAG: every source checked."""
    b = api.HostBatch().add_layered(1 << 16, 64, 1.0 / 64, [3])
    gb = b.view()
    rep = c4check.check(ctx, ctx.upload(b), gb, P.default_cost_table(), n_sample=gb.n_tasks)
    assert rep["mismatch"] == [], rep


@needs_ref
@pytest.mark.gpu
def test_c4_config_scale_against_reference(ctx):
    """BASELINE configs[3] itself: generate_layered_dag(1048576, 1024, 1/256,
    seed 1)."""
    hb = api.HostBatch().add_layered(1 << 20, 1024, 1.0 / 256, [1])
    rep = c4check.check(ctx, ctx.upload(hb), hb.view(), P.default_cost_table(), n_sample=96)
    assert rep["mismatch"] == [], rep
