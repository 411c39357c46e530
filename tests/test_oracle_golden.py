"""CPU: the C restatement (oracle/oracle.c) against the reference's golden
fixtures and the known-answer tests of the reference's own suite
(proj/tests/test_attributes.cpp, test_regulator.cpp, test_engine.cpp,
proj/README.md goldens)."""
import math

import numpy as np
import pytest

from golden_util import SIM_KEYS, Fixture, names, reg_rows
from oracle import pyoracle as po
from paper_2404_03226_b200 import abi
from paper_2404_03226_b200 import platform as P
from paper_2404_03226_b200.batch import GraphBatch, TaskGraph, TaskNode

FIXTURES = names()


@pytest.mark.parametrize("name", FIXTURES)
def test_oracle_attributes_match_reference(name):
    f = Fixture(name)
    a = po.attributes(f.batch, f.costs, abi.ATTR_ALL, f.prio)
    for k in ("ability", "efficiency", "static_priority", "unit_time_ms"):
        np.testing.assert_array_equal(a[k], f.z["attr_" + k], err_msg=k)
    c = po.attributes(f.batch, f.costs, abi.ATTR_CALIBRATE)
    for k in ("w0_ms", "best_score", "w0_score", "evaluations"):
        np.testing.assert_array_equal(c[k], f.z["calib_" + k], err_msg=k)
    np.testing.assert_array_equal(po.attributes(f.batch, f.costs, abi.ATTR_DEPTH)["depth"], f.z["depth"])
    np.testing.assert_array_equal(po.attributes(f.batch, f.costs, abi.ATTR_LAYERS)["layer"], f.z["layer"])
    np.testing.assert_array_equal(po.attributes(f.batch, f.costs, abi.ATTR_RANK)["static_priority"], f.z["rank"])
    for w in (0.5, 1.0, 4.0, 16.0):
        e = po.attributes(f.batch, f.costs, abi.ATTR_EFFICIENCY, unit_time=np.full(f.batch.n_graphs, w))
        np.testing.assert_array_equal(e["efficiency"], f.z[f"eff_w{w}"])


@pytest.mark.parametrize("name", FIXTURES)
def test_oracle_simulation_matches_reference(name):
    f = Fixture(name)
    for pname in f.platform_names:
        pl = f.platform(pname)
        reg = f.reg_cfgs(pname, po)
        for pol in abi.POLICIES:
            r = po.simulate(f.batch, [pl], pol, reg=reg, attrs=f.attrs(), record=True)
            want = f.sim(pname, pol)
            for k in SIM_KEYS:
                np.testing.assert_array_equal(r[k], want[k], err_msg=f"{pname}/{pol}/{k}")
            if pol == "inspirit":
                np.testing.assert_array_equal(reg_rows(r["reg_state"], f.batch.n_graphs), want["reg"])


def _one(tg, names=None):
    return GraphBatch.from_taskgraphs([tg], names)


def chain3():
    return TaskGraph("c", [TaskNode(0, "UNIT"), TaskNode(1, "UNIT", [0]), TaskNode(2, "UNIT", [1])])


def diamond():
    return TaskGraph("d", [TaskNode(0, "A"), TaskNode(1, "B", [0]), TaskNode(2, "C", [0]), TaskNode(3, "D", [1, 2])])


def test_known_answers_attributes():
    # tests/test_attributes.cpp:37-43
    costs = P.default_cost_table()
    assert po.attributes(_one(chain3()), costs, abi.ATTR_ABILITY)["ability"].tolist() == [2, 1, 0]
    assert po.attributes(_one(diamond()), costs, abi.ATTR_ABILITY)["ability"].tolist() == [3, 1, 1, 0]
    # :55-67 efficiency on a unit chain
    unit = P.CostTable()
    unit.set("UNIT", P.GPU, 1.0)
    b = _one(chain3())
    for w, want in ((0.5, [0, 0, 0]), (1.0, [1, 1, 0]), (2.0, [2, 1, 0])):
        assert po.attributes(b, unit, abi.ATTR_EFFICIENCY, unit_time=[w])["efficiency"].tolist() == want
    with pytest.raises(po.OracleError) as e:
        po.attributes(b, unit, abi.ATTR_EFFICIENCY, unit_time=[-1.0])
    assert e.value.status == abi.TBSIM_E_INVALID_ARGUMENT
    # :69-84 worst path, not the shortest
    t = P.CostTable()
    for n, ms in (("A", 1.0), ("B", 2.0), ("C", 3.0), ("D", 1.0)):
        t.set(n, P.GPU, ms)
    d = _one(diamond())
    assert po.attributes(d, t, abi.ATTR_EFFICIENCY, unit_time=[3.0])["efficiency"].tolist() == [2, 1, 1, 0]
    assert po.attributes(d, t, abi.ATTR_EFFICIENCY, unit_time=[4.0])["efficiency"].tolist() == [3, 1, 1, 0]
    # :137-147 single task: ties keep the smallest candidate
    single = _one(TaskGraph("s", [TaskNode(0, "UNIT")]))
    c = po.attributes(single, costs, abi.ATTR_CALIBRATE)
    assert c["w0_ms"][0] == 2.0 and c["best_score"][0] == 1 and c["w0_score"][0] == 1
    assert c["unit_time_ms"][0] == math.ldexp(2.0, -4)
    # :159-163 upward rank {3000,2000,1000}; :174-176 depth
    assert po.attributes(_one(chain3()), costs, abi.ATTR_RANK)["static_priority"].tolist() == [3000, 2000, 1000]
    assert po.attributes(_one(chain3()), costs, abi.ATTR_DEPTH)["depth"].tolist() == [2, 1, 0]
    assert po.attributes(_one(diamond()), t, abi.ATTR_DEPTH)["depth"].tolist() == [2, 1, 1, 0]


def test_chain_wave_calibration_and_optimum():
    f = Fixture("chain_wave")
    # tests/test_attributes.cpp:149-157
    assert f.z["calib_w0_ms"][0] == 2.0 and f.z["attr_unit_time_ms"][0] == 1.0
    assert f.z["calib_best_score"][0] == 3 and f.z["calib_w0_score"][0] == 3
    # tests/test_engine.cpp:80-103: fifo 5, inspirit 4 (= optimum) on homog2
    assert f.z["sim_homog2_fifo_makespan_ms"][0] == 5.0
    assert f.z["sim_homog2_inspirit_makespan_ms"][0] == 4.0
    assert Fixture("chain_wave_depth").z["sim_homog2_dmdap_makespan_ms"][0] == 4.0


def test_readme_goldens():
    # proj/README.md:81-88,117-125 (re-verified bit-exact by the survey)
    z = Fixture("cholesky").z
    sizes = [4, 6, 8, 10, 12]
    i8, i12 = sizes.index(8), sizes.index(12)
    assert round(z["sim_26cpu_2gpu_dmda_makespan_ms"][i8], 4) == 58.2484
    assert round(z["sim_26cpu_2gpu_inspirit_makespan_ms"][i8], 4) == 54.22
    assert z["sim_26cpu_2gpu_inspirit_pop_mode_counts"][3 * i8:3 * i8 + 3].tolist() == [0, 120, 0]
    assert round(z["sim_26cpu_2gpu_dmda_makespan_ms"][i12], 3) == 115.162
    assert round(z["sim_26cpu_2gpu_inspirit_makespan_ms"][i12], 4) == 112.9496


# ----------------------------------------------------------- regulator
def _cfg(**kw):
    c = abi.RegulatorCfg()
    base = dict(task_window=2, s_inc=1, k_inc=1.0, s_dec=2, c=1, dec_step=2, slope_samples=8)
    base.update(kw)
    for k, v in base.items():
        setattr(c, k, v)
    return c


def test_calculate_k_hand_samples():
    # tests/test_regulator.cpp:36-45
    assert po.calculate_k([]) == 0.0
    assert po.calculate_k([(0.0, 5)]) == 0.0
    assert po.calculate_k([(0.0, 0), (1.0, 2), (2.0, 4)]) == pytest.approx(2.0)
    assert po.calculate_k([(0.0, 3), (1.0, 3), (2.0, 3)]) == 0.0
    assert po.calculate_k([(0.0, 0), (1.0, 1), (2.0, 0)]) == pytest.approx(0.0)
    assert po.calculate_k([(0.0, 0), (2.0, 8)]) == pytest.approx(4.0)
    assert po.calculate_k([(5.0, 1), (5.0, 9)]) == 0.0


def test_regulator_growth_phase():
    # tests/test_regulator.cpp:59-84
    cfg = _cfg(task_window=1, s_inc=1, k_inc=0.5, dec_step=1000)
    st = abi.fresh_regulator_state()
    po.regulator_step(st, cfg, 2, 0.0)
    assert (st.phase, st.mode, st.peak, st.prev_nready) == (abi.PHASE_INC, abi.MODE_EFFICIENCY, 2, 2)
    po.regulator_step(st, cfg, 4, 1.0)
    assert st.mode == abi.MODE_ABILITY and st.cur_k == pytest.approx(2.0) and st.peak == 4
    po.regulator_step(st, cfg, 5, 2.0)
    assert st.mode == abi.MODE_ABILITY
    po.regulator_step(st, cfg, 6, 100.0)
    assert st.cur_k < 0.5 and st.mode == abi.MODE_EFFICIENCY


def test_regulator_drain_bands():
    # tests/test_regulator.cpp:111-158
    cfg = _cfg(task_window=1, s_inc=1000, dec_step=2, s_dec=5, c=1)
    st = abi.fresh_regulator_state()
    st.peak, st.prev_nready, st.last_trigger_nready = 20, 20, 20
    steps = [(18, 1.0, abi.PHASE_INC, abi.MODE_EFFICIENCY, 1), (17, 2.0, abi.PHASE_DEC, abi.MODE_ABILITY, 1),
             (13, 3.0, abi.PHASE_DEC, abi.MODE_ABILITY, 1), (11, 4.0, abi.PHASE_DEC, abi.MODE_LOCALITY, 1),
             (10, 5.0, abi.PHASE_DEC, abi.MODE_LOCALITY, 2), (12, 6.0, abi.PHASE_DEC, abi.MODE_ABILITY, 2),
             (5, 7.0, abi.PHASE_DEC, abi.MODE_LOCALITY, 3)]
    for cur, now, phase, mode, count in steps:
        po.regulator_step(st, cfg, cur, now)
        assert (st.phase, st.mode, st.s_dec_count) == (phase, mode, count), cur
    assert st.peak == 20


def test_regulator_ring_and_window():
    # tests/test_regulator.cpp:47-57, 176-184
    cfg = _cfg(task_window=5)
    st = abi.fresh_regulator_state()
    po.regulator_step(st, cfg, 3, 1.0)
    assert st.n_samples == 1 and st.mode == abi.MODE_EFFICIENCY and st.peak == 0
    cfg = _cfg(task_window=1000, slope_samples=3)
    st = abi.fresh_regulator_state()
    for i in range(5):
        po.regulator_step(st, cfg, i, float(i))
    assert [(st.sample_time[i], st.sample_nready[i]) for i in range(st.n_samples)] == [(2.0, 2), (3.0, 3), (4.0, 4)]


def test_default_regulator_config():
    # tests/test_regulator.cpp:227-247: cholesky 8 on 26cpu_2gpu -> 7/28/28/7/4/7/8
    b = po.gen_cholesky(8, 64)
    cfg = po.default_regulator_config(b, 0, P.make_preset("26cpu_2gpu"))
    assert (cfg.task_window, cfg.s_inc, cfg.k_inc, cfg.s_dec, cfg.c, cfg.dec_step, cfg.slope_samples) == \
        (7, 28, 28.0, 7, 4, 7, 8)
    small = GraphBatch.from_taskgraphs([TaskGraph("c", [TaskNode(0, "UNIT"), TaskNode(1, "UNIT", [0])])], P.TYPE_NAMES)
    cfg = po.default_regulator_config(small, 0, P.make_preset("homog2"))
    assert (cfg.task_window, cfg.s_inc, cfg.s_dec, cfg.c, cfg.dec_step) == (2, 2, 2, 1, 2)


def test_oracle_errors():
    costs = P.default_cost_table()
    cyc = GraphBatch.from_taskgraphs([TaskGraph("x", [TaskNode(0, "UNIT", [1]), TaskNode(1, "UNIT", [0])])],
                                     P.TYPE_NAMES)
    with pytest.raises(po.OracleError, match="dependency cycle"):
        po.attributes(cyc, costs, abi.ATTR_LAYERS)
    reg = [po.default_regulator_config(cyc, 0, P.make_preset("homog2"))]
    with pytest.raises(po.OracleError, match="simulation stuck with 2 tasks unfinished: 0 1"):
        po.simulate(cyc, [P.make_preset("homog2")], "fifo", reg=reg)
    g = GraphBatch.from_taskgraphs([TaskGraph("x", [TaskNode(0, "GONLY_TYPE")])])
    pl = P.make_preset("homog2")
    pl.costs = P.CostTable()
    pl.costs.set("GONLY_TYPE", P.GPU, 1.0)
    r = abi.RegulatorCfg()
    r.slope_samples = 8
    with pytest.raises(po.OracleError, match="no worker can run task type GONLY_TYPE"):
        po.simulate(g, [pl], "dmda", reg=[r])
