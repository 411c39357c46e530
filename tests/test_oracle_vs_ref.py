"""CPU: the restatement against the compiled reference itself (oracle/_ref)
on many random inputs, when the reference library is present."""
import numpy as np
import pytest

from oracle import pyoracle as po
from oracle import pyref
from paper_2404_03226_b200 import abi
from paper_2404_03226_b200 import platform as P
from paper_2404_03226_b200.batch import GraphBatch

pytestmark = pytest.mark.skipif(not pyref.available(), reason="oracle/_ref not built")
MIXED = ["LAYERK0", "LAYERK1", "LAYERK2", "LAYERK3", "UNIT"]


def _graphs():
    gs = [pyref.gen_random(300 + i, 8 + (i * 7) % 53, 0.06 + 0.02 * (i % 4), MIXED, i % 2 == 0) for i in range(30)]
    gs += [pyref.gen_layered(60 + 13 * i, 2 + i % 9, 0.02 + 0.02 * (i % 5), 1000 + i) for i in range(20)]
    return GraphBatch.concat(gs)


def test_attributes_random_graphs():
    b = _graphs()
    costs = P.default_cost_table()
    keys = {abi.ATTR_ALL: ("ability", "efficiency", "static_priority", "unit_time_ms"),
            abi.ATTR_CALIBRATE: ("unit_time_ms", "w0_ms", "best_score", "w0_score", "evaluations"),
            abi.ATTR_DEPTH: ("depth",), abi.ATTR_LAYERS: ("layer",), abi.ATTR_RANK: ("static_priority",)}
    for req, ks in keys.items():
        r, o = pyref.attributes(b, costs, req), po.attributes(b, costs, req)
        for k in ks:
            np.testing.assert_array_equal(r[k], o[k], err_msg=f"{req}:{k}")


@pytest.mark.parametrize("preset", ["26cpu_2gpu", "26cpu_1gpu", "2gpu", "homog2"])
def test_simulation_random_graphs(preset):
    b = _graphs()
    costs = P.default_cost_table()
    a = pyref.attributes(b, costs, abi.ATTR_ALL)
    pl = P.make_preset(preset)
    reg = [po.default_regulator_config(b, g, pl) for g in range(b.n_graphs)]
    for pol in abi.POLICIES:
        r = pyref.simulate(b, [pl], pol, attrs=a)
        o = po.simulate(b, [pl], pol, reg=reg, attrs=a)
        for k in r:
            if k != "reg_state":
                np.testing.assert_array_equal(r[k], o[k], err_msg=f"{preset}/{pol}/{k}")
