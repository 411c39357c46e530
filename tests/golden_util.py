"""Loading of the committed reference fixtures (tests/golden/*.npz)."""
import glob
import os

import numpy as np

from paper_2404_03226_b200 import abi
from paper_2404_03226_b200 import platform as P
from paper_2404_03226_b200.batch import GraphBatch

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

PLATFORMS = {
    "homog2": lambda: P.make_preset("homog2"),
    "26cpu_2gpu": lambda: P.make_preset("26cpu_2gpu"),
    "2gpu": lambda: P.make_preset("2gpu"),
    "4c1g": lambda: P.assemble("4c1g", 4, 1),
    "8c2g": lambda: P.assemble("8c2g", 8, 2),
    "32c4g": lambda: P.assemble("32c4g", 32, 4),
}

SIM_KEYS = ("worker", "start_ms", "end_ms", "makespan_ms", "pop_mode_counts", "push_time", "push_task",
            "pop_time", "pop_task", "pop_worker", "sample_time", "sample_nready")


def names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(HERE, "*.npz")))


class Fixture:
    def __init__(self, name):
        self.name = name
        z = np.load(os.path.join(HERE, name + ".npz"))
        self.z = z
        tn = [str(x) for x in z["type_names"]]
        self.batch = GraphBatch(z["task_base"], z["edge_base"], z["handle_base"], z["in_base"], z["out_base"],
                                z["dep_off"], z["dep"], z["in_off"], z["in_"], z["out_off"], z["out"], z["type"],
                                z["handle_bytes"], tn, z["task_id"])
        self.costs = P.CostTable()
        for i, n in enumerate(tn):
            if z["cost_cpu"][i] > 0:
                self.costs.set(n, P.CPU, float(z["cost_cpu"][i]))
            if z["cost_gpu"][i] > 0:
                self.costs.set(n, P.GPU, float(z["cost_gpu"][i]))
        self.prio = int(z["prio_kind"])
        self.platform_names = [str(x) for x in z["platforms"]] if "platforms" in z else []

    def platform(self, name):
        pl = PLATFORMS[name]()
        pl.costs = self.costs
        return pl

    def attrs(self):
        return {"ability": self.z["attr_ability"], "efficiency": self.z["attr_efficiency"],
                "static_priority": self.z["attr_static_priority"]}

    def sim(self, pname, policy):
        return {k: self.z[f"sim_{pname}_{policy}_{k}"] for k in SIM_KEYS} | {
            "reg": self.z[f"sim_{pname}_{policy}_reg"], "reg_cur_k": self.z[f"sim_{pname}_{policy}_reg_cur_k"]}

    def reg_cfgs(self, pname, oracle_mod):
        pl = self.platform(pname)
        return [oracle_mod.default_regulator_config(self.batch, g, pl) for g in range(self.batch.n_graphs)]


def reg_rows(states, G):
    return np.array([[s.mode, s.phase, s.peak, s.prev_nready, s.last_trigger_nready, s.s_dec_count]
                     for s in states[:G]], np.int64)
