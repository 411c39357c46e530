"""C4 attribute-pass experiment: kernel times of the 1M-task DAG's attribute
pipeline under sweep-tile / structure-grid variants, with every variant's
outputs required identical to the first one's (diagnostic, run on the box).

    python scripts/c4_exp.py [--tiles 0,8,16] [--reps 3]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_03226_b200 import abi, api  # noqa: E402
from paper_2404_03226_b200 import platform as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tiles", default="0")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    ctx = api.Context(0)
    db = ctx.generate_layered(1 << 20, 1024, 1.0 / 256, np.array([1], np.uint64))
    costs = P.default_cost_table()
    names = ["k_structure", "k_closure", "k_tile_plan", "k_sweep", "k_finalize", "k_structure_out"]
    base = None
    for s in [int(x) for x in a.tiles.split(",")]:
        ctx.set_sweep_tile(s)
        ctx.set_timing(True)
        for r in range(a.reps):
            out = ctx.attributes(db, costs, abi.ATTR_ALL)
            km = {k: round(ctx.last_kernel_ms(k), 3) for k in names}
            print(json.dumps({"tile": s, "rep": r, "kernel_ms": km, "total": round(sum(km.values()), 3)}), flush=True)
        key = {k: np.asarray(out[k]).copy() for k in ("ability", "efficiency", "static_priority", "unit_time_ms")}
        if base is None:
            base = key
        else:
            for k in key:
                assert np.array_equal(key[k], base[k]), f"tile {s}: {k} differs"
            print(json.dumps({"tile": s, "identical_to_first": True}), flush=True)


if __name__ == "__main__":
    main()
