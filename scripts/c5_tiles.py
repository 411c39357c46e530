"""C5-shaped attribute pass per sweep tile width (diagnostic): 2048 device-
generated 4096-task layered DAGs, k_sweep time for each forced width, outputs
required identical to the automatic choice."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_03226_b200 import abi, api  # noqa: E402
from paper_2404_03226_b200 import platform as P  # noqa: E402

ctx = api.Context(0)
db = ctx.generate_layered(4096, 10, 0.05, np.arange(2048, dtype=np.uint64))
costs = P.default_cost_table()
base = None
for tile in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,32,64").split(",")]:
    ctx.set_sweep_tile(tile)
    ctx.set_timing(True)
    for _ in range(2):
        out = ctx.attributes(db, costs, abi.ATTR_ALL)
    print(json.dumps({"tile": tile, "k_sweep": round(ctx.last_kernel_ms("k_sweep"), 3),
                      "k_structure": round(ctx.last_kernel_ms("k_structure"), 3)}), flush=True)
    key = {k: np.asarray(out[k]).copy() for k in ("ability", "efficiency", "static_priority")}
    if base is None:
        base = key
    else:
        for k in key:
            assert np.array_equal(key[k], base[k]), f"tile {tile}: {k} differs"
