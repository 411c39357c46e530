#!/usr/bin/env python
"""k_simulate time per C5 worker mix: G 4096-task layered DAGs all on one
platform (argv: G [mix ...]); prints one line per mix."""
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__file__) + "/..")
from paper_2404_03226_b200 import api  # noqa: E402
from paper_2404_03226_b200 import platform as P  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 1184
mixes = [tuple(int(x) for x in m.split("c")[0:1] + m.split("c")[1].rstrip("g").split()) for m in sys.argv[2:]] \
    or [(4, 1), (8, 2), (16, 2), (32, 4)]
ctx = api.Context(0)
seeds = np.arange(G, dtype=np.uint64)
db = ctx.generate_layered(4096, 10, 0.05, seeds)
for c, g in mixes:
    pl = [P.assemble(f"{c}c{g}g", c, g)]
    ctx.schedule(db, pl, "inspirit")
    ctx.set_timing(True)
    ms = []
    for _ in range(2):
        ctx.schedule(db, pl, "inspirit")
        ms.append((ctx.last_kernel_ms("k_simulate"), ctx.last_kernel_ms("k_simulate_rerun")))
    ctx.set_timing(False)
    print(f"{c}c{g}g G={G} k_simulate={ms[-1][0]:.2f} ms rerun={ms[-1][1]:.2f} ms shape={ctx.last_sim_shape()}",
          flush=True)
