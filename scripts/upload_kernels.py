#!/usr/bin/env python
"""Times the per-batch upload kernels (k_ingest_pack, or k_ingest + k_sim_pack
with TBSIM_SPLIT_INGEST=1) on C2's host
batch and on C5-shaped DAGs (diagnostic)."""
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__file__) + "/..")
from paper_2404_03226_b200 import api  # noqa: E402
from paper_2404_03226_b200 import platform as P  # noqa: E402

ctx = api.Context(0)
for n, G in ((1000, 4096), (4096, 2048)):
    hb = api.HostBatch().add_layered(n, 10, 0.05, np.arange(G, dtype=np.uint64))
    pl = [P.assemble("8c2g", 8, 2)]
    ctx.upload(hb)
    ctx.set_timing(True)
    for _ in range(2):  # timings are collected by the next call
        db = ctx.upload(hb)
        ctx.schedule(db, pl, "fifo", want_attrs=False)
    ctx.set_timing(False)
    print(f"layered({n}) x {G}: k_ingest {ctx.last_kernel_ms('k_ingest'):.3f} ms, "
          f"k_sim_pack {ctx.last_kernel_ms('k_sim_pack'):.3f} ms, "
          f"k_ingest_pack {ctx.last_kernel_ms('k_ingest_pack'):.3f} ms, "
          f"k_bytes_dict {ctx.last_kernel_ms('k_bytes_dict'):.3f} ms", flush=True)
