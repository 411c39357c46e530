"""Host-side timeline of the C2 end-to-end loop (diagnostic): where the
non-kernel time per step goes."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2404_03226_b200 import api  # noqa: E402
from paper_2404_03226_b200 import platform as P  # noqa: E402

ctx = api.Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
hb = api.HostBatch().add_layered(1000, 10, 0.05, np.arange(4096, dtype=np.uint64))
T, G = hb.view().n_tasks, hb.view().n_graphs
pl = [P.assemble("8c2g", 8, 2)]
pinned = {"worker": torch.empty(T, dtype=torch.int32, pin_memory=True).numpy(),
          "start_ms": torch.empty(T, dtype=torch.float64, pin_memory=True).numpy(),
          "end_ms": torch.empty(T, dtype=torch.float64, pin_memory=True).numpy(),
          "makespan_ms": torch.empty(G, dtype=torch.float64, pin_memory=True).numpy(),
          "completed": torch.empty(G, dtype=torch.int64, pin_memory=True).numpy()}
up = torch.cuda.Stream()
ctx.set_upload_stream(up.cuda_stream)
ctx.set_async_results(True)
for rep in range(2):
    nxt = ctx.upload(hb)
    tu, ts, tf = [], [], []
    t_start = time.perf_counter()
    for k in range(10):
        cur = nxt
        a = time.perf_counter()
        if k + 1 < 10:
            nxt = ctx.upload(hb)
        b = time.perf_counter()
        ctx.schedule(cur, pl, "inspirit", want_attrs=False, out_arrays=pinned, want_states=False)
        c = time.perf_counter()
        cur.free()
        d = time.perf_counter()
        tu.append(b - a); ts.append(c - b); tf.append(d - c)
    ctx.synchronize()
    total = time.perf_counter() - t_start
print(f"per step: total {1e3 * total / 10:.2f} ms, upload call {1e3 * np.mean(tu):.3f}, schedule call {1e3 * np.mean(ts):.3f}, free {1e3 * np.mean(tf):.3f}")
