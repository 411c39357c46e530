"""Diagnostic (not a bench value): where the C2 end-to-end step loses time
against the device-timed step.  Times, with CUDA events over K steps:
  A  schedule() on a resident batch, results to pinned host arrays (async)
  B  A + the next batch uploaded on the upload stream every step
  C  uploads alone (H2D + k_ingest + k_bytes_dict + k_sim_pack)
  D  schedule_device() on a resident batch (the bench's `value` step)"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2404_03226_b200 import api  # noqa: E402
from paper_2404_03226_b200 import platform as P  # noqa: E402

K = 10
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
dev = {"worker": torch.empty(T, dtype=torch.int32, device="cuda"),
       "start_ms": torch.empty(T, dtype=torch.float64, device="cuda"),
       "end_ms": torch.empty(T, dtype=torch.float64, device="cuda"),
       "makespan_ms": torch.empty(G, dtype=torch.float64, device="cuda")}
ptrs = {k: v.data_ptr() for k, v in dev.items()}
up = torch.cuda.Stream()
ctx.set_upload_stream(up.cuda_stream)
ctx.set_async_results(True)
db = ctx.upload(hb)
ctx.synchronize()


def timed(fn):
    for _ in range(2):
        fn(2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    fn(K)
    ctx.synchronize()
    torch.cuda.synchronize()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / K


def a(k):
    for _ in range(k):
        ctx.schedule(db, pl, "inspirit", want_attrs=False, out_arrays=pinned, want_states=False)


def b(k):
    nxt = ctx.upload(hb)
    for i in range(k):
        cur = nxt
        if i + 1 < k:
            nxt = ctx.upload(hb)
        ctx.schedule(cur, pl, "inspirit", want_attrs=False, out_arrays=pinned, want_states=False)
        cur.free()


def c(k):
    for _ in range(k):
        x = ctx.upload(hb)
        x.free()


def d(k):
    for _ in range(k):
        ctx.schedule_device(db, pl, "inspirit", ptrs)


for name, fn in (("A resident, host results", a), ("B + upload each step", b), ("C uploads only", c),
                 ("D resident, device results", d)):
    print(f"{name:30s} {timed(fn):8.3f} ms/step")
