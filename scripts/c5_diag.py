"""Diagnostic (not a bench value): the C5 end-to-end step's parts -- device
generation alone, scheduling a resident batch, and both -- with results in
pinned host arrays and asynchronous calls, as bench.py's C5 e2e."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2404_03226_b200 import api, platform as P
ctx = api.Context(0); stream = torch.cuda.current_stream(); ctx.set_stream(stream.cuda_stream)
G, n = 8192, 4096
seeds = np.arange(G, dtype=np.uint64)
mixes = [(4, 1), (8, 2), (16, 2), (32, 4)]
pls = [P.assemble(f"{c}c{g}g", c, g) for c, g in mixes]
pof = (seeds % 4).astype(np.int32)
def t(fn, k=3):
    fn(); fn(); ctx.synchronize(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k): fn()
    ctx.synchronize(); torch.cuda.synchronize(); e1.record(stream); e1.synchronize()
    return e0.elapsed_time(e1) / k
def gen():
    db = ctx.generate_layered(n, 10, 0.05, seeds); db.free()
res = ctx.generate_layered(n, 10, 0.05, seeds)
T = G * n
pinned = {"worker": torch.empty(T, dtype=torch.int32, pin_memory=True).numpy(),
          "start_ms": torch.empty(T, dtype=torch.float64, pin_memory=True).numpy(),
          "end_ms": torch.empty(T, dtype=torch.float64, pin_memory=True).numpy(),
          "makespan_ms": torch.empty(G, dtype=torch.float64, pin_memory=True).numpy(),
          "completed": torch.empty(G, dtype=torch.int64, pin_memory=True).numpy()}
ctx.set_async_results(True)
def sched():
    ctx.schedule(res, pls, "inspirit", platform_of=pof, want_attrs=False, want_states=False, out_arrays=pinned)
def both():
    db = ctx.generate_layered(n, 10, 0.05, seeds)
    ctx.schedule(db, pls, "inspirit", platform_of=pof, want_attrs=False, want_states=False, out_arrays=pinned)
    db.free()
print("gen only", t(gen), "sched resident", t(sched), "gen+sched", t(both))
names = ("k_structure", "k_sweep", "k_finalize", "k_sim_keys", "k_simulate", "k_simulate_rerun", "k_sim_scatter",
         "k_xfer_table", "k_tile_plan")
for mode in ("async host outputs", "sync device outputs"):
    ctx.set_timing(True)
    if mode.startswith("async"):
        sched()
        ctx.synchronize()
    else:
        ctx.set_async_results(False)
        dev = {k: torch.empty(v.shape, dtype=torch.from_numpy(v).dtype, device="cuda") for k, v in pinned.items()
               if k != "completed"}
        ctx.schedule_device(res, pls, "inspirit", {k: v.data_ptr() for k, v in dev.items()}, platform_of=pof)
    print(mode, {k: round(ctx.last_kernel_ms(k), 2) for k in names})
    ctx.set_timing(False)
