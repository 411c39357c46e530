"""GPU, two processes: the real bench.py sharded path (seed shards per rank,
schedule on the device, the final all-gather of makespans and assignments)
equals one process scheduling all the seeds.  Both ranks share cuda:0
(TBSIM_ONE_GPU=1), so the collective runs over gloo instead of NCCL
(TBSIM_DIST_BACKEND=gloo); the product path per rank is the same."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_2404_03226_b200 import api
from paper_2404_03226_b200 import platform as P

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("workload", ["c2", "c5"])
def test_two_rank_bench_gathers_single_process_results(ctx, tmp_path, workload):
    per_rank = 48
    dump = tmp_path / "gathered.npz"
    env = dict(os.environ, TBSIM_ONE_GPU="1", TBSIM_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", "bench.py", "--gpus", "2",
           "--workload", workload, "--n-dags", str(per_rank), "--steps", "2", "--warmup", "3", "--no-c4",
           "--no-cpu-baseline", "--dump-gathered", str(dump)]
    r = subprocess.run(cmd, cwd=ROOT, env=env, timeout=900, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    z = np.load(dump)
    seeds = np.arange(2 * per_rank)
    if workload == "c2":
        hb = api.HostBatch().add_layered(1000, 10, 0.05, seeds)
        want = ctx.schedule(ctx.upload(hb), [P.assemble("8c2g", 8, 2)], "inspirit")
    else:
        pls = [P.assemble(f"{c}c{g}g", c, g) for c, g in ((4, 1), (8, 2), (16, 2), (32, 4))]
        want = ctx.schedule(ctx.generate_layered(4096, 10, 0.05, seeds), pls, "inspirit",
                            platform_of=(seeds % 4).astype(np.int32))
    half = int(want["makespan_ms"].shape[0]) // 2
    t_half = int(np.sum(want["worker"].shape)) // 2
    for prefix in ("value_", "e2e_"):
        for k in ("makespan_ms", "worker", "start_ms", "end_ms"):
            np.testing.assert_array_equal(z[prefix + k], want[k], err_msg=prefix + k)
    np.testing.assert_array_equal(z["e2e_own_makespan"], want["makespan_ms"][:half])
    np.testing.assert_array_equal(z["e2e_own_worker"], want["worker"][:t_half])
