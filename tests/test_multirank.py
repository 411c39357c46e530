"""CPU, world_size 2 over gloo: the multi-GPU host path (seed sharding +
final all-gather of makespans/assignments) reproduces a single-process run."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2404_03226_b200 import shard

PER_RANK = 6


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _schedule_oracle(seeds):
    from oracle import pyoracle as po
    from paper_2404_03226_b200 import abi
    from paper_2404_03226_b200 import platform as P
    from paper_2404_03226_b200.batch import GraphBatch
    b = GraphBatch.concat([po.gen_layered(120, 6, 0.1, int(s)) for s in seeds])
    pl = P.assemble("8c2g", 8, 2)
    a = po.attributes(b, P.default_cost_table(), abi.ATTR_ALL)
    reg = [po.default_regulator_config(b, g, pl) for g in range(b.n_graphs)]
    r = po.simulate(b, [pl], "inspirit", reg=reg, attrs=a, record=False)
    return r["makespan_ms"], r["worker"]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seeds = shard.shard_seeds(rank, world, PER_RANK)
    ms, w = _schedule_oracle(seeds)
    all_ms, all_w = shard.all_gather_results(dist, torch.from_numpy(ms), torch.from_numpy(w))
    if rank == 0:
        q.put((all_ms.numpy(), all_w.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gather_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    all_ms, all_w = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ms, w = _schedule_oracle(np.arange(2 * PER_RANK))
    np.testing.assert_array_equal(all_ms, ms)
    np.testing.assert_array_equal(all_w, w)


def test_split_range_covers_everything():
    for n in (0, 1, 7, 4096, 65536):
        for world in (1, 2, 3, 8):
            parts = [shard.split_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
