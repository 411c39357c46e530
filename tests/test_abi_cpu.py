"""CPU: the C-ABI library loads, exports every symbol include/tbsim_b200.h
declares, its host generators reproduce the reference's graphs, and it fails
loudly (no CPU fallback) when no GPU is present."""
import os
import re
import subprocess

import numpy as np
import pytest

from golden_util import Fixture
from oracle import pyoracle as po
from paper_2404_03226_b200 import abi, api
from paper_2404_03226_b200 import platform as P
from paper_2404_03226_b200.lib import EXPORTS, LIB_PATH, load

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_and_exports_agree():
    hdr = open(os.path.join(ROOT, "include", "tbsim_b200.h")).read()
    declared = set(re.findall(r"\b(tbsim_[a-z_0-9]+)\s*\(", hdr))
    assert declared == set(EXPORTS), declared ^ set(EXPORTS)
    L = load()
    for s in EXPORTS:
        assert getattr(L, s) is not None
    syms = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True, text=True).stdout
    for s in EXPORTS:
        assert re.search(rf"\bT {s}\b", syms), s


def test_type_table_and_default_costs_match_python_twin():
    L = load()
    assert L.tbsim_type_count() == len(P.TYPE_NAMES)
    assert [L.tbsim_type_name(i).decode() for i in range(len(P.TYPE_NAMES))] == P.TYPE_NAMES
    import ctypes as C
    cpu = (C.c_double * len(P.TYPE_NAMES))()
    gpu = (C.c_double * len(P.TYPE_NAMES))()
    assert L.tbsim_default_costs(cpu, gpu) == 0
    pc, pg = P.default_cost_table(with_qr=True).arrays(P.TYPE_NAMES)
    assert list(cpu) == pc.tolist() and list(gpu) == pg.tolist()


def _same_graph(a, b):
    for k in ("dep_off", "dep", "in_off", "in_", "out_off", "out", "type", "handle_bytes"):
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k), err_msg=k)


def test_host_generators_reproduce_reference_fixtures():
    hb = api.HostBatch()
    for n in (4, 6, 8, 10, 12):
        hb.add_cholesky(n, 960 * 960 * 4)
    for n in (3, 6, 10):
        hb.add_lu(n, 160 * 160 * 4)
    hb.add_layered(1000, 10, 0.05, [0, 1])
    hb.add_layered(30, 3, 0.03, [0])
    v = hb.view()
    chol, lu, lay = Fixture("cholesky").batch, Fixture("lu").batch, Fixture("layered_1k").batch
    for i in range(5):
        _same_graph(v._one(i), chol._one(i))
    for i in range(3):
        _same_graph(v._one(5 + i), lu._one(i))
    for i in range(2):
        _same_graph(v._one(8 + i), lay._one(i))
    _same_graph(v._one(10), Fixture("layered_small").batch._one(0))


def test_host_layered_generator_matches_oracle_many_seeds():
    seeds = list(range(20, 60))
    v = api.HostBatch().add_layered(400, 8, 0.07, seeds, threads=4).view()
    for i, s in enumerate(seeds):
        _same_graph(v._one(i), po.gen_layered(400, 8, 0.07, s))


def test_generator_argument_errors():
    with pytest.raises(api.TbsimInvalidArgument, match="autogen: n_tasks must be >= n_layers"):
        api.HostBatch().add_layered(3, 5, 0.1, [0])
    with pytest.raises(api.TbsimInvalidArgument, match="cholesky: nblocks must be >= 1"):
        api.HostBatch().add_cholesky(0, 4)
    with pytest.raises(api.TbsimInvalidArgument, match="lu: block_bytes must be > 0"):
        api.HostBatch().add_lu(3, 0)


def test_qr_generator_structure():
    # GEQRT/UNMQR/TSQRT/TSMQR counts: sum_{m=1..n} m^2 tasks; acyclic
    for n in (1, 3, 6, 40):
        v = api.HostBatch().add_qr(n, 4096).view()
        assert v.n_tasks == sum(m * m for m in range(1, n + 1))
        counts = np.bincount(v.type, minlength=len(P.TYPE_NAMES))
        ids = {k: P.TYPE_ID[k] for k in ("GEQRT", "UNMQR", "TSQRT", "TSMQR")}
        assert counts[ids["GEQRT"]] == n
        assert counts[ids["UNMQR"]] == n * (n - 1) // 2 == counts[ids["TSQRT"]]
        assert counts[ids["TSMQR"]] == sum(m * m for m in range(n))
        lay = po.attributes(v, P.default_cost_table(with_qr=True), abi.ATTR_LAYERS)["layer"]
        assert lay.max() >= 0  # no cycle error


def test_default_regulator_config_matches_oracle():
    b = po.gen_cholesky(8, 64)
    want = po.default_regulator_config(b, 0, P.make_preset("26cpu_2gpu"))
    got = api.default_regulator_config(28, 1.0)
    for k in ("task_window", "s_inc", "k_inc", "s_dec", "c", "dec_step", "slope_samples"):
        assert getattr(got, k) == getattr(want, k), k


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(api.TbsimError) as e:
        api.Context(0)
    assert e.value.status == abi.TBSIM_E_CUDA


def test_csr_cache_round_trip_and_errors(tmp_path):
    """Binary CSR cache (tbsim_hostbatch_save / _load):
    every section and the type-name table survive; a malformed file raises
    invalid_argument."""
    from paper_2404_03226_b200 import api
    hb = api.HostBatch().add_layered(300, 7, 0.1, [1, 2, 3]).add_cholesky(5, 1000).add_qr(4, 640)
    p = str(tmp_path / "b.csr")
    hb.save(p)
    a, b = hb.view(), api.HostBatch.load(p).view()
    for k in ("task_base", "edge_base", "handle_base", "in_base", "out_base", "dep_off", "dep", "in_off", "in_",
              "out_off", "out", "type", "handle_bytes"):
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k), err_msg=k)
    assert b.type_names == a.type_names
    (tmp_path / "bad.csr").write_bytes(b"TBSIMCSR" + b"\x02\x00\x00\x00" + bytes(64))
    with pytest.raises(api.TbsimInvalidArgument):
        api.HostBatch.load(str(tmp_path / "bad.csr"))
    with pytest.raises(api.TbsimError):
        api.HostBatch.load(str(tmp_path / "absent.csr"))


def test_csr_cache_keeps_task_ids_and_custom_type_names(tmp_path):
    """A batch built from TaskGraphs with arbitrary ids and type names (the
    NDJSON case) round-trips through the binary cache with its id and name
    tables."""
    from paper_2404_03226_b200 import api
    from paper_2404_03226_b200.batch import GraphBatch, TaskGraph, TaskNode
    g = TaskGraph("x", [TaskNode(17, "ALPHA"), TaskNode(5, "BETA", [17], [100], [101]),
                        TaskNode(9, "ALPHA", [17, 5], [101], [])], [(100, 64), (101, 4096)])
    gb = GraphBatch.from_taskgraphs([g])
    hb = api.HostBatch().add_batch(gb)
    p = str(tmp_path / "x.csr")
    hb.save(p)
    back = api.HostBatch.load(p).view()
    np.testing.assert_array_equal(back.task_id, [17, 5, 9])
    np.testing.assert_array_equal(back.dep, gb.dep)
    np.testing.assert_array_equal(back.handle_bytes, [64, 4096])
    assert [back.type_names[t] for t in back.type] == [gb.type_names[t] for t in gb.type]
