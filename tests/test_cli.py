"""The tbsim command-line front end (paper_2404_03226_b200/tbsim, built from
csrc/cli/main.cpp): the reference's tests/test_cli.cpp cases, same commands,
outputs and exit codes (0 ok, 1 usage, 2 runtime failure).  Parsing, graph
generation and file errors run on the CPU; attrs / sim / bench need the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2404_03226_b200", "tbsim")
pytestmark = pytest.mark.skipif(not os.path.exists(BIN), reason="tbsim CLI not built")


def run(args, cwd=None):
    r = subprocess.run([BIN] + args.split(), capture_output=True, text=True, cwd=cwd, timeout=600)
    return r.returncode, r.stdout + r.stderr


def test_no_subcommand_is_a_usage_error():
    assert run("")[0] == 1


def test_help_lists_the_subcommands():
    rc, out = run("--help")
    assert rc == 0
    for s in ("gen", "attrs", "sim", "bench"):
        assert s in out


def test_gen_writes_a_loadable_graph_and_reports_its_shape(tmp_path):
    rc, out = run(f"--out-dir {tmp_path} gen cholesky --nblocks 4")
    assert rc == 0, out
    path = os.path.join(str(tmp_path), "cholesky_n4.dag")
    assert out == f"wrote {path}: 20 tasks, 30 edges\n"
    assert os.path.getsize(path) > 0


def test_gen_requires_its_size_argument(tmp_path):
    assert run(f"--out-dir {tmp_path} gen cholesky")[0] == 1
    assert run(f"--out-dir {tmp_path} gen cholesky --nblocks -3")[0] == 1


def test_gen_autogen_is_reproducible_per_seed(tmp_path):
    a, b, c = (os.path.join(str(tmp_path), f"{x}.dag") for x in "abc")
    common = " gen autogen --tasks 60 --layers 6 --out "
    assert run("--seed 11" + common + a)[0] == 0
    assert run("--seed 11" + common + b)[0] == 0
    assert run("--seed 12" + common + c)[0] == 0
    assert open(a).read() == open(b).read()
    assert open(a).read() != open(c).read()


def test_bad_arguments_exit_1_runtime_failures_exit_2(tmp_path):
    dag = os.path.join(str(tmp_path), "g.dag")
    assert run(f"gen cholesky --nblocks 2 --out {dag}")[0] == 0
    assert run(f"sim --dag {dag} --policy warp")[0] == 1
    assert run(f"--platform a --platform b sim --dag {dag}")[0] == 1
    rc, out = run(f"sim --dag {tmp_path}/absent.dag")
    assert rc == 2 and "error: cannot open" in out
    rc, out = run(f"--platform bogus sim --dag {dag}")
    assert rc == 2 and "error: " in out


def test_bench_rejects_unknown_apps_and_policies_at_parse_time():
    assert run("bench --app raytrace --sizes 2")[0] == 1
    assert run("bench --app lu --sizes 2 --policies warp")[0] == 1


@pytest.mark.gpu
def test_attrs_writes_a_csv_and_reports_the_calibration(tmp_path):
    dag = os.path.join(str(tmp_path), "g.dag")
    assert run(f"gen lu --nblocks 3 --out {dag}")[0] == 0
    rc, out = run(f"--out-dir {tmp_path} attrs --dag {dag}")
    assert rc == 0, out
    assert f"wrote {os.path.join(str(tmp_path), 'attributes.csv')}: 14 rows\n" in out
    assert "unit_time_ms: " in out and "11 evaluations)" in out
    csv = open(os.path.join(str(tmp_path), "attributes.csv")).read()
    assert csv.startswith("task_id,type,layer,ability,efficiency,static_priority\n")


@pytest.mark.gpu
def test_sim_prints_the_makespan(tmp_path):
    dag = os.path.join(str(tmp_path), "g.dag")
    assert run(f"gen cholesky --nblocks 4 --out {dag}")[0] == 0
    rc, out = run(f"sim --dag {dag} --policy dmda")
    assert rc == 0, out
    for s in ("dag: cholesky_n4 (20 tasks)\n", "platform: 26cpu_2gpu\n", "policy: dmda\n", "makespan_ms: "):
        assert s in out
    assert "regulator:" not in out


@pytest.mark.gpu
def test_sim_with_the_adaptive_policy_reports_regulator_and_pop_counts(tmp_path):
    dag = os.path.join(str(tmp_path), "g.dag")
    assert run(f"gen cholesky --nblocks 8 --out {dag}")[0] == 0
    rc, out = run(f"sim --dag {dag} --policy inspirit")
    assert rc == 0, out
    assert "regulator: task_window=7 s_inc=28 k_inc=28 s_dec=7 c=4 dec_step=7 slope_samples=8\n" in out
    assert "pops_by_mode: ability=" in out
    # README golden (proj/README.md:81-88): inspirit on Cholesky 8 / 26cpu_2gpu
    assert "makespan_ms: 54.22\n" in out
    rc, out = run(f"sim --dag {dag} --policy inspirit --s-inc 3 --k-inc 0.5")
    assert rc == 0 and "s_inc=3 k_inc=0.5" in out


@pytest.mark.gpu
def test_sim_trace_writes_the_three_trace_csvs(tmp_path):
    dag = os.path.join(str(tmp_path), "g.dag")
    assert run(f"gen heat --nblocks 3 --timesteps 4 --out {dag}")[0] == 0
    rc, out = run(f"--out-dir {tmp_path} sim --dag {dag} --policy inspirit --trace --window 2.5")
    assert rc == 0, out
    assert f"trace: {tmp_path}" in out and "window 2.5 ms)" in out
    rd = lambda f: open(os.path.join(str(tmp_path), f)).read()
    assert rd("gantt.csv").startswith("task_id,type,worker,start_ms,end_ms\n")
    assert rd("nready_time.csv").startswith("time_ms,nready\n")
    assert rd("push_pop.csv").startswith("window_start_ms,pushes,pops\n")


@pytest.mark.gpu
def test_bench_writes_its_csv_and_reports_failed_cells(tmp_path):
    rc, out = run(f"--out-dir {tmp_path} --jobs 1 bench --app lu --sizes 3 4 --policies fifo dmda")
    assert rc == 0, out
    assert f"wrote {os.path.join(str(tmp_path), 'bench.csv')}: 4 rows\n" in out
    assert "cells failed" not in out
    csv = open(os.path.join(str(tmp_path), "bench.csv")).read()
    assert csv.startswith("app,size,platform,policy,makespan_ms,speedup_vs_baseline,status\n")
    rc, out = run(f"--out-dir {tmp_path} --platform 26cpu_2gpu --platform nope --jobs 1 bench --app lu --sizes 3 "
                  f"--policies dmda --out {tmp_path}/b2.csv")
    assert rc == 0 and "1 cells failed; see status column" in out
