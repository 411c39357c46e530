"""TEST INFRASTRUCTURE: C4-scale parity of the attribute path against the
reference itself (oracle/_ref/libtbsim_ref_c4.so, see oracle/ref_c4.cpp).

C4 is one 1M-task DAG (generate_layered_dag(1048576, 1024, 1/256, 1)).  The
reference's ability, upward rank, depth and layers run in full (~40 s on 8
host cores) and must equal the device's bit for bit.  A full efficiency
evaluation takes the reference ~10^4 core-seconds and calibration needs 11
of them, so efficiency is pinned per window on sampled sources with the
reference's own per-source kernel efficiency_of (src/attributes.cpp:110-137),
and the calibration is pinned by re-scoring the device's 11 full per-window
efficiency vectors with a numpy restatement of score_of
(src/attributes.cpp:200-217).  Used by tests/test_c4_parity.py and by
bench.py's C4 cpu_baseline leg; never by the product.
"""
from __future__ import annotations

import os

import numpy as np

from paper_2404_03226_b200 import abi

from . import pyref

N_WINDOWS = 11


def class_scores(eff_by_window: np.ndarray, layer: np.ndarray, type_: np.ndarray) -> np.ndarray:
    """score_of (src/attributes.cpp:200-217) for each row of eff_by_window:
    distinct reduced fractions sum/cnt over (layer, type) classes."""
    key = layer.astype(np.int64) * 1024 + type_.astype(np.int64)
    _, cls = np.unique(key, return_inverse=True)
    n_cls = int(cls.max()) + 1 if len(cls) else 0
    cnt = np.bincount(cls, minlength=n_cls).astype(np.int64)
    out = np.zeros(len(eff_by_window), np.int64)
    for k, eff in enumerate(eff_by_window):
        s = np.zeros(n_cls, np.int64)
        np.add.at(s, cls, eff.astype(np.int64))
        d = np.gcd(np.where(s == 0, cnt, s), cnt)
        pairs = np.stack([s // d, cnt // d], axis=1)
        out[k] = len(np.unique(pairs, axis=0))
    return out


def gpu_window_efficiency(ctx, db, costs, w0: float) -> np.ndarray:
    """Device efficiency at each calibration window W_k = ldexp(w0, k-4)."""
    return np.stack([ctx.attributes(db, costs, abi.ATTR_EFFICIENCY, unit_time=[np.ldexp(w0, k - 4)])["efficiency"]
                     for k in range(N_WINDOWS)])


def check(ctx, db, gb, costs, threads: int = 0, n_sample: int = 64, seed: int = 0) -> dict:
    """Compare the device's attributes of graph 0 of `db` (host copy `gb`)
    with the reference.  Returns a report; `report["mismatch"]` lists every
    failed comparison (empty when everything is bit-exact)."""
    threads = threads or os.cpu_count() or 1
    ref = pyref.C4Ref(gb, costs)
    rs = ref.structure(threads=threads)
    dev_all = ctx.attributes(db, costs, abi.ATTR_ALL)
    dev = {"ability": dev_all["ability"], "static_priority": dev_all["static_priority"],
           "depth": ctx.attributes(db, costs, abi.ATTR_DEPTH)["depth"],
           "layer": ctx.attributes(db, costs, abi.ATTR_LAYERS)["layer"]}
    cal = ctx.attributes(db, costs, abi.ATTR_CALIBRATE)
    mismatch = [k for k in dev if not np.array_equal(np.asarray(dev[k]), np.asarray(rs[k]))]
    if float(cal["w0_ms"][0]) != rs["w0_ms"]:
        mismatch.append("w0_ms")
    w0 = rs["w0_ms"]
    windows = [float(np.ldexp(w0, k - 4)) for k in range(N_WINDOWS)]
    eff_k = gpu_window_efficiency(ctx, db, costs, w0)
    n = gb.sizes(0)
    rng = np.random.default_rng(seed)
    src = np.sort(rng.choice(n, size=min(n_sample, n), replace=False))
    ref_eff, setup_s, calls_s = ref.efficiency_sample(src, windows, threads=threads)
    if not np.array_equal(eff_k[:, src].T, ref_eff):
        mismatch.append("efficiency_sample")
    # calibration: re-score the device's per-window vectors (strict >: the
    # first maximum wins, attributes.cpp:225)
    scores = class_scores(eff_k, dev["layer"], gb.type[gb.task_base[0]:gb.task_base[1]])
    best = int(np.argmax(scores))
    if (int(cal["best_score"][0]), int(cal["w0_score"][0]), int(cal["evaluations"][0])) != \
            (int(scores[best]), int(scores[4]), N_WINDOWS):
        mismatch.append("calibration_scores")
    if float(cal["unit_time_ms"][0]) != windows[best] or float(dev_all["unit_time_ms"][0]) != windows[best]:
        mismatch.append("unit_time_ms")
    if not np.array_equal(dev_all["efficiency"], eff_k[best]):
        mismatch.append("efficiency_at_calibrated_window")
    # reference compute_attributes time: ability + layers (calibration
    # classes) + rank in full; 12 efficiency evaluations (11 calibration + 1
    # final) extrapolated from the sampled efficiency_of calls
    eval_s = calls_s * n / (len(src) * N_WINDOWS)
    total_s = rs["seconds"]["ability"] + rs["seconds"]["layers"] + rs["seconds"]["rank"] + 12 * (eval_s + setup_s)
    return {"mismatch": mismatch, "n_tasks": n, "threads": threads, "sample_sources": int(len(src)),
            "windows": windows, "scores": scores.tolist(), "best_window": best,
            "ref_seconds": dict(rs["seconds"], efficiency_setup=setup_s, efficiency_sample_calls=calls_s,
                                efficiency_eval_extrapolated=eval_s),
            "ref_compute_attributes_s_extrapolated": total_s,
            "checked": ["ability", "static_priority (UpwardRank)", "depth", "layer", "w0_ms",
                        f"efficiency at all 11 windows on {len(src)} sampled sources (reference efficiency_of)",
                        "calibration scores/unit time from the device's 11 full per-window vectors",
                        "final efficiency == window vector at the calibrated W"]}
