#!/usr/bin/env python3
"""Generate the committed golden fixtures under tests/golden/ -- TEST
INFRASTRUCTURE ONLY.

The reference stores no golden files (its pins are in-code KATs over seeded
generators), so the fixtures are produced here by running the
REFERENCE ITSELF, compiled in place from /root/reference/proj/src by
oracle/Makefile (oracle/_ref/libalsncg_ref.so; its als.cpp is the restated
Eigen-free column solve).  Inputs come from the
oracle-side workload generator (oracle/alsncg_oracle.c orc_synth_generate),
which tests/test_golden.py pins bitwise to the product's generator.

  python tests/golden/make_golden.py c0         # seconds
  python tests/golden/make_golden.py c1_ttt     # ~1 h on 8 cores (ALS-NCG to 1e-6)
  python tests/golden/make_golden.py gen        # generator / CSR digests

Outputs (JSON, small): c0_trace.json, c1_ttt_trace.json, generator_digests.json.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import CONFIGS, Oracle, generate, make_config, ref_available  # noqa: E402


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def oracle():
    if not ref_available():
        raise SystemExit("oracle/_ref not built: make -C oracle ref")
    return Oracle("ref")


def trace_json(recs):
    return [dict(iter=t["iter"], loss=t["loss"], grad_norm=t["grad_norm"],
                 backtracks=t["backtracks"], restarted=bool(t["restarted"]),
                 shuffled_columns=t["shuffled_columns"]) for t in recs]


def c0():
    c = CONFIGS[0]
    R = generate(0)
    orc = oracle()
    out = {"what": "BASELINE config 0 through the compiled reference (oracle/_ref)",
           "config": {k: c[k] for k in ("n_u", "n_m", "nnz", "n_f", "lam", "seed")}}
    for algo, n_iter in (("ncg", 20), ("als", 20)):
        cfg = make_config(lambda_=c["lam"], n_f=c["n_f"], max_iters=n_iter, tol=0.0, seed=0,
                          n_blocks=4, n_workers=4)
        x, recs, info = (orc.ncg_solve if algo == "ncg" else orc.als_solve)(R, cfg)
        out[algo] = {"solver": {"max_iters": n_iter, "tol": 0.0, "seed": 0, "n_blocks": 4},
                     "trace": trace_json(recs), "result": info,
                     "model_sha256": sha(x), "model_head": x[:16].tolist(),
                     "model_norm": float(np.linalg.norm(x))}
    # kernel-level goldens at x0 (seed 0) and a seeded direction
    x0 = orc.random_init(c["n_f"], c["n_u"], c["n_m"], 0)
    rng = np.random.default_rng(7)
    p = rng.standard_normal(x0.size) * 0.1
    g = orc.gradient(R, c["n_f"], x0, c["lam"])
    users, fb = orc.half_sweep(R, True, c["n_f"], x0[c["n_f"] * c["n_u"]:], c["lam"])
    out["x0"] = {"seed": 0, "sha256": sha(x0), "loss": orc.loss(R, c["n_f"], x0, c["lam"]),
                 "gradient_sha256": sha(g), "gradient_norm": float(np.linalg.norm(g)),
                 "gradient_head": g[:16].tolist(),
                 "quartic_p_seed": 7, "quartic_p_scale": 0.1,
                 "quartic_n_chunks_1": orc.quartic(R, c["n_f"], x0, p, c["lam"], 1).tolist(),
                 "user_half_sweep_sha256": sha(users), "user_half_sweep_head": users[:16].tolist(),
                 "user_half_sweep_norm": float(np.linalg.norm(users))}
    write("c0_trace.json", out)


def c1_ttt():
    c = CONFIGS[1]
    t0 = time.time()
    R = generate(1)
    gen_s = time.time() - t0
    cores = os.cpu_count() or 1
    orc = oracle()
    cfg = make_config(lambda_=c["lam"], n_f=c["n_f"], max_iters=2000, tol=1e-6, seed=0,
                      n_blocks=16, n_workers=cores, trace_every=1, paper_timing=1)
    t0 = time.time()
    x, recs, info = orc.ncg_solve(R, cfg)
    wall = time.time() - t0
    el = [r["elapsed_seconds"] for r in recs]
    out = {"what": "BASELINE config 1 ALS-NCG to (1/N)||g|| < 1e-6 through the compiled reference "
                   "(oracle/_ref), trace every iteration",
           "config": {k: c[k] for k in ("n_u", "n_m", "nnz", "n_f", "lam", "seed")},
           "solver": {"tol": 1e-6, "seed": 0, "n_blocks": 16, "n_workers": cores,
                      "alpha0": 10.0, "armijo_c": 0.5, "tau": 0.9, "max_backtracks": 100},
           "result": info, "trace": trace_json(recs),
           "model_sha256": sha(x), "model_norm": float(np.linalg.norm(x)),
           "host": {"cores": cores, "generate_seconds": gen_s, "solve_wall_seconds": wall,
                    "paper_elapsed_seconds": el[-1] if el else None,
                    "mean_iteration_seconds_k_ge_2": (el[-1] - el[1]) / max(len(el) - 2, 1)
                    if len(el) > 2 else None}}
    write("c1_ttt_trace.json", out)


def gen():
    out = {}
    for idx in (0, 1):
        c = CONFIGS[idx]
        R = generate(idx)
        out[f"config{idx}"] = {"n_u": c["n_u"], "n_m": c["n_m"], "nnz": c["nnz"], "seed": c["seed"],
                               "triples_sha256": sha(*R.triples),
                               "csr_sha256": sha(R.uptr, R.uidx, R.uval),
                               "csc_sha256": sha(R.iptr, R.iidx, R.ival),
                               "value_histogram": np.unique(R.uval, return_counts=True)[1].tolist(),
                               "max_item_count": int(R.item_count().max()),
                               "max_user_count": int(R.user_count().max())}
    write("generator_digests.json", out)


def write(name, obj):
    path = os.path.join(HERE, name)
    with open(path, "w") as f:
        json.dump(obj, f, indent=1)
    print("wrote", path, flush=True)


if __name__ == "__main__":
    for what in sys.argv[1:] or ["c0", "gen"]:
        {"c0": c0, "c1_ttt": c1_ttt, "gen": gen}[what]()
