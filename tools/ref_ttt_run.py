"""Runs the REFERENCE (oracle/_ref, compiled in place) on config 1 to
(1/N)||g|| < 1e-6 with a chosen n_blocks (the quartic's chunk count, which only
changes summation order) and writes its trace as JSON -- the sensitivity check
of the iteration count to rounding order.  Test infrastructure only.
  python tools/ref_ttt_run.py N_BLOCKS OUT.json"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.pyoracle import CONFIGS, Oracle, generate, make_config  # noqa: E402

nb, out = int(sys.argv[1]), sys.argv[2]
c = CONFIGS[1]
R = generate(1)
cores = os.cpu_count() or 1
cfg = make_config(lambda_=c["lam"], n_f=c["n_f"], max_iters=2000, tol=1e-6, seed=0, n_blocks=nb,
                  n_workers=cores, trace_every=1, paper_timing=1)
t0 = time.time()
x, recs, info = Oracle("ref").ncg_solve(R, cfg)
json.dump({"n_blocks": nb, "cores": cores, "wall_s": time.time() - t0, "result": info,
           "trace": [dict(iter=r["iter"], loss=r["loss"], grad_norm=r["grad_norm"],
                          backtracks=r["backtracks"], restarted=bool(r["restarted"])) for r in recs]},
          open(out, "w"), indent=1)
print("done", info)
