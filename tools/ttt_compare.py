"""Config 1, ALS-NCG to (1/N)||g|| < 1e-6 on the B200, compared record by
record with the reference's committed trace (tests/golden/c1_ttt_trace.json):
first iteration whose backtrack count or restart flag differs, relative loss
and gradient-norm differences along the way, final counts.
  python tools/ttt_compare.py [--ref-nblocks N]   (development / report aid)"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1508_03110_b200 as P  # noqa: E402

g = json.load(open(os.path.join(ROOT, "tests", "golden", "c1_ttt_trace.json")))
c, s = g["config"], g["solver"]
R = P.generate(1)
cfg = P.SolverConfig(lambda_=c["lam"], n_f=c["n_f"], max_iters=400, tol=s["tol"], seed=s["seed"],
                     n_blocks=s["n_blocks"], trace_every=1, paper_timing=True)
res = P.ncg.als_ncg_solve(R, cfg)
mine = res.trace.records
ref = g["trace"]
first = None
rows = []
for a, b in zip(mine, ref):
    dl = abs(a.loss - b["loss"]) / abs(b["loss"])
    dg = abs(a.grad_norm - b["grad_norm"]) / b["grad_norm"]
    same = a.backtracks == b["backtracks"] and a.restarted == b["restarted"]
    if not same and first is None:
        first = a.iter
    rows.append((a.iter, a.backtracks, b["backtracks"], dl, dg))
print(f"GPU: {res.iterations} iterations (converged={res.converged}, restarts={res.restarts}, "
      f"final (1/N)||g|| {res.final_grad_norm:.6e}); reference: {g['result']['iterations']} iterations "
      f"(restarts={g['result']['restarts']}, final {g['result']['final_grad_norm']:.6e})")
print(f"first iteration with a different backtrack count / restart flag: {first}")
for it, bm, br, dl, dg in rows:
    if it < 12 or it % 10 == 0 or (first is not None and abs(it - first) <= 2) or it >= min(len(mine), len(ref)) - 4:
        print(f"  iter {it:4d}  backtracks gpu {bm:3d} ref {br:3d}  |dloss|/loss {dl:.2e}  |dgn|/gn {dg:.2e}")
