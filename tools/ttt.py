"""Time-to-tolerance on BASELINE config 1: ALS-NCG until
(1/N)||g|| < tol (ncg.cpp:285-286), paper_timing (trace loss excluded).
   python tools/ttt.py [tol] [max_iters] [n_f]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_03110_b200 as P

tol = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-6
max_iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
n_f = int(sys.argv[3]) if len(sys.argv) > 3 else 100
c = P.CONFIGS[1]
R = P.generate(1)
ctx = P.default_context()
R.device(ctx)
cfg = P.SolverConfig(lambda_=c["lam"], n_f=n_f, max_iters=max_iters, tol=tol, seed=0, paper_timing=True,
                     trace_every=50)
t0 = time.time()
res = P.ncg.als_ncg_solve(R, cfg)
wall = time.time() - t0
tr = res.trace.records
print(f"converged={res.converged} iterations={res.iterations} final_grad_norm={res.final_grad_norm:.3e} "
      f"time_to_tolerance={tr[-1].elapsed_seconds:.2f}s wall={wall:.2f}s "
      f"restarts={res.restarts if hasattr(res, 'restarts') else '?'}")
for r in tr[:: max(1, len(tr) // 12)]:
    print(f"  k={r.iter:5d} loss={r.loss:.6e} gnorm={r.grad_norm:.3e} t={r.elapsed_seconds:.2f}s")
