"""ALS-NCG with and without CUDA-graph replay of the gradient / P(x) / gbar sequence
(ALSNCG_GRAPH=1): traces must be identical, per-iteration wall time is printed.
  python tools/graph_probe.py [config] [n_f] [iters]     (run once per setting of ALSNCG_GRAPH)"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_03110_b200 as P

cfg_idx = int(sys.argv[1]) if len(sys.argv) > 1 else 0
c = P.CONFIGS[cfg_idx]
n_f = int(sys.argv[2]) if len(sys.argv) > 2 else c["n_f"]
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 200
R = P.generate(cfg_idx)
ctx = P.default_context()
R.device(ctx)
cfg = P.SolverConfig(lambda_=c["lam"], n_f=n_f, max_iters=10**6, tol=0.0, seed=0, trace_every=10**9)
s = P.ncg.Solver(R, cfg)
s.step(5); ctx.synchronize()
t = time.perf_counter(); s.step(iters); ctx.synchronize(); dt = (time.perf_counter() - t) / iters
st = s.state()
print(json.dumps({"graph": bool(os.environ.get("ALSNCG_GRAPH")), "config": cfg_idx, "n_f": n_f,
                  "ms_per_iteration": dt * 1e3, "grad_norm": st["grad_norm"], "iterations": st["iterations"]}))
