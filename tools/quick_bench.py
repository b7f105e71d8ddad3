"""Quick device timing of the ALS-NCG iteration on a BASELINE config with
per-kernel CUDA-event stats (development aid; bench.py is the contract)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_03110_b200 as P

cfg_idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n_f = int(sys.argv[2]) if len(sys.argv) > 2 else P.CONFIGS[cfg_idx]["n_f"]
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 5
c = P.CONFIGS[cfg_idx]
t = time.time(); R = P.generate(cfg_idx); print(f"generate {time.time()-t:.1f}s nnz={R.nnz()}", flush=True)
ctx = P.default_context()
t = time.time(); R.device(ctx); print(f"upload {time.time()-t:.2f}s", flush=True)
cfg = P.SolverConfig(lambda_=c["lam"], n_f=n_f, max_iters=1000, tol=0.0, seed=0,
                     trace_every=10**9 if os.environ.get("NO_TRACE") else 1)  # NO_TRACE: paper_timing-like
t = time.time(); s = P.ncg.Solver(R, cfg); ctx.synchronize(); print(f"setup {time.time()-t:.2f}s", flush=True)
s.step(1); ctx.synchronize()
ctx.reset_stats(); ctx.set_profiling(True)
t = time.time(); s.step(iters); ctx.synchronize(); dt = (time.time()-t)/iters
ctx.set_profiling(False)
print(f"f={n_f}: {dt*1e3:.2f} ms/iter  {R.nnz()/dt/1e9:.3f} G ratings/s")
st = ctx.kernel_stats()
for k, (n, ms) in sorted(st.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:28s} {n:6d} launches {ms/iters:9.3f} ms/iter")
print(s.state())
