import sys, os, time, ctypes as C, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1508_03110_b200 as P
from paper_1508_03110_b200 import _lib
c = P.CONFIGS[1]
R = P.generate(1)
ctx = P.Context(0)
L = _lib.lib()
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
host = [pin(R.uptr), pin(R.uidx), pin(R.uval), pin(R.iptr), pin(R.iidx), pin(R.ival)]
model = torch.empty(100 * (R.n_users() + R.n_items()), dtype=torch.float64).pin_memory()
for iters in (0, 1, 10, 10, 10, 10, 10, 10):
    ccfg = P.SolverConfig(lambda_=c["lam"], n_f=100, max_iters=max(iters, 1), tol=0.0, seed=0, paper_timing=True).to_c()
    recs = (_lib.TraceRecordC * (iters + 2))(); res = _lib.ResultC(); n = C.c_int(0)
    t0 = time.perf_counter(); h = C.c_void_p()
    _lib.check(L.alsncg_ratings_upload(ctx.handle, R.n_users(), R.n_items(), R.nnz(), *[C.c_void_p(t.data_ptr()) for t in host], C.byref(h)))
    ctx.synchronize(); t1 = time.perf_counter()
    if iters > 0:
        _lib.check(L.alsncg_ncg_solve(h, C.byref(ccfg), _lib.SNAPSHOT_FN(), None, C.byref(res), C.c_void_p(model.data_ptr()), recs, iters + 2, C.byref(n)))
    t2 = time.perf_counter()
    _lib.check(L.alsncg_ratings_free(h)); t3 = time.perf_counter()
    print(f"iters={iters}: upload {1e3*(t1-t0):.1f} ms, solve {1e3*(t2-t1):.1f} ms, free {1e3*(t3-t2):.1f} ms, trace elapsed {[round(recs[i].elapsed_seconds*1e3,1) for i in range(min(n.value,3))]}")
