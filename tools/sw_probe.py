import sys, os, ctypes, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1508_03110_b200 as P
from paper_1508_03110_b200 import _lib
c = P.CONFIGS[1]
R = P.generate(1)
ctx = P.default_context()
R.device(ctx)
cfg = P.SolverConfig(lambda_=c["lam"], n_f=100, max_iters=10, tol=0.0, seed=0)
s = P.ncg.Solver(R, cfg)   # setup runs P(x0): user then item half-sweep; the probe keeps the LAST launch
ctx.synchronize()
buf = (ctypes.c_ulonglong * (64 * 64))()
print("rc", _lib.lib().alsncg_debug_sw_probe_13(buf))
a = np.frombuffer(buf, dtype=np.uint64).reshape(64, 64).astype(np.int64)
for b in range(0, 64, 8):
    row = a[b]
    t0 = row[0]
    print("col", b, "load", row[1] - t0, "back", row[61] - row[60], "total", row[61] - t0)
    print("   T  ", [int(row[3 + 4 * J] - row[2 + 4 * J]) for J in range(13)])
    print("   U0 ", [int(row[5 + 4 * J] - row[4 + 4 * J]) for J in range(12)])
    print("   F  ", [int(row[2 + 4 * (J + 1)] - row[5 + 4 * J]) for J in range(12)])
    print("   bar", [int(row[4 + 4 * J] - row[3 + 4 * J]) for J in range(13)])
