"""Development aid: phase clocks of k_hs_solve_ws (build NB=13 with
EXTRA=-DAB2_WS_PROBE tools/rebuild_nb.sh 13)."""
import sys, os, ctypes, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1508_03110_b200 as P
from paper_1508_03110_b200 import _lib
c = P.CONFIGS[1]
R = P.generate(1)
ctx = P.default_context()
R.device(ctx)
cfg = P.SolverConfig(lambda_=c["lam"], n_f=100, max_iters=10, tol=0.0, seed=0)
s = P.ncg.Solver(R, cfg)   # setup runs P(x0); the probe keeps the LAST solve launch (items)
s.step(1)
ctx.synchronize()
buf = (ctypes.c_ulonglong * (64 * 64))()
print("rc", _lib.lib().alsncg_debug_ws_probe_13(buf))
a = np.frombuffer(buf, dtype=np.uint64).reshape(64, 64).astype(np.int64)
for b in range(0, 64, 8):
    row = a[b]
    t0 = row[0]
    print("cta", b, "warpid pivot/dmma", row[62], row[63], "load", row[1] - t0, "fwd", row[60] - row[1],
          "back", row[61] - row[60], "total", row[61] - t0)
    print("   wait ", [int(row[2 + 3 * J] - (row[4 + 3 * (J - 1)] if J else row[1])) for J in range(13)])
    print("   F    ", [int(row[3 + 3 * J] - row[2 + 3 * J]) for J in range(13)])
    print("   DMMA ", [int(row[4 + 3 * J] - row[3 + 3 * J]) for J in range(12)])
