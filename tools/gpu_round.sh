#!/bin/bash
# One GPU-box pass: GPU tests, smoke, bench (config 1), ncu launch list, ncu --set full of the hot kernels.
# usage: tools/gpu_round.sh TAG [skip-tests]
set -u
TAG=${1:-r02}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi -L > $O/gpu.txt 2>&1
if [ "${2:-}" != "skip-tests" ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
  timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
fi
timeout 900 python bench.py > $O/bench_c1.json 2> $O/bench_c1.err; echo "bench exit $?" >> $O/bench_c1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-ttt > $O/ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_hs_solve_ws|k_quartic|k_gradient$|k_hs_gram_ws' --launch-skip 6 -c 5 \
  -o $O/hot python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-ttt > $O/ncu_full.log 2>&1
echo done
