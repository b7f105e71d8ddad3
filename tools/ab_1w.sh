set -u
O=gpurun_out/${1:-ab1w}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "half_sweep" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for mx in 0 26; do
  for nf in 31 40 50 60 75 90 100; do
    ALSNCG_SOLVE_1W_MAX=$mx NO_TRACE=1 timeout 300 python tools/quick_bench.py 1 $nf 3 > $O/m${mx}_f$nf.log 2>&1
  done
done
grep -H "halfsweep_solve " $O/*.log
