set -u
O=gpurun_out/${1:-f200a}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "half_sweep" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 1200 python -m pytest tests/test_gpu_scale.py -x -q -k "half_sweeps_every_column and (200 or 100)" > $O/pytest_scale.log 2>&1; tail -3 $O/pytest_scale.log
for nf in ${NFS:-200 160 136 100}; do
  NO_TRACE=1 timeout 600 python tools/quick_bench.py 1 $nf 3 > $O/f$nf.log 2>&1
  grep -H "ms/iter \|halfsweep_gram\|halfsweep_solve " $O/f$nf.log
done
