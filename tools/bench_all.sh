#!/bin/bash
# Bench lines of every BASELINE config on one GPU (profiles/bench_<tag>_*.json).
# usage: tools/bench_all.sh TAG
set -u
TAG=${1:-r02}
O=gpurun_out/$TAG; mkdir -p $O
for nf in 10 25 50 200; do
  timeout 1200 python bench.py --config 2 --nf $nf --no-cpu > $O/bench_c2_nf$nf.json 2> $O/bench_c2_nf$nf.err
done
timeout 1500 python bench.py --config 3 --no-cpu > $O/bench_c3.json 2> $O/bench_c3.err
timeout 2400 python bench.py --config 4 --no-cpu --steps 5 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --config 0 --no-cpu > $O/bench_c0.json 2> $O/bench_c0.err
echo done
