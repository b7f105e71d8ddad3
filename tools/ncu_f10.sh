set -u
O=gpurun_out/ncu_f10; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_hs_main' --launch-skip 2 -c 2 \
  -o $O/hs python bench.py --config 2 --nf 10 --steps 1 --warmup 1 --no-cpu --no-e2e --no-ttt > $O/ncu.log 2>&1
ncu -i $O/hs.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
tail -3 $O/ncu.log
