set -u
O=gpurun_out/ncu_resid; mkdir -p $O
ALSNCG_RING=0 timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_quartic|k_gradient' --launch-skip 4 -c 3 \
  -o $O/resid python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-ttt > $O/ncu.log 2>&1
tail -3 $O/ncu.log
