set -u
O=gpurun_out/${1:-abl}; mkdir -p $O
for lib in paper_1508_03110_b200/libalsncg_b200.so abl/lib_*.so; do
  n=$(basename $lib .so)
  for nf in ${NFS:-100 50}; do
    ALSNCG_LIB=$PWD/$lib NO_TRACE=1 timeout 300 python tools/quick_bench.py ${CFG:-1} $nf ${IT:-3} > $O/${n}_f$nf.log 2>&1
  done
done
grep -H "${PAT:-halfsweep_gram\|halfsweep_solve }" $O/*.log
