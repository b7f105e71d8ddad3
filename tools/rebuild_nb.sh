#!/bin/bash
# Development aid: rebuild only the half-sweep unit(s) for the given block
# counts (k_hs_inst.cu with -DAB2_HS_NB=n) and relink the library, leaving the
# other per-NB objects as they are.   tools/rebuild_nb.sh 13 [7 ...]
set -e
cd "$(dirname "$0")/../paper_1508_03110_b200/csrc"
B="$(pwd)/build"
keep=()
for n in $(seq 1 26); do
  skip=0
  for m in "$@"; do [ "$n" = "$m" ] && skip=1; done
  [ $skip = 0 ] && keep+=(-o $B/k_hs_nb$n.o)
done
for m in "$@"; do rm -f $B/k_hs_nb$m.o; done
make -s -j 8 "${keep[@]}" ${EXTRA:+NVFLAGS_EXTRA="$EXTRA"}
