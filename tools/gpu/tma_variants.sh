#!/bin/bash
# time TMA-ring build variants (lib/libgabp_b200<TAG>.so) on configs 1 and 2
for t in "$@"; do
  for c in ${CONFIGS:-1 2}; do
    GABP_SLICE_VARIANT=2 GABP_LIB=paper_0810_1119_b200/lib/libgabp_b200$t.so python tools/profile_sweep.py --config $c --gather slice --sweeps 30 2>&1 | sed "s/^/[$t] /"
  done
done
