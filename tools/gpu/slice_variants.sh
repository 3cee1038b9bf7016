#!/bin/bash
# time the slice kernel build variants (paper_0810_1119_b200/lib/libgabp_b200_<TAG>.so)
for t in "$@"; do
  for c in 1 2; do
    GABP_LIB=paper_0810_1119_b200/lib/libgabp_b200$t.so python tools/profile_sweep.py --config $c --gather slice --sweeps 20 --solve 2>&1 | sed "s/^/[$t] /"
  done
done
