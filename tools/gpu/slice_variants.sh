#!/bin/bash
# time slice-kernel build variants (lib/libgabp_b200<TAG>.so) x kernel variant (0 ldg, 1 pipe)
for t in "$@"; do
  for v in 0 1; do
    for c in 1 2; do
      GABP_SLICE_VARIANT=$v GABP_LIB=paper_0810_1119_b200/lib/libgabp_b200$t.so python tools/profile_sweep.py --config $c --gather slice --sweeps 20 2>&1 | sed "s/^/[$t v$v] /"
    done
  done
done
