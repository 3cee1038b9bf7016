#!/bin/bash
# time slice-kernel variants (GABP_SLICE_VARIANT: 0 ldg, 1 pipe, 2 tma) on configs 1 and 2
for c in ${CONFIGS:-1 2}; do
  for v in ${VARIANTS:-0 2}; do
    GABP_SLICE_VARIANT=$v python tools/profile_sweep.py --config $c --gather slice --sweeps 30 --solve 2>&1 | sed "s/^/[c$c v$v] /"
  done
done
