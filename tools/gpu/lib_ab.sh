#!/bin/bash
# A/B of tagged library builds (make DEFS=... TAG=_x) on one config: ms/sweep and frac
# usage: tools/gpu/lib_ab.sh "<tags>" [config] [reps]
L=$PWD/paper_0810_1119_b200/lib
for i in $(seq ${3:-2}); do
  for t in $1; do
    [ "$t" = base ] && lib=$L/libgabp_b200.so || lib=$L/libgabp_b200_$t.so
    echo -n "$t: "
    GABP_LIB=$lib python tools/config_probe.py --config ${2:-1} --sweeps 30 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_sweep'], round(d['frac_of_measured_hbm'],4))"
  done
done
