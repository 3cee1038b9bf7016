export GABP_HOST_TIMING=1
for c in 0 1; do
  python tools/probe_ab.py --config $c 2>&1 | grep -v "run_solve\|graph_create\|build" | tail -2
  GABP_NO_PROBE=1 python tools/probe_ab.py --config $c 2>&1 | grep -v "run_solve\|graph_create\|build" | tail -2
done
python tools/probe_ab.py --config 1 --schedule parallel 2>&1 | tail -2
GABP_NO_PROBE=1 python tools/probe_ab.py --config 1 --schedule parallel 2>&1 | tail -2
