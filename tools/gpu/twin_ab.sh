timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
for r in 1 2; do
python tools/config_probe.py --config 1 --sweeps 50 2>&1 | grep -o '"ms_per_sweep": [0-9.]*' | sed 's/^/tail /'
GABP_TWIN_LAUNCH=1 python tools/config_probe.py --config 1 --sweeps 50 2>&1 | grep -o '"ms_per_sweep": [0-9.]*' | sed 's/^/twin /'
done
python tools/probe_ab.py --config 1 --reps 5
GABP_TWIN_LAUNCH=1 python tools/probe_ab.py --config 1 --reps 5
python tools/probe_ab.py --config 0 --reps 2
python tools/config_probe.py --config 2 --sweeps 20 2>&1 | grep -o '"ms_per_sweep": [0-9.]*' | sed 's/^/c2 /'
