# exact twin: device tail launch (default) against a host launch per sweep (GABP_TWIN_LAUNCH=1)
for r in 1 2; do
python tools/config_probe.py --config 1 --sweeps 50 2>&1 | grep -o '"ms_per_sweep": [0-9.]*' | sed 's/^/tail /'
GABP_TWIN_LAUNCH=1 python tools/config_probe.py --config 1 --sweeps 50 2>&1 | grep -o '"ms_per_sweep": [0-9.]*' | sed 's/^/twin /'
done
