for c in 1 2 3 4; do python tools/config_probe.py --config $c --sweeps 30 >> gpurun_out/configs.jsonl 2>gpurun_out/config$c.err; done
python bench.py > gpurun_out/bench_final.log 2>&1
