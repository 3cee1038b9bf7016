# round evidence: per-config probes, launch list of the bench command, full ncu of one
# full group launch (config 1) and of the dense pair kernel (config 3)
for c in 1 2 3 4; do python tools/config_probe.py --config $c --sweeps 30 >> gpurun_out/configs.jsonl 2>gpurun_out/config$c.err; done
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1
python tools/profile_sweep.py --config 1 --sweeps 4 > gpurun_out/plain_p.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:slice_kernel_grp -s 3 -c 1 -o gpurun_out/grp_c1 python tools/profile_sweep.py --config 1 --sweeps 4 > gpurun_out/ncu_p.log 2>&1
python tools/config_probe.py --config 3 --sweeps 6 > gpurun_out/plain_d.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dense -s 4 -c 2 -o gpurun_out/dense_c3 python tools/config_probe.py --config 3 --sweeps 6 > gpurun_out/ncu_d.log 2>&1
