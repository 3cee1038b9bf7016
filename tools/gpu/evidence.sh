# round evidence: bench line, launch list of the bench command, full ncu of one full group launch
python bench.py > gpurun_out/bench_full.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1
python tools/profile_sweep.py --config 1 --sweeps 4 > gpurun_out/plain_p.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:slice_kernel_grp -s 3 -c 1 -o gpurun_out/grp_c1 python tools/profile_sweep.py --config 1 --sweeps 4 > gpurun_out/ncu_p.log 2>&1
