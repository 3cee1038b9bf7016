# round-2 evidence: per-config probes, the launch list of the bench command, one full ncu
# capture per dominant kernel (each only after its command exited 0 without ncu)
set -u
O=gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
for c in 1 3; do python tools/config_probe.py --config $c --sweeps 30 >> $O/r02_configs.jsonl 2>$O/config$c.err; done
python tools/grid_probe.py --dims 2 --p 4096 --sweeps 30 >> $O/r02_configs.jsonl 2>$O/grid2.err
python tools/grid_probe.py --dims 3 --p 512 --sweeps 20 >> $O/r02_configs.jsonl 2>$O/grid3.err
python tools/small_probe.py >> $O/r02_small.log 2>&1
python tools/par_probe.py --config 1 --modes slice,rows >> $O/r02_par_probe.jsonl 2>$O/par.err
# bench launch list
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/r02_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_b.log 2>&1
# config 1: group kernel, one steady full launch
python tools/profile_sweep.py --config 1 --sweeps 8 > $O/plain_p.log 2>&1 && \
$NCU -k regex:slice_kernel_grp -s 6 -c 1 -o $O/r02_slice_grp_c1 python tools/profile_sweep.py --config 1 --sweeps 8 > $O/ncu_p.log 2>&1
# config 2: diagonal-layout kernel on the 4096^2 grid
python tools/grid_probe.py --dims 2 --p 4096 --sweeps 8 --reps 1 > $O/plain_g2.log 2>&1 && \
$NCU -k regex:dia_sweep_kernel -s 6 -c 1 -o $O/r02_dia_c2 python tools/grid_probe.py --dims 2 --p 4096 --sweeps 8 --reps 1 > $O/ncu_g2.log 2>&1
# config 4 stand-in for ncu replay (ncu saves and restores device memory per pass): 320^3
python tools/grid_probe.py --dims 3 --p 320 --sweeps 8 --reps 1 > $O/plain_g3.log 2>&1 && \
$NCU -k regex:dia_sweep_kernel -s 6 -c 1 -o $O/r02_dia_p320 python tools/grid_probe.py --dims 3 --p 320 --sweeps 8 --reps 1 > $O/ncu_g3.log 2>&1
# config 3: dense kernels (walk + pairs of one sweep)
python tools/config_probe.py --config 3 --sweeps 6 > $O/plain_d.log 2>&1 && \
$NCU -k regex:dense_ -s 8 -c 2 -o $O/r02_dense_c3 python tools/config_probe.py --config 3 --sweeps 6 > $O/ncu_d.log 2>&1
# parallel schedule, config 1: warp-per-row kernel
python tools/par_probe.py --config 1 --modes rows --solve 0 --sweeps 6 > $O/plain_r.log 2>&1 && \
$NCU -k regex:rowpar_kernel -s 5 -c 1 -o $O/r02_rowpar_c1 python tools/par_probe.py --config 1 --modes rows --solve 0 --sweeps 6 > $O/ncu_r.log 2>&1
ls -la $O
