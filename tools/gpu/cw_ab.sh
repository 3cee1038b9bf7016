# narrow-launch timing + launch list of one solve (config 1), GPU tests
python tools/probe_ab.py --config 1 > gpurun_out/cw.log 2>&1
python tools/probe_ab.py --config 0 --reps 2 >> gpurun_out/cw.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
python tools/probe_ab.py --config 1 --reps 1 > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:slice_kernel --csv --log-file gpurun_out/cw_launches.csv python tools/probe_ab.py --config 1 --reps 1 > gpurun_out/ncu.log 2>&1
