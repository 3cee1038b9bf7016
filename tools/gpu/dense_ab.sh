timeout 600 python -m pytest tests -m gpu -x -q -k "dense or config3" > gpurun_out/dense_tests.log 2>&1; echo "rc=$?" >> gpurun_out/dense_tests.log
python tools/config_probe.py --config 3 --sweeps 30 > gpurun_out/c3p.log 2>&1
GABP_LIB=$PWD/paper_0810_1119_b200/lib/libgabp_b200_old.so python tools/config_probe.py --config 3 --sweeps 30 >> gpurun_out/c3p.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:dense --csv --log-file gpurun_out/c3_launches.csv python tools/config_probe.py --config 3 --sweeps 6 > gpurun_out/ncu.log 2>&1
GABP_LIB=$PWD/paper_0810_1119_b200/lib/libgabp_b200_old.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:dense --csv --log-file gpurun_out/c3_launches_old.csv python tools/config_probe.py --config 3 --sweeps 6 > gpurun_out/ncu2.log 2>&1
