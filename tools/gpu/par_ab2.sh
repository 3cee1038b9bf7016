python tools/probe_ab.py --config 1 --schedule parallel --reps 3 > gpurun_out/par2.log 2>&1
GABP_PAR_PERSIST=0 python tools/probe_ab.py --config 1 --schedule parallel --reps 3 >> gpurun_out/par2.log 2>&1
python -c "import torch; p=torch.cuda.get_device_properties(0); print(p)" >> gpurun_out/par2.log 2>&1
python tools/profile_sweep.py --config 1 --schedule parallel --sweeps 4 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:slice_kernel_par -s 6 -c 1 -o gpurun_out/par_c1d python tools/profile_sweep.py --config 1 --schedule parallel --sweeps 4 > gpurun_out/ncu.log 2>&1
