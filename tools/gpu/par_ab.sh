# parallel-schedule GPU tests and solve timings (configs 1, 2)
timeout 900 python -m pytest tests -m gpu -x -q -k "parallel or probe or sched" > gpurun_out/par_tests.log 2>&1; echo "rc=$?" >> gpurun_out/par_tests.log
python tools/probe_ab.py --config 1 --schedule parallel --reps 3 > gpurun_out/par.log 2>&1
python tools/probe_ab.py --config 2 --schedule parallel --reps 1 >> gpurun_out/par.log 2>&1
