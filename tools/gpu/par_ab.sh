timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
python tools/probe_ab.py --config 1 --schedule parallel --reps 3 > gpurun_out/par.log 2>&1
python tools/probe_ab.py --config 2 --schedule parallel --reps 1 >> gpurun_out/par.log 2>&1
