mkdir -p gpurun_out/r02q
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02q/pytest.txt 2>&1; tail -n 4 gpurun_out/r02q/pytest.txt
timeout 300 python tools/time_stages.py --reps 10 > gpurun_out/r02q/stages.txt 2>&1; cat gpurun_out/r02q/stages.txt
