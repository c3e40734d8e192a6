mkdir -p gpurun_out/r02o
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02o/pytest.txt 2>&1; tail -n 4 gpurun_out/r02o/pytest.txt
bash tools/gpu_ab.sh gpurun_out/r02o cfg2 orig default
