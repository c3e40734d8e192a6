mkdir -p gpurun_out/r02s
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_range.py tests/test_gpu_sched.py -q -x > gpurun_out/r02s/pytest.txt 2>&1; tail -n 2 gpurun_out/r02s/pytest.txt
bash tools/gpu_ab.sh gpurun_out/r02s cfg2 prev faA faB default prev default
