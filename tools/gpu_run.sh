export SYNPERF_LIB=variants/lib_pf.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_range.py -q -x -k "attention or range" > /tmp/pt.txt 2>&1; tail -n 2 /tmp/pt.txt
unset SYNPERF_LIB
bash tools/gpu_ab.sh gpurun_out/r02aj cfg2 cur pf cur pf
