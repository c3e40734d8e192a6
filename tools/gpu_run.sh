mkdir -p gpurun_out/r02z
timeout 900 ncu --set full --import-source on --clock-control none -k regex:predict_tcgen05_fused -s 3 -c 1 -o gpurun_out/r02z/fused python bench.py --workload cfg3 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r02z/ncu.log 2>&1
ls gpurun_out/r02z
