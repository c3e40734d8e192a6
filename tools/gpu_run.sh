bash tools/gpu_ab.sh gpurun_out/r02t cfg2 em1 em3 em4 em1 em3
