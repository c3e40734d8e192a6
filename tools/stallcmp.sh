mkdir -p gpurun_out/cmp
for v in red lin; do
SYNPERF_LIB=variants/lib_$v.so ncu --section WarpStateStats --section InstructionStats --section SchedulerStats --section LaunchStats --section Occupancy -k regex:featurize_attention_cross -s 1 -c 1 -o gpurun_out/cmp/$v python tools/time_stages.py --reps 1 > gpurun_out/cmp/$v.log 2>&1
ncu -i gpurun_out/cmp/$v.ncu-rep --page raw --csv > gpurun_out/cmp/$v.csv
done
