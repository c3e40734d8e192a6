mkdir -p gpurun_out/r02m
python tools/sanitize.py > gpurun_out/r02m/plain.txt 2>&1; tail -1 gpurun_out/r02m/plain.txt
for t in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize.py > gpurun_out/r02m/sanitizer_$t.txt 2>&1
  echo "$t rc=$?"; tail -3 gpurun_out/r02m/sanitizer_$t.txt
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --dist-backend gloo --steps 3 --workload cfg3 --scale 0.1 > gpurun_out/r02m/n2_cfg3.json 2> gpurun_out/r02m/n2_cfg3.err; echo n2cfg3 rc=$?; tail -c 600 gpurun_out/r02m/n2_cfg3.json; tail -3 gpurun_out/r02m/n2_cfg3.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 2 --dist-backend gloo --steps 3 --workload cfg2 --scale 0.05 > gpurun_out/r02m/n2_cfg2.json 2> gpurun_out/r02m/n2_cfg2.err; echo n2cfg2 rc=$?; tail -c 300 gpurun_out/r02m/n2_cfg2.json; tail -3 gpurun_out/r02m/n2_cfg2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29557 bench.py --gpus 2 --dist-backend gloo --steps 3 --workload cfg4 --scale 0.05 > gpurun_out/r02m/n2_cfg4.json 2> gpurun_out/r02m/n2_cfg4.err; echo n2cfg4 rc=$?; tail -c 300 gpurun_out/r02m/n2_cfg4.json; tail -3 gpurun_out/r02m/n2_cfg4.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29558 bench.py --gpus 2 --dist-backend gloo --steps 3 --workload cfg5 --scale 0.01 > gpurun_out/r02m/n2_cfg5.json 2> gpurun_out/r02m/n2_cfg5.err; echo n2cfg5 rc=$?; tail -c 300 gpurun_out/r02m/n2_cfg5.json; tail -3 gpurun_out/r02m/n2_cfg5.err
