timeout 600 python tools/e2e_chunks.py --workload cfg2 --chunks 1,3,3,1 4 6 1,2,3,3,2,1 1,4,4,1 1,2,2,2,2,1 8 1,3,3,3,1
timeout 600 python tools/e2e_chunks.py --workload cfg3 --chunks 4 8 2 1,3,3,1
