mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_chain.py -x -q -k "B1024 or B2048 or B256 or tail or split or cluster" 2>&1 | tail -8 > gpurun_out/r02w.txt
timeout 600 python scripts/pick_top.py 256 512 1024 2048 >> gpurun_out/r02w.txt 2>&1
timeout 300 python scripts/dump_trace.py 1024 z3tail_r '{"tile_n":256,"cta_group":2,"prod_tile_n":512,"cons_tile_n":512,"prod_splits":3,"cons_tail":[22,3]}' >> gpurun_out/r02w.txt 2>&1
cat gpurun_out/r02w.txt
