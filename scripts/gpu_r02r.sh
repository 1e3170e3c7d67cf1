mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_chain.py tests/test_gpu_balanced.py -x -q 2>&1 | tail -6 > gpurun_out/r02r.txt
timeout 900 python scripts/pick_top.py 512 1024 2048 >> gpurun_out/r02r.txt 2>&1
cat gpurun_out/r02r.txt
