# balanced (stream-K) schedule: tests, then timing vs planner pick vs cuBLAS
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_balanced.py -x -q 2>&1 | tail -15 > gpurun_out/r02n.txt
timeout 900 python scripts/balanced_bench.py 256 512 1024 2048 >> gpurun_out/r02n.txt 2>&1
cat gpurun_out/r02n.txt
