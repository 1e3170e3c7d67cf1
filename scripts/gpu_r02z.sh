mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/r02z.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02z_bench.log 2>&1
tail -1 gpurun_out/r02z_bench.log >> gpurun_out/r02z.txt
cat gpurun_out/r02z.txt
