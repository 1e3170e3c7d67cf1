mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/r02x.txt
timeout 400 python scripts/ab_red.py >> gpurun_out/r02x.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 2>&1 | tail -1 >> gpurun_out/r02x.txt
cat gpurun_out/r02x.txt
