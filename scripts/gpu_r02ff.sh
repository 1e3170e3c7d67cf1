mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ready_first.py -x -q 2>&1 | tail -15 > gpurun_out/r02ff.txt
timeout 900 python scripts/rf_bench.py >> gpurun_out/r02ff.txt 2>&1
cat gpurun_out/r02ff.txt
