mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_conv_halo.py -x -q 2>&1 | tail -25 > gpurun_out/r02y.txt
timeout 600 python scripts/conv_halo_bench.py >> gpurun_out/r02y.txt 2>&1
cat gpurun_out/r02y.txt
