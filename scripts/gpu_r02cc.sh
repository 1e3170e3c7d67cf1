mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/r02cc.txt
timeout 300 python scripts/conv_halo_diag.py 2>&1 | grep "B=256" >> gpurun_out/r02cc.txt
timeout 600 python scripts/conv_halo_bench.py >> gpurun_out/r02cc.txt 2>&1
cat gpurun_out/r02cc.txt
