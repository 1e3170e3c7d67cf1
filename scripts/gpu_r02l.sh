# co-resident mode tests, then the full GPU suite
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_coresident.py -x -q 2>&1 | tail -15 > gpurun_out/r02l.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 >> gpurun_out/r02l.txt
cat gpurun_out/r02l.txt
