# session-3 re-entry check of HEAD: full GPU suite + the driver's bench invocation
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 > gpurun_out/r02s3.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02s3_bench.log 2>&1
tail -1 gpurun_out/r02s3_bench.log >> gpurun_out/r02s3.txt
cat gpurun_out/r02s3.txt
