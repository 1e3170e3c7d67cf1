mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_symm_allreduce.py tests/test_gpu_bench_parity.py -x -q -k "symm or vgg" 2>&1 | tail -15 > gpurun_out/r02q.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-sweep --fused-allreduce 2>&1 | tail -1 >> gpurun_out/r02q.txt
cat gpurun_out/r02q.txt
