# unified operand ring: GEMM efficiency, GPU tests, bench
mkdir -p gpurun_out
timeout 600 python scripts/gemm_eff.py 1024 6144 12288 1024 12288 6144 18944 6144 12288 > gpurun_out/gemm_eff_r02c.txt 2>&1
cat gpurun_out/gemm_eff_r02c.txt
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_r02c.log
cat gpurun_out/pytest_r02c.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-sweep > gpurun_out/bench_r02c.log 2>&1
tail -c 1500 gpurun_out/bench_r02c.log
