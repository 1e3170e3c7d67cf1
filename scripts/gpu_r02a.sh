# round-2 first GPU call: cluster-pair bring-up, full GPU suite, bench headline
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_r02a.txt
timeout 300 python -m pytest tests/test_gpu_cluster_pairs.py -x -q 2>&1 | tail -25 > gpurun_out/pytest_qd.log
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -40 > gpurun_out/pytest_r02a.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02a.log 2>&1
tail -c 2500 gpurun_out/bench_r02a.log
cat gpurun_out/pytest_qd.log
tail -5 gpurun_out/pytest_r02a.log
