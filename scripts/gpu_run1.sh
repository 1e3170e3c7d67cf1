set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_r02a.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02a.log 2>&1
tail -c 3000 gpurun_out/bench_r02a.log
timeout 600 python scripts/timeline.py 1024 stream:row:row:band4:0:0:1/1:512/512 fused:row:row:band4:0:0:1/1:512/512:22,3 fused:row:row:band4:0:0:3/1:512/512 fused:row:row:band4:0:0:3/1:512/512:18,3 fused:row:row:band4:0:0:2/1:512/512:22,3 > gpurun_out/timeline_r02a.txt 2>&1
cat gpurun_out/pytest_r02a.log
