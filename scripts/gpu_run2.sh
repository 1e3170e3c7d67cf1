# QD (two-pair cluster) bring-up: short, time-boxed tests first
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_cluster_pairs.py -x -q 2>&1 | tail -25 > gpurun_out/pytest_qd.log
cat gpurun_out/pytest_qd.log
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -25 > gpurun_out/pytest_r02b.log
cat gpurun_out/pytest_r02b.log
timeout 600 python scripts/timeline.py 1024 fused:row:row:band4:0:0:1/1:512/512:22,3 > gpurun_out/timeline_r02b.txt 2>&1
timeout 600 python scripts/timeline.py 1024 fused:row:row:band4:0:0:1/1:512/512:0,1:2 fused:row:row:row:0:0:1/1:512/512:0,1:2 fused:row:row:band4:0:0:1/1:512/512:22,3:2 fused:row:row:band4:0:0:2/1:512/512:22,3:2 stream:row:row:band4:0:0:1/1:512/512:0,1:2 >> gpurun_out/timeline_r02b.txt 2>&1
cat gpurun_out/timeline_r02b.txt
