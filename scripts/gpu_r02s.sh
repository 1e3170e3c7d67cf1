mkdir -p gpurun_out
timeout 900 python scripts/pick_top.py 512 1024 2048 > gpurun_out/r02s.txt 2>&1
cat gpurun_out/r02s.txt
