mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_split_fixup.py -x -q 2>&1 | tail -15 > gpurun_out/r02ii.txt
timeout 300 python scripts/ab_lib.py >> gpurun_out/r02ii.txt 2>&1
TS_LIB_PATH=ab/lib_r12.so timeout 300 python scripts/ab_lib.py >> gpurun_out/r02ii.txt 2>&1
timeout 900 python scripts/fixup_bench.py >> gpurun_out/r02ii.txt 2>&1
cat gpurun_out/r02ii.txt
