mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > gpurun_out/r02v_tests.txt 2>&1
tail -5 gpurun_out/r02v_tests.txt > gpurun_out/r02v.txt
( time timeout 1200 python bench.py --steps 20 --warmup 5 ) > gpurun_out/r02v_bench.log 2>&1
tail -c 2500 gpurun_out/r02v_bench.log >> gpurun_out/r02v.txt
cat gpurun_out/r02v.txt
