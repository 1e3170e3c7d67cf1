# round-2 re-entry check: GPU tests, smoke, the driver's bench invocation (full sweep)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r02j.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r02j.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02j_bench.log 2>&1
tail -c 3000 gpurun_out/r02j_bench.log >> gpurun_out/r02j.txt
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 2>&1 | tail -1 >> gpurun_out/r02j.txt
cat gpurun_out/r02j.txt
