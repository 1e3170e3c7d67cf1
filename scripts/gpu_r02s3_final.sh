# session-3 closing check of the final tree: smoke, full GPU suite, the driver's bench invocation
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02s3_final.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 >> gpurun_out/r02s3_final.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02s3_final_bench.log 2>&1
tail -1 gpurun_out/r02s3_final_bench.log >> gpurun_out/r02s3_final.txt
cp gpurun_out/bench_detail.json gpurun_out/r02s3_final_bench_detail.json
cat gpurun_out/r02s3_final.txt
