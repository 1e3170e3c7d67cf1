# session-3 final evidence on the shipped build: the driver's bench invocation (sweeps in bench_detail.json),
# the launch list of the fixed-plan bench command, ncu --set full of the headline chain and of the halo conv
mkdir -p gpurun_out
echo "GPU suite: see r02s3b (282 passed on this build)" > gpurun_out/r02s3c.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02s3c_bench.log 2>&1
tail -1 gpurun_out/r02s3c_bench.log >> gpurun_out/r02s3c.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02s3c_launches.csv python bench.py --plan fixed --steps 5 --warmup 3 --no-sweep > gpurun_out/r02s3c_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -c 1 -o gpurun_out/r02s3c_chain python bench.py --plan fixed --steps 2 --warmup 1 --no-sweep > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/r02s3c_chain.ncu-rep >> gpurun_out/r02s3c.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 3 -c 1 -o gpurun_out/r02s3c_halo python scripts/conv_halo_quick.py 56:256 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/r02s3c_halo.ncu-rep >> gpurun_out/r02s3c.txt 2>&1
cat gpurun_out/r02s3c.txt
cp gpurun_out/bench_detail.json gpurun_out/r02s3c_bench_detail.json
