# round-2 final evidence: GPU suite, headline bench, launch list of the bench command, full
# ncu capture of the headline chain kernel
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/r02jj.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02jj_bench.log 2>&1
tail -1 gpurun_out/r02jj_bench.log >> gpurun_out/r02jj.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02jj_launches.csv python bench.py --plan fixed --steps 5 --warmup 3 --no-sweep > gpurun_out/r02jj_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -c 1 -o gpurun_out/r02jj_chain python bench.py --plan fixed --steps 2 --warmup 1 --no-sweep > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/r02jj_chain.ncu-rep >> gpurun_out/r02jj.txt 2>&1
cat gpurun_out/r02jj.txt
