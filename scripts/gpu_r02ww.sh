# round-2 final evidence: full GPU suite, headline bench (driver invocation), launch list of
# the fixed-plan bench command, full ncu captures of the headline chain and of the halo conv
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/r02ww.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02ww_bench.log 2>&1
tail -1 gpurun_out/r02ww_bench.log >> gpurun_out/r02ww.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02ww_launches.csv python bench.py --plan fixed --steps 5 --warmup 3 --no-sweep > gpurun_out/r02ww_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -c 1 -o gpurun_out/r02ww_chain python bench.py --plan fixed --steps 2 --warmup 1 --no-sweep > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/r02ww_chain.ncu-rep >> gpurun_out/r02ww.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 3 -c 1 -o gpurun_out/r02ww_halo python scripts/conv_halo_quick.py 56:256 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/r02ww_halo.ncu-rep >> gpurun_out/r02ww.txt 2>&1
cat gpurun_out/r02ww.txt
