# generations (measured side), co-resident timing, ncu capture of the shipped fixed plan
mkdir -p gpurun_out
timeout 600 python scripts/gen_trace.py 1024 pick=pick 'fixed={"tile_n":256,"cta_group":2,"prod_tile_n":512,"cons_tile_n":512,"cons_tail":[22,2],"cons_order":"band4"}' > gpurun_out/r02m.txt 2>&1
timeout 600 python scripts/gen_trace.py 2048 pick=pick >> gpurun_out/r02m.txt 2>&1
timeout 300 python scripts/coresident_bench.py 256 1024 2048 >> gpurun_out/r02m.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -c 1 -o gpurun_out/fixed_r02m python bench.py --plan fixed --steps 2 --warmup 1 --no-sweep > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/fixed_r02m.ncu-rep >> gpurun_out/r02m.txt 2>&1
cat gpurun_out/r02m.txt
