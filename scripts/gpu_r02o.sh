mkdir -p gpurun_out
timeout 300 python scripts/dump_trace.py 1024 bal '{"tile_n":256,"cta_group":2,"prod_tile_n":512,"cons_tile_n":512,"balanced":true}' > gpurun_out/r02o.txt 2>&1
timeout 300 python scripts/dump_trace.py 1024 split2 '{"tile_n":256,"cta_group":2,"prod_tile_n":512,"cons_tile_n":512,"prod_splits":2,"cons_order":"band4"}' >> gpurun_out/r02o.txt 2>&1
timeout 300 python scripts/dump_trace.py 512 bal512 '{"tile_n":256,"cta_group":2,"prod_tile_n":512,"cons_tile_n":512,"balanced":true}' >> gpurun_out/r02o.txt 2>&1
cat gpurun_out/r02o.txt
