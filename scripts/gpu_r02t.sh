mkdir -p gpurun_out
timeout 300 python scripts/dump_trace.py 1024 z3tail '{"tile_n":256,"cta_group":2,"prod_tile_n":512,"cons_tile_n":512,"prod_splits":3,"cons_tail":[22,3]}' > gpurun_out/r02t.txt 2>&1
timeout 300 python scripts/dump_trace.py 1024 z1tail '{"tile_n":256,"cta_group":2,"prod_tile_n":512,"cons_tile_n":512,"cons_order":"band4","cons_tail":[22,3]}' >> gpurun_out/r02t.txt 2>&1
cat gpurun_out/r02t.txt
