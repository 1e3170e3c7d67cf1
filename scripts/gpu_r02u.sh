mkdir -p gpurun_out
timeout 900 python scripts/pick_top.py 512 1024 2048 > gpurun_out/r02u.txt 2>&1
timeout 300 python scripts/dump_trace.py 1024 w384 '{"tile_n":256,"cta_group":2,"prod_tile_n":384,"cons_tile_n":512,"cons_tail":[22,3]}' >> gpurun_out/r02u.txt 2>&1
cat gpurun_out/r02u.txt
