# B=256 per-unit timelines of a few plans
mkdir -p gpurun_out
: > gpurun_out/r02hh.txt
python scripts/dump_trace.py 256 b256_qd '{"tile_n":256,"cta_group":2,"prod_tile_n":512,"cons_tile_n":512,"prod_splits":2,"cluster_pairs":2}' >> gpurun_out/r02hh.txt 2>&1
python scripts/dump_trace.py 256 b256_z3 '{"tile_n":256,"cta_group":2,"prod_tile_n":512,"cons_tile_n":512,"prod_splits":3}' >> gpurun_out/r02hh.txt 2>&1
python scripts/dump_trace.py 256 b256_z6c3 '{"tile_n":256,"cta_group":2,"prod_tile_n":512,"cons_tile_n":512,"prod_splits":6,"cons_splits":3}' >> gpurun_out/r02hh.txt 2>&1
for n in b256_qd b256_z3 b256_z6c3; do python scripts/unit_timeline.py gpurun_out/trace_$n.json --units 3 >> gpurun_out/r02hh.txt 2>&1; done
cat gpurun_out/r02hh.txt
