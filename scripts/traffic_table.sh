# DRAM bytes per launch (ncu, one launch each) for the B=1024 configurations the planner
# picks between; feeds profiles/roofline_traffic.json.
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for cfg in "row 512 512 4 3 1 1 0,1" "row 512 512 4 3 1 1 22,2" "row 512 512 4 3 1 1 22,3" \
           "row 512 512 4 3 2 1 0,1" "row 512 512 4 3 2 1 22,2" "row 512 512 4 3 2 1 22,3" \
           "row 512 512 1 3 1 1 0,1" "tile 512 512 4 3 2 1 0,1"; do
  echo "== $cfg"
  timeout 120 ncu --metrics $M --clock-control none -k regex:chain_kernel -s 2 -c 1 \
    python scripts/prof_one.py 1024 fused $cfg 2>&1 | grep -E "dram__|gpu__time"
done
