# DRAM traffic and time of the split-K B=1024 pick with and without the partial-plane L2
# hints (flag bit 26), one ncu launch each, then untraced timings.
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for cfg in "row 512 512 4 3 2 1" "row 512 512 4 3 2 2"; do
  for fl in 0 0x4000000; do
    echo "== $cfg flags $fl"
    TS_EXTRA_FLAGS=$fl timeout 120 ncu --metrics $M --clock-control none -k regex:chain_kernel -s 2 -c 1 \
      python scripts/prof_one.py 1024 fused $cfg 2>&1 | grep -E "dram__|gpu__time"
  done
done
