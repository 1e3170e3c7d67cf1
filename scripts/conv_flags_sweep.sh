for a in "1 56 64 64 1" "8 56 64 64 1" "32 56 64 64 1" "8 28 128 128 1" "32 28 128 128 1" "1 14 256 64 4" "32 14 256 256 1" "8 7 512 128 4" "32 7 512 256 4"; do
  timeout 120 python scripts/conv_flags.py $a 2>&1 | grep -E "stream:|fused:|bit 21"
done
