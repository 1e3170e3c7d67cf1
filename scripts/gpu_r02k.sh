# mainloop isolation: 256x256 and 256x512 pair tiles, producer-only (bit 13: no MMA),
# MMA without operand waits (bit 19), weights only (bit 15)
mkdir -p gpurun_out
for tn in 256 512; do
timeout 300 python scripts/mainloop_probe.py 4096 6144 12288 $tn 2 base=0 nomma=8192 nowait=524288 noact=32768 2>&1 | grep -v "tiles in flight" >> gpurun_out/r02k.txt
done
cat gpurun_out/r02k.txt
