mkdir -p gpurun_out
(
timeout 300 python scripts/mainloop_probe.py 18944 6144 12288 512 2 base=0 anorm=2048 abnorm=2560 norot=16384 nowait=524288 noact=32768
timeout 300 python scripts/mainloop_probe.py 18944 6144 12288 256 2 base=0 anorm=2048 nowait=524288 noact=32768
timeout 300 python scripts/mainloop_probe.py 1024 6144 12288 384 2 base=0 nowait=524288
timeout 300 python scripts/mainloop_probe.py 1024 6144 12288 512 2 base=0 nowait=524288
) > gpurun_out/mainloop_r02d.txt 2>&1
cat gpurun_out/mainloop_r02d.txt | grep -v "tiles in flight"
