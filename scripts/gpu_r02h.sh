mkdir -p gpurun_out
for v in main c9 c14; do
  echo "######## $v"
  if [ $v = main ]; then unset TS_LIB_PATH; else export TS_LIB_PATH=$PWD/variants/$v.so; fi
  timeout 200 python scripts/mainloop_probe.py 1024 6144 12288 512 2 base=0 nowait=524288 2>&1 | grep -v "tiles in flight"
  timeout 200 python scripts/mainloop_probe.py 4096 6144 12288 256 2 base=0 nowait=524288 2>&1 | grep -v "tiles in flight"
  timeout 200 python scripts/mainloop_probe.py 1024 6144 12288 384 2 base=0 2>&1 | grep -v "tiles in flight"
done > gpurun_out/r02h.txt 2>&1
unset TS_LIB_PATH
timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep --plan fixed 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['value'], 'stream', d['stream_sync_us'], 'cublas', d['cublas_us'], 'kernel', d['kernel_us'], d['clocks'])" >> gpurun_out/r02h.txt 2>&1
cat gpurun_out/r02h.txt
