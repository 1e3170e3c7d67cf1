mkdir -p gpurun_out
for v in v1 v2 v3; do
  echo "######## $v"
  export TS_LIB_PATH=$PWD/variants/$v.so
  timeout 200 python scripts/mainloop_probe.py 1024 6144 12288 512 2 base=0 2>&1 | grep -v "tiles in flight"
  timeout 200 python scripts/mainloop_probe.py 1024 12288 6144 512 2 base=0 2>&1 | grep -v "tiles in flight"
  timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep --plan fixed 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['value'], 'stream', d['stream_sync_us'], 'cublas', d['cublas_us'], 'kernel', d['kernel_us'], d['clocks'])"
done > gpurun_out/variants_r02e.txt 2>&1
export TS_LIB_PATH=$PWD/variants/v3.so
timeout 600 python -m pytest tests/test_gpu_chain.py tests/test_gpu_bench_parity.py -x -q 2>&1 | tail -5 >> gpurun_out/variants_r02e.txt
cat gpurun_out/variants_r02e.txt
