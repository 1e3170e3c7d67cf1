mkdir -p gpurun_out
(
timeout 200 python scripts/mainloop_probe.py 1024 6144 12288 512 2 base=0 2>&1 | grep -v "tiles in flight"
timeout 200 python scripts/mainloop_probe.py 1024 12288 6144 512 2 base=0 2>&1 | grep -v "tiles in flight"
timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep --plan fixed 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['value'], 'stream', d['stream_sync_us'], 'cublas', d['cublas_us'], 'kernel', d['kernel_us'], d['clocks'])"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
) > gpurun_out/r02f.txt 2>&1
cat gpurun_out/r02f.txt
