mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r02i.txt
B29=536870912
timeout 600 python scripts/timeline.py 1024 fused:row:row:band4:0:0:2/1:512/512 fused:row:row:band4:$B29:0:2/1:512/512 fused:row:row:band4:0:0:1/1:512/512:22,2 fused:row:row:band4:$B29:0:1/1:512/512:22,2 2>&1 | grep -v "tiles in flight" >> gpurun_out/r02i.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['value'], d['config']['chain'], 'stream', d['stream_sync_us'], 'cublas', d['cublas_us'], 'kernel', d['kernel_us'], d['clocks'])" >> gpurun_out/r02i.txt 2>&1
cat gpurun_out/r02i.txt
