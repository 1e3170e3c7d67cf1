mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bench_parity.py -x -q -k "swiglu" 2>&1 | tail -5 > gpurun_out/r02bb.txt
timeout 900 python -c "
import sys; sys.path.insert(0, '.')
from paper_2305_13450_b200 import planner
for r in planner.sweep_swiglu(device='cuda'):
    print({k: (round(v, 1) if isinstance(v, float) else v) for k, v in r.items()})
" >> gpurun_out/r02bb.txt 2>&1
cat gpurun_out/r02bb.txt
