# A/B: HEAD build (acq.so) vs lazy trace timestamps + early return once the producer-done
# watermark is known (lazy.so = the tree's build); then the full GPU suite on the tree
mkdir -p gpurun_out
for l in acq lazy acq lazy; do TS_LIB_PATH=variants/$l.so timeout 400 python scripts/ab_wait.py; done > gpurun_out/ab_lazy.txt 2>&1
for l in acq lazy; do echo "== $l"; TS_LIB_PATH=variants/$l.so timeout 200 python scripts/conv_fused_diag.py 28:128:256:128:1 7:512:32:128:1:2; done >> gpurun_out/ab_lazy.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 >> gpurun_out/ab_lazy.txt
cat gpurun_out/ab_lazy.txt
