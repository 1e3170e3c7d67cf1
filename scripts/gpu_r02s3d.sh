# A/B: shipped build (lazy.so) vs relaxed semaphore probes + one fence.acq_rel.gpu (rel.so, -DTS_EXP_RELAXED)
mkdir -p gpurun_out
for l in lazy rel lazy rel; do TS_LIB_PATH=variants/$l.so timeout 400 python scripts/ab_wait.py; done > gpurun_out/ab_rel.txt 2>&1
for l in lazy rel; do echo "== $l"; TS_LIB_PATH=variants/$l.so timeout 200 python scripts/conv_fused_diag.py 28:128:256:128:1 7:512:32:128:1:2; done >> gpurun_out/ab_rel.txt 2>&1
cat gpurun_out/ab_rel.txt
