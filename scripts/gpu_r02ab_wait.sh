mkdir -p gpurun_out
for l in acq nofence acq nofence; do TS_LIB_PATH=variants/$l.so timeout 400 python scripts/ab_wait.py; done > gpurun_out/ab_wait.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 >> gpurun_out/ab_wait.txt
cat gpurun_out/ab_wait.txt
