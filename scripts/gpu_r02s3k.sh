# A/B: HEAD build (base.so) vs halo-conv waits probing up to five producer tiles per round
# trip (batch.so = the tree's build); then the halo-conv GPU tests on the tree
mkdir -p gpurun_out
for l in base batch base batch; do TS_LIB_PATH=variants/$l.so timeout 300 python scripts/conv_halo_quick.py 56:1 56:8 56:32 56:128 56:256 224:8 224:32 2>&1 | sed "s/^/$l /"; done > gpurun_out/ab_halo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_conv_halo.py tests/test_gpu_bench_parity.py -m gpu -x -q 2>&1 | tail -3 >> gpurun_out/ab_halo.txt
cat gpurun_out/ab_halo.txt
