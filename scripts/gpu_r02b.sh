# GEMM efficiency probe: ours (256x512 pair, two-pair cluster, 256x256) vs cuBLAS, plus
# ncu captures of cuBLAS and our kernel on GPT-3 G1 (stream mode)
mkdir -p gpurun_out
timeout 600 python scripts/gemm_eff.py 8192 8192 8192 1024 6144 12288 1024 12288 6144 18944 6144 12288 > gpurun_out/gemm_eff_r02b.txt 2>&1
cat gpurun_out/gemm_eff_r02b.txt
cat > /tmp/cub.py <<'PY'
import torch
x=torch.randn(1024,12288,device='cuda').half(); w=torch.randn(6144,12288,device='cuda').half()
for _ in range(3): y=x@w.t()
x2=torch.randn(18944,12288,device='cuda').half()
for _ in range(2): y=x2@w.t()
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none -k regex:nvjet -c 4 -o gpurun_out/cublas_r02b python /tmp/cub.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:chain_kernel -c 2 -o gpurun_out/ours_g1_r02b python scripts/gemm_eff.py prof 1024 6144 12288 512 2 2 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:chain_kernel -c 1 -o gpurun_out/ours_big_r02b python scripts/gemm_eff.py prof 18944 6144 12288 512 2 1 1 > /dev/null 2>&1
ls -la gpurun_out
