mkdir -p gpurun_out
cat > /tmp/conv_prof.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts
torch.manual_seed(0)
for hw, c, b, kw in ((56, 64, 128, dict(tile_n=64, cta_group=1, halo=True)),
                     (56, 64, 128, dict(tile_n=64, cta_group=1)),
                     (28, 128, 128, dict(tile_n=128, cta_group=1))):
    x = torch.randn(b, hw, hw, c, device="cuda").half()
    w1 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
    w2 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
    ch = ts.ConvChain(x, w1, w2, **kw)
    for _ in range(2):
        ch()
    torch.cuda.synchronize()
PY
timeout 900 ncu --set full --clock-control none -k regex:chain_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/conv_halo56 python /tmp/conv_prof.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:chain_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/conv_im2col56 python /tmp/conv_prof.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:chain_kernel --launch-skip 5 --launch-count 1 -o gpurun_out/conv_im2col28 python /tmp/conv_prof.py > /dev/null 2>&1
for f in conv_halo56 conv_im2col56 conv_im2col28; do echo "=== $f"; python scripts/ncu_summary.py gpurun_out/$f.ncu-rep; done > gpurun_out/r02aa.txt 2>&1
cat gpurun_out/r02aa.txt
