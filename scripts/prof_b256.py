"""One launch of the B=256 GPT-3 MLP plan the planner picks on most boxes (256x512 tiles on
two-pair clusters, GeMM1 in two split-K slices) after warm-up, for an ncu capture:
    ncu --set full -k regex:chain_kernel -s 3 -c 1 python scripts/prof_b256.py"""
import sys
import torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts

H, F = 12288, 6144
torch.manual_seed(0)
x = torch.randn(256, H, device="cuda").half()
w1 = (torch.randn(F, H, device="cuda") / H ** 0.5).half()
w2 = (torch.randn(H, F, device="cuda") / F ** 0.5).half()
ch = ts.MlpChain(x, w1, w2, tile_n=256, cta_group=2, prod_tile_n=512, cons_tile_n=512,
                 prod_splits=2, cluster_pairs=2)
for _ in range(4):
    ch()
torch.cuda.synchronize()
