import sys
import torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts
torch.manual_seed(0)
m, k, n1, n2 = 512, 1024, 1024, 2048
x = torch.randn(m, k, device="cuda").half()
w1 = (torch.randn(n1, k, device="cuda") / k ** 0.5).half()
w2 = (torch.randn(n2, n1, device="cuda") / n1 ** 0.5).half()
h = torch.nn.functional.gelu(x.float() @ w1.float().t(), approximate="tanh").half()
y = h.float() @ w2.float().t()
p0 = h[256:512, :512].float() @ w2[:512, :512].float().t()
p1 = h[256:512, 512:].float() @ w2[:512, 512:].float().t()
for name, fl in [("tail2", 0), ("tail2_noredmma", 1 << 30)]:
    ch = ts.MlpChain(x, w1, w2, tile_n=256, cta_group=2, prod_tile_n=512, cons_tile_n=512,
                     extra_flags=fl, cons_tail=(4, 2))
    ch.cs.stages[1].ws.fill_(0.0)
    ch()
    torch.cuda.synchronize()
    d = ch.y[256:512, :512].float()
    print(name, "y-(p0+p1)", (d - p0 - p1).abs().max().item(), " y-p1", (d - p1).abs().max().item(),
          " y-p0", (d - p0).abs().max().item())
    diff = d - p0 - p1
    print("   diff row0 cols0..5", diff[0, :6].cpu().numpy().round(2), " row200", diff[200, :6].cpu().numpy().round(2))
