"""Per-item pipeline stamps (clock64, diagnostic flag bit 7) of the halo conv pair: for the
first 40 items of a few CTAs, the producer claim / window issue, the MMA warp's take /
window-ready / commit, and the epilogue's take / accumulator-ready / stores-issued / end.
Prints per-phase medians in cycles and one CTA's timeline."""
import statistics
import sys
import torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts
from paper_2305_13450_b200 import _lib
hw, b = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "56:256").split(":"))
mode = sys.argv[2] if len(sys.argv) > 2 else "stream"
c = int(sys.argv[3]) if len(sys.argv) > 3 else 64
tn = int(sys.argv[4]) if len(sys.argv) > 4 else 64
halo = c == 64 and tn == 64
torch.manual_seed(0)
w1 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
w2 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
x = torch.randn(b, hw, hw, c, device="cuda").half()
ch = ts.ConvChain(x, w1, w2, tile_n=tn, cta_group=1, mode=mode, halo=halo, extra_flags=1 << 7)
ch.cs.enable_trace(148 * 40 * 12 * 8 // _lib.TRACE_REC_BYTES + 64)
for _ in range(3):
    ch()
torch.cuda.synchronize()
ch.cs._trace.zero_()
ch()
torch.cuda.synchronize()
raw = ch.cs._trace[: 148 * 40 * 12 * 8].view(torch.int64).view(148, 40, 12).cpu().tolist()
names = ["M take", "M win-ready", "M committed", "E take", "E acc-ready", "E stored", "E end",
         "P claimed", "P window-issued"]
def d(a, bb):
    return [r[bb] - r[a] for cta in raw for r in cta[2:38] if r[a] and r[bb]]
def dn(a, bb):  # next item's a minus this item's b
    out = []
    for cta in raw:
        for i in range(2, 37):
            if cta[i + 1][a] and cta[i][bb]:
                out.append(cta[i + 1][a] - cta[i][bb])
    return out
rows = [("MMA: take -> window ready", d(0, 1)), ("MMA: window ready -> committed (issue)", d(1, 2)),
        ("MMA: committed -> next take", dn(0, 2)),
        ("EPI: take -> acc ready", d(3, 4)), ("EPI: acc ready -> stores issued", d(4, 5)),
        ("EPI: stores issued -> end (bar, post)", d(5, 6)), ("EPI: end -> next take", dn(3, 6)),
        ("PROD: claimed -> window issued", d(7, 8)), ("PROD: window issued -> next claim", dn(7, 8)),
        ("item period (MMA take -> next take)", dn(0, 0)), ("item period (EPI end -> next end)", dn(6, 6)),
        ("MMA commit -> EPI acc ready", [r[4] - r[2] for cta in raw for r in cta[2:38] if r[4] and r[2]])]
print(f"conv {hw}x{hw}x{c} tile_n {tn} halo {halo} B={b} {mode}: per-item phases, cycles (median / p10 / p90 over CTAs x items 2..37)")
for name, v in rows:
    if v:
        v = sorted(v)
        print(f"  {name:42s} {statistics.median(v):8.0f} {v[len(v)//10]:8.0f} {v[9*len(v)//10]:8.0f}")
cta = raw[5]
t0 = min(x for r in cta for x in r[:9] if x)
print("CTA 5, items 0..9 (cycles from its first stamp):", " | ".join(names))
for i in range(10):
    print(f"  {i:2d} " + " ".join(f"{(cta[i][k] - t0) if cta[i][k] else -1:8d}" for k in range(9)))
# producer: claimed -> dependency waits done (slot 10, fused mode)
w = [r[10] - r[7] for cta in raw for r in cta[2:38] if r[10] and r[7]]
if w:
    w = sorted(w)
    print(f"  {'PROD: claimed -> dependency waits done':42s} {statistics.median(w):8.0f} {w[len(w)//10]:8.0f} {w[9*len(w)//10]:8.0f}")
w = [r[11] - r[1] for cta in raw for r in cta[2:38] if r[11] and r[1]]
if w:
    w = sorted(w)
    print(f"  {'MMA: first K-block (operand wait)':42s} {statistics.median(w):8.0f} {w[len(w)//10]:8.0f} {w[9*len(w)//10]:8.0f}")
