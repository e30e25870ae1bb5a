"""Per-panel role timestamps of spmm_tc_pair_kernel CTA (0,0) (NM_TC_DBG |= 64).
Slots: 0 MMA warp b_full ok, 1 t_full ok, 2 MMAs issued; 3 gather s_full ok, 4 t_free ok, 5 arrived."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_01253_b200 import nmspmm, synth
args = [int(x) for x in sys.argv[1:]]
m, n, k, N, M, L = args[:6] if len(args) >= 6 else (128, 128, 8192, 16, 32, 32)
A = torch.from_numpy(synth.uniform((m, k), 1, 1)).cuda().bfloat16()
B = torch.from_numpy(synth.uniform((k, n), 2, 2)).cuda().bfloat16()
PW = nmspmm.nm_prepack(nmspmm.nm_compress(B, N, M, L))
C = torch.zeros(m, n, device="cuda", dtype=torch.bfloat16)
names = ["mma b_full", "mma t_full", "mma issued", "ga s_full", "ga t_free", "ga arrived"]
npan = PW.desc.npanels if hasattr(PW, "desc") else None
for base in [0, 1, 2, 24, 25, 31]:
    os.environ["NM_TC_DBG"] = str(base | 64)
    for _ in range(3):
        C.zero_()
        nmspmm.nm_spmm_prepacked(A, PW, out=C)
    torch.cuda.synchronize()
    raw = C.view(torch.int64).view(-1).cpu()
    rows = []
    for pnl in range(raw.numel() // 12):
        r = raw[pnl * 12: pnl * 12 + 6]
        if int(r[0]) == 0 and pnl > 0:
            break
        rows.append(r)
    t = torch.stack(rows)
    t = t - int(t[0][t[0] > 0].min())
    P = t.shape[0]
    print(f"== dbg {base}: {P} panels")
    print("panel " + " ".join(f"{x:>11s}" for x in names))
    for pnl in list(range(0, 4)) + list(range(P // 2, P // 2 + 4)):
        print(f"{pnl:5d} " + " ".join(f"{int(v):11d}" for v in t[pnl]))
    d = (t[-1] - t[4]) / (P - 5)
    iss = (t[4:, 2] - t[4:, 1]).float().mean()
    gat = (t[4:, 5] - t[4:, 4]).float().mean()
    print("steady clk/panel:", [round(float(x)) for x in d], f" MMA issue {iss:.0f}  gather work {gat:.0f}")
