"""Per-CTA timeline of spmm_tc_sp_kernel (NM_SP_DBG=256): start/end %globaltimer, SM, stages.
Usage: sp_timeline.py [m n k N M L]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
from paper_2503_01253_b200 import nmspmm, synth
m, n, k, N, M, L = [int(x) for x in (sys.argv[1:] or [4096, 4096, 4096, 16, 32, 32])]
A = torch.from_numpy(synth.uniform((m, k), 1, 1)).cuda().bfloat16()
B = torch.from_numpy(synth.uniform((k, n), 2, 2)).cuda().bfloat16()
W = nmspmm.nm_compress(B, N, M, L)
PW = nmspmm.nm_prepack(W)
C = torch.zeros(m, n, device="cuda", dtype=torch.bfloat16)
os.environ["NM_SP_DBG"] = "256"
for _ in range(3):
    nmspmm.nm_spmm_prepacked(A, PW, out=C)
torch.cuda.synchronize()
plan = nmspmm.nm_plan_query(m, n, k, N, M, L, torch.bfloat16, "bf16_tc")
ntiles = ((n + plan["bn"] - 1) // plan["bn"]) * ((m + plan["bm"] - 1) // plan["bm"])
raw = C.view(-1).view(torch.int64)[: 4 * (ntiles + 200)].view(-1, 4).cpu().numpy()
raw = raw[raw[:, 1] > 0]
t0 = raw[:, 0].min()
st, en, sm, ns = (raw[:, 0] - t0) / 1e3, (raw[:, 1] - t0) / 1e3, raw[:, 2], raw[:, 3]
dur = en - st
print(f"CTAs {len(raw)}  kernel span {en.max():.1f} us  CTA duration mean {dur.mean():.1f} min {dur.min():.1f} max {dur.max():.1f} us")
print(f"stages mean {ns.mean():.1f} min {ns.min()} max {ns.max()};  us per stage: mean {np.mean(dur / np.maximum(ns, 1)):.3f}")
order = np.argsort(st)
for i in list(range(0, 6)) + list(range(140, 156)) + list(range(len(raw) - 6, len(raw))):
    if i < len(raw):
        j = order[i]
        print(f"  #{i:4d} start {st[j]:8.1f} end {en[j]:8.1f} dur {dur[j]:6.1f} sm {sm[j]:3d} stages {ns[j]}")
# idle gaps per SM
gaps = []
for s_ in np.unique(sm):
    idx = np.where(sm == s_)[0]
    o = idx[np.argsort(st[idx])]
    for a, b in zip(o[:-1], o[1:]):
        gaps.append(st[b] - en[a])
if gaps:
    print(f"per-SM gap between consecutive CTAs: mean {np.mean(gaps):.2f} us max {np.max(gaps):.2f}")
print(f"SMs used {len(np.unique(sm))}, busy fraction {dur.sum() / (len(np.unique(sm)) * en.max()):.3f}")
