"""Per-CTA timeline of spmm_tc_sp_kernel (NM_SP_DBG=256 | mask): %globaltimer start/end, SM,
stages, and clock64 at start / accumulators complete / end -> the SM clock each CTA ran at, the
main-loop clocks per stage and the fixed (prologue + epilogue) cost per CTA.  The C stores are
skipped in this mode.  Usage: sp_timeline.py [m n k N M L], SP_MASKS="0 17 27 2" (extra NM_SP_DBG bits:
1 no gathers, 2 no MMAs, 16 no weights, 17 MMA only, 27 sync skeleton)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2503_01253_b200 import nmspmm, synth

m, n, k, N, M, L = [int(x) for x in (sys.argv[1:] or [4096, 4096, 4096, 16, 32, 32])]
A = torch.from_numpy(synth.uniform((m, k), 1, 1)).cuda().bfloat16()
B = torch.from_numpy(synth.uniform((k, n), 2, 2)).cuda().bfloat16()
W = nmspmm.nm_compress(B, N, M, L)
PW = nmspmm.nm_prepack(W)
C = torch.zeros(m, n, device="cuda", dtype=torch.bfloat16)
names = {0: "full", 17: "MMA only", 27: "sync skeleton", 2: "no MMA", 1: "no gather", 16: "no weights"}
for mask in [int(x) for x in os.environ.get("SP_MASKS", "0 17 27 2").split()]:
    os.environ["NM_SP_DBG"] = str(256 | mask)
    C.zero_()
    for _ in range(3):
        nmspmm.nm_spmm_prepacked(A, PW, out=C)
    torch.cuda.synchronize()
    raw = C.view(-1).view(torch.int64)[: 8 * 4096].view(-1, 8).cpu().numpy()
    raw = raw[raw[:, 1] > 0]
    t0 = raw[:, 0].min()
    st, en, sm, ns = (raw[:, 0] - t0) / 1e3, (raw[:, 1] - t0) / 1e3, raw[:, 2], raw[:, 3]
    c0, ca, ce = raw[:, 4], raw[:, 5], raw[:, 6]
    dur = en - st
    ghz = (ce - c0) / np.maximum(raw[:, 1] - raw[:, 0], 1)
    loop = (ca - c0) / np.maximum(ns, 1)
    epi_us = (ce - ca) / ghz / 1e3
    print(f"== {m}x{n}x{k} {N}:{M} L{L} mask {mask} ({names.get(mask, '')}): CTAs {len(raw)}, kernel span {en.max():.1f} us, "
          f"SM clock {np.median(ghz):.3f} GHz (min {ghz.min():.3f})")
    print(f"   CTA duration mean {dur.mean():.1f} us (min {dur.min():.1f} max {dur.max():.1f}); stages mean {ns.mean():.1f} "
          f"(min {ns.min()} max {ns.max()})")
    print(f"   start -> accumulators complete: {np.median(loop):.0f} clk per stage (median over CTAs; incl. prologue); "
          f"accumulators -> end (epilogue): {np.median(epi_us):.2f} us")
    gaps = []
    for s_ in np.unique(sm):
        idx = np.where(sm == s_)[0]
        o = idx[np.argsort(st[idx])]
        for a, b in zip(o[:-1], o[1:]):
            gaps.append(st[b] - en[a])
    if gaps:
        print(f"   per-SM gap between consecutive CTAs: mean {np.mean(gaps):.2f} us max {np.max(gaps):.2f}; "
              f"SMs used {len(np.unique(sm))}, busy fraction {dur.sum() / (len(np.unique(sm)) * en.max()):.3f}")
os.environ.pop("NM_SP_DBG", None)
