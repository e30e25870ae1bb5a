"""Per-panel cost of spmm_tc_pair_kernel stages at one wave: tc_ablate2.py"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_01253_b200 import nmspmm, synth
for (m, n, k, N, M, L) in [(128, 128, 32768, 16, 32, 32), (512, 4736, 32768, 16, 32, 32), (4096, 4096, 4096, 16, 32, 32)]:
    A = torch.from_numpy(synth.uniform((m, k), 1, 1)).cuda().bfloat16()
    B = torch.from_numpy(synth.uniform((k, n), 2, 2)).cuda().bfloat16()
    W = nmspmm.nm_compress(B, N, M, L)
    PW = nmspmm.nm_prepack(W)
    C = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    plan = nmspmm.nm_plan_query(m, n, k, N, M, L, torch.bfloat16, "bf16_tc")
    npan = k // plan.get("bk", 128) if isinstance(plan, dict) else k // 128
    for dbg in [0, 1, 2, 7, 31]:
        os.environ["NM_TC_DBG"] = str(dbg)
        for _ in range(2):
            nmspmm.nm_spmm_prepacked(A, PW, out=C)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(5):
            nmspmm.nm_spmm_prepacked(A, PW, out=C)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        waves = -(-((m + 127) // 128) * ((n + 127) // 128) // 148)
        print(f"{m}x{n}x{k} dbg={dbg:2d} {ms*1e3:9.1f} us  waves={waves} clk/panel={ms*1e-3*1.965e9/waves/npan:8.0f}", flush=True)
    print(plan)
