"""Quick tcgen05 sanity check (run under `timeout`): one small case vs the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle
from paper_2503_01253_b200 import nmspmm, synth
m, n, k, N, M, L = [int(x) for x in (sys.argv[1:] or [128, 128, 128, 16, 32, 32])]
A = synth.integer((m, k), 1, 1); B = synth.integer((k, n), 2, 2)
vals, D = oracle.compress(synth.to_bf16_bits(B), N, M, L)
W = nmspmm.NmWeight(torch.from_numpy(oracle.bf16_to_f32(vals)).cuda().bfloat16(), torch.from_numpy(D).cuda(), k, N, M, L)
C = nmspmm.nm_spmm(torch.from_numpy(A).cuda().bfloat16(), W, out_dtype=torch.float32, math="bf16_tc")
torch.cuda.synchronize()
ref = oracle.spmm_sparse_f64(synth.to_bf16_bits(A), vals, D, k, N, M, L)
got = C.cpu().numpy().astype(np.float64)
print("plan", nmspmm.nm_plan_query(m, n, k, N, M, L, torch.bfloat16, "bf16_tc"))
print("exact", np.array_equal(got, ref), "max abs diff", np.abs(got - ref).max())
bad = np.argwhere(got != ref)
print("n bad", len(bad), bad[:10])
print(got[:4, :8]); print(ref[:4, :8])
