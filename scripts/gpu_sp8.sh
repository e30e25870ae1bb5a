#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "sp_edges or (tc and sp)" > gpurun_out/pytest_sp.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sp.log
for TR in 0 16 32; do for H in 1 2; do
  NM_SP_TMA_ROWS=$TR NM_SP_H=$H SP_DBGS="0" timeout 300 python scripts/sp_ablate.py 2>&1 | sed "s/^/TR=$TR H=$H cfg2: /" >> gpurun_out/sp_tr.log
  NM_SP_TMA_ROWS=$TR NM_SP_H=$H SP_DBGS="0" timeout 300 python scripts/sp_ablate.py 2048 22016 8192 4 32 32 2>&1 | sed "s/^/TR=$TR H=$H cfg4: /" >> gpurun_out/sp_tr.log
done; done
