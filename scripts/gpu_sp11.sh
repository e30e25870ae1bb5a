#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "sp_edges or (tc and sp)" > gpurun_out/pytest_sp.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sp.log
for TC in 0 1; do
  NM_SP_TMA_C=$TC SP_DBGS="0" timeout 300 python scripts/sp_ablate.py 2>&1 | sed "s/^/TMAC=$TC cfg2: /" >> gpurun_out/sp11.log
  NM_SP_TMA_C=$TC SP_DBGS="0" timeout 300 python scripts/sp_ablate.py 2048 22016 8192 4 32 32 2>&1 | sed "s/^/TMAC=$TC cfg4: /" >> gpurun_out/sp11.log
  NM_SP_TMA_C=$TC SP_DBGS="0" timeout 300 python scripts/sp_ablate.py 2048 11008 4096 12 32 32 2>&1 | sed "s/^/TMAC=$TC cfg3_62: /" >> gpurun_out/sp11.log
done
SP_MASKS=0 timeout 200 python scripts/sp_trace.py > gpurun_out/sp_trace11.log 2>&1
