#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "sp_edges or (tc and sp)" > gpurun_out/pytest_sp.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sp.log
for H in 1 2; do
NM_SP_H=$H timeout 300 python scripts/sp_ablate.py > gpurun_out/sp_ablate_h$H.log 2>&1
NM_SP_H=$H timeout 300 python scripts/sp_ablate.py 2048 22016 8192 4 32 32 > gpurun_out/sp_ablate_cfg4_h$H.log 2>&1
done
