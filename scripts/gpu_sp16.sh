#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
NM_SP_PAIR=1 timeout 90 python -m pytest tests/test_gpu_parity.py -q -x -k "sp_edges" > gpurun_out/pytest_sp2a.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sp2a.log
NM_SP_PAIR=1 timeout 180 python -m pytest tests/test_gpu_parity.py -q -x -k "(tc and sp) or token_tiles" > gpurun_out/pytest_sp2b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sp2b.log
for PR in 1; do
for c in "4096 4096 4096 16 32 32" "2048 11008 4096 12 32 32" "2048 11008 4096 8 32 32"; do
  NM_SP_PAIR=$PR SP_DBGS="0" timeout 60 python scripts/sp_ablate.py $c 2>&1 | sed "s/^/PAIR=$PR $c: /" >> gpurun_out/sp16.log
done; done
