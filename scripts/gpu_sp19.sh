#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
NM_SP_MC=1 timeout 120 python -m pytest tests/test_gpu_parity.py -q -x -k "sp_edges" > gpurun_out/pytest_mc_a.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mc_a.log
NM_SP_MC=1 timeout 240 python -m pytest tests/test_gpu_parity.py -q -x -k "(tc and sp) or token_tiles or tail_split" > gpurun_out/pytest_mc_b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mc_b.log
for MC in 1 0; do
for c in "4096 4096 4096 16 32 32" "2048 11008 4096 12 32 32" "2048 11008 4096 8 32 32" "2048 22016 8192 4 32 32" "8192 8192 8192 16 32 32"; do
  NM_SP_MC=$MC SP_DBGS="0" timeout 60 python scripts/sp_ablate.py $c 2>&1 | sed "s/^/MC=$MC $c: /" >> gpurun_out/sp19.log
done; done
NM_SP_MC=1 timeout 100 python scripts/sp_timeline.py > gpurun_out/timeline_mc.log 2>&1
