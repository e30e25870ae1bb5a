#!/bin/bash
# round-2 check: build, slot-kernel timings (before the long test run), GPU tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
for c in "4096 4096 4096 16 32 32" "2048 11008 4096 12 32 32" "2048 11008 4096 8 32 32" "2048 22016 8192 4 32 32" "256 22016 8192 4 32 32" "8192 8192 8192 16 32 32"; do
  SP_DBGS="0 1 27" timeout 120 python scripts/sp_ablate.py $c 2>&1 | sed "s/^/$c: /"
done > gpurun_out/sp_r2a.log 2>&1
for S in 2 4 6; do NM_SP_SPLIT=$S SP_DBGS="0" timeout 60 python scripts/sp_ablate.py 256 22016 8192 4 32 32 2>&1 | sed "s/^/split=$S m256: /"; done >> gpurun_out/sp_r2a.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
