#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
for c in "4096 4096 4096 16 32 32" "2048 11008 4096 12 32 32" "2048 11008 4096 8 32 32" "2048 22016 8192 4 32 32" "256 22016 8192 4 32 32" "8192 8192 8192 16 32 32"; do
  SP_DBGS="0 1 27" timeout 120 python scripts/sp_ablate.py $c 2>&1 | sed "s/^/$c: /"
done > gpurun_out/sp_r2c.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tc or sp or tf32 or slot or peers or scaled or host" > gpurun_out/pytest_sp.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sp.log
