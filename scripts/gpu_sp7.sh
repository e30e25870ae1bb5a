#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "sp_edges" > gpurun_out/pytest_sp.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sp.log
for HN in "2 192" "2 160" "2 128" "2 224" "1 256" "1 192" "1 128"; do
  set -- $HN
  NM_SP_H=$1 NM_SP_NT=$2 SP_DBGS="0 2" timeout 300 python scripts/sp_ablate.py 2>&1 | sed "s/^/H=$1 NT=$2 cfg2: /" >> gpurun_out/sp_nt.log
  NM_SP_H=$1 NM_SP_NT=$2 SP_DBGS="0" timeout 300 python scripts/sp_ablate.py 2048 22016 8192 4 32 32 2>&1 | sed "s/^/H=$1 NT=$2 cfg4: /" >> gpurun_out/sp_nt.log
done
