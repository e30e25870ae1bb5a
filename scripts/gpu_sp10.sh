#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for HN in "2 160" "2 224" "2 128" "1 192"; do
  set -- $HN
  NM_SP_H=$1 NM_SP_NT=$2 SP_DBGS="0" timeout 300 python scripts/sp_ablate.py 2>&1 | sed "s/^/H=$1 NT=$2 cfg2: /" >> gpurun_out/sp10.log
  NM_SP_H=$1 NM_SP_NT=$2 SP_DBGS="0" timeout 300 python scripts/sp_ablate.py 2048 22016 8192 4 32 32 2>&1 | sed "s/^/H=$1 NT=$2 cfg4: /" >> gpurun_out/sp10.log
  NM_SP_H=$1 NM_SP_NT=$2 SP_DBGS="0" timeout 300 python scripts/sp_ablate.py 2048 11008 4096 12 32 32 2>&1 | sed "s/^/H=$1 NT=$2 cfg3_62: /" >> gpurun_out/sp10.log
  NM_SP_H=$1 NM_SP_NT=$2 SP_DBGS="0" timeout 300 python scripts/sp_ablate.py 2048 11008 4096 8 32 32 2>&1 | sed "s/^/H=$1 NT=$2 cfg3_75: /" >> gpurun_out/sp10.log
done
for H in 1 2; do NM_SP_H=$H SP_DBGS="0" timeout 300 python scripts/sp_ablate.py 2048 11008 4096 8 32 32 2>&1 | sed "s/^/H=$H default cfg3_75: /" >> gpurun_out/sp10.log; done
