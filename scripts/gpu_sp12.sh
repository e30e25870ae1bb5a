#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for NT in 160 176 192 208 224; do
  NM_SP_NT=$NT SP_DBGS="0" timeout 300 python scripts/sp_ablate.py 2>&1 | sed "s/^/NT=$NT cfg2: /" >> gpurun_out/sp12.log
  NM_SP_NT=$NT SP_DBGS="0" timeout 300 python scripts/sp_ablate.py 2048 11008 4096 12 32 32 2>&1 | sed "s/^/NT=$NT cfg3_62: /" >> gpurun_out/sp12.log
  NM_SP_NT=$NT SP_DBGS="0" timeout 300 python scripts/sp_ablate.py 2048 11008 4096 8 32 32 2>&1 | sed "s/^/NT=$NT cfg3_75: /" >> gpurun_out/sp12.log
done
