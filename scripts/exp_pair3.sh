#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in "4096 4096 4096 16 32 32" "8192 8192 8192 16 32 32"; do
  for pr in 1 0; do
  NM_SP_PAIR=$pr SP_DBGS="0 25 27 4096 4121 17 9 1 2 8" timeout 120 python scripts/sp_ablate.py $c 2>&1 | sed "s/^/pair=$pr $c: /"
  done
done > gpurun_out/sp_pair3.log 2>&1
