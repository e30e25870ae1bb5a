#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python scripts/sp2_trace.py > gpurun_out/sp2_trace.log 2>&1
for c in "4096 4096 4096 16 32 32" "8192 8192 8192 16 32 32"; do
  NM_SP_PAIR=1 SP_DBGS="0 27 1024 3072 1051 3099 155 1" timeout 120 python scripts/sp_ablate.py $c 2>&1 | sed "s/^/$c: /"
done > gpurun_out/sp_pair2.log 2>&1
