#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for H in 1 2; do
for shape in "2048 11008 4096 12 32 32" "2048 11008 4096 8 32 32" "4096 4096 4096 8 32 64" "4096 4096 4096 16 32 128"; do
  SP_DBGS="0" NM_SP_H=$H timeout 300 python scripts/sp_ablate.py $shape 2>&1 | sed "s/^/H=$H $shape: /" >> gpurun_out/sp_h.log
done
done
