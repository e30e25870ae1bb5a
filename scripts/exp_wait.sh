#!/bin/bash
mkdir -p gpurun_out
for c in "4096 4096 4096 16 32 32" "8192 8192 8192 16 32 32" "256 22016 8192 4 32 32"; do
  NM_SP_PAIR=0 SP_DBGS="0 1024 2048 3072 4096 8192 12288 27 1051 4123" timeout 300 python scripts/sp_ablate.py $c 2>&1 | sed "s/^/$c: /"
done > gpurun_out/sp_wait.log 2>&1
python scripts/prepack_sizes.py > gpurun_out/prepack_sizes.csv 2>&1
