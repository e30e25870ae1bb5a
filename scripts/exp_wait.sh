#!/bin/bash
mkdir -p gpurun_out
for c in "4096 4096 4096 16 32 32" "8192 8192 8192 16 32 32" "256 22016 8192 4 32 32" "256 13824 5120 4 32 32" "2048 22016 8192 4 32 32"; do
  NM_SP_PAIR=0 SP_DBGS="0 16384 1024 2048 3072 4096 8192 12288 27" timeout 300 python scripts/sp_ablate.py $c 2>&1 | sed "s/^/$c: /"
done > gpurun_out/sp_wait.log 2>&1
python scripts/prepack_sizes.py > gpurun_out/prepack_sizes.csv 2>&1
timeout 900 python scripts/sp_split_probe.py > gpurun_out/sp_split_probe.log 2>&1
python scripts/mc_probe.py > gpurun_out/mc_probe.log 2>&1
./scripts/ubench_sp_ts > gpurun_out/ubench_sp_ts.log 2>&1
