#!/bin/bash
# A/B of the slot kernel's full-barrier arrivals: per-thread noinc (0) vs per-warp wait_group (1)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for wa in 1 0; do
  export NM_SP_WARP_ARRIVE=$wa
  timeout 60 python scripts/tc_quick.py 1000 1024 2048 16 32 32 2>&1 | grep exact | sed "s/^/wa=$wa parity 16:32: /"
  timeout 60 python scripts/tc_quick.py 700 1280 4096 4 32 32 2>&1 | grep exact | sed "s/^/wa=$wa parity 4:32: /"
  for c in "4096 4096 4096 16 32 32" "2048 11008 4096 8 32 32" "2048 22016 8192 4 32 32" "256 22016 8192 4 32 32"; do
    SP_DBGS="0 27" timeout 60 python scripts/sp_ablate.py $c 2>&1 | sed "s/^/wa=$wa $c: /"
  done
done > gpurun_out/exp_arrive.log 2>&1
