#!/bin/bash
# TMEM-weight slot kernel (TW, default) vs smem-image kernel (NM_SP_TW=0): parity tests, kernel times
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tc or sp or bf16 or prepacked or peers or scaled or host" > gpurun_out/pytest_tw.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tw.log
for c in "4096 4096 4096 16 32 32" "2048 11008 4096 12 32 32" "2048 11008 4096 8 32 32" "2048 22016 8192 4 32 32" "256 22016 8192 4 32 32" "8192 8192 8192 16 32 32"; do
  for tw in 1 0; do
    for h in 2 1; do
      NM_SP_TW=$tw NM_SP_H=$h SP_DBGS="0" timeout 300 python scripts/sp_ablate.py $c 2>&1 | sed "s/^/tw=$tw H=$h $c: /"
    done
  done
done > gpurun_out/tw_ab.log 2>&1
