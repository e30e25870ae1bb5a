#!/bin/bash
# CTA-pair slot kernel: build, its parity tests, then kernel times pair vs one-CTA (+ dbg ablations)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_pair.py -q -x > gpurun_out/pytest_pair.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pair.log
for c in "4096 4096 4096 16 32 32" "2048 11008 4096 12 32 32" "2048 11008 4096 8 32 32" "8192 8192 8192 16 32 32"; do
  for pr in 1 0; do
    NM_SP_PAIR=$pr SP_DBGS="${DBGS:-0 1 2 27}" timeout 120 python scripts/sp_ablate.py $c 2>&1 | sed "s/^/pair=$pr $c: /"
  done
done > gpurun_out/sp_pair.log 2>&1
