#!/bin/bash
# sparse-TC parity subset + kernel times on the BASELINE bf16 shapes
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 240 python -m pytest tests/test_gpu_parity.py -q -x -k "sp_edges or (tc and sp) or token_tiles or tail_split" > gpurun_out/pytest_sp.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sp.log
for c in "4096 4096 4096 16 32 32" "2048 11008 4096 12 32 32" "2048 11008 4096 8 32 32" "2048 22016 8192 4 32 32" "8192 8192 8192 16 32 32"; do
  SP_DBGS="0" timeout 60 python scripts/sp_ablate.py $c 2>&1 | sed "s/^/$c: /"
done > gpurun_out/sp_quick.log 2>&1
