#!/bin/bash
mkdir -p gpurun_out
timeout 120 ./scripts/ubench_ring > gpurun_out/ubench_ring.log 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SP_DBGS="0 1 2 16 19 27 155" timeout 120 python scripts/sp_ablate.py 4096 4096 4096 16 32 32 > gpurun_out/sp_ablate_cfg2.log 2>&1
