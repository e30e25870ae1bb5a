#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python scripts/sp_ablate.py > gpurun_out/sp_ablate5.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_sync scripts/ubench_sync.cu -lcuda && timeout 60 /tmp/ubench_sync > gpurun_out/ubench_sync.log 2>&1
