#!/bin/bash
# sparse-tensor-core slot path: parity first, then bf16 bench lines
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "sp_edges" > gpurun_out/pytest_sp_edges.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sp_edges.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "tc" > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
for cfg in cfg2 cfg3_62 cfg3_75 cfg4_65b; do
  timeout 300 python bench.py --quick --dtype bf16 --steps 10 --warmup 3 --config $cfg > gpurun_out/sp_${cfg}.json 2>&1
done
