#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tc or bf16" > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
for cfg in cfg2 cfg3_62 cfg3_75 cfg4_65b; do
  timeout 300 python bench.py --quick --dtype bf16 --steps 10 --warmup 3 --config $cfg > gpurun_out/tc_${cfg}.json 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_tc -s 3 -c 1 -o gpurun_out/prof_tc -f python bench.py --dtype bf16 --profile --steps 2 --warmup 3 > gpurun_out/ncu_tc.out 2>&1
