#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python scripts/tc_quick.py 128 128 128 16 32 32 > gpurun_out/tc_quick.log 2>&1; echo "rc=$?" >> gpurun_out/tc_quick.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tc or bf16" > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
for pr in 1 0; do for cfg in cfg2 cfg3_62 cfg3_75 cfg4_65b; do
  NM_TC_PAIR=$pr timeout 300 python bench.py --quick --dtype bf16 --steps 10 --warmup 3 --config $cfg > gpurun_out/tcp_${pr}_${cfg}.json 2>&1
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_tc_pair -s 3 -c 1 -o gpurun_out/prof_tcp -f python bench.py --dtype bf16 --profile --steps 2 --warmup 3 > gpurun_out/ncu_tcp.out 2>&1
