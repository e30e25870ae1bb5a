#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "tc or bf16" -x > gpurun_out/pytest_tc.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_tc.log
timeout 300 python bench.py --dtype bf16 --steps 20 --warmup 5 --quick > gpurun_out/bench_bf16_quick.json 2>&1
timeout 300 python bench.py --dtype bf16 --steps 20 --warmup 5 --quick --config cfg4_65b >> gpurun_out/bench_bf16_quick.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_tc -s 3 -c 1 -o gpurun_out/prof_tc -f python bench.py --dtype bf16 --profile --steps 2 --warmup 3 > gpurun_out/ncu_tc.out 2>&1
