#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py --dtype bf16 --steps 20 --warmup 5 > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_tc -s 3 -c 1 -o gpurun_out/prof_tc -f python bench.py --dtype bf16 --profile --steps 2 --warmup 3 > gpurun_out/ncu_tc.out 2>&1
