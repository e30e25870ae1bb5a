#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for H in 1 2; do
NM_SP_H=$H timeout 600 ncu --set full --clock-control none -k regex:spmm_tc_sp -s 3 -c 1 -o gpurun_out/prof_sp_h$H -f python bench.py --dtype bf16 --profile --steps 2 --warmup 3 > gpurun_out/ncu_sp_h$H.out 2>&1
done
