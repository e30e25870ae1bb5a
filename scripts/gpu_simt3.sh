#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "f32" > gpurun_out/pytest_simt.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_simt.log
for mode in 1 3; do
for cfg in cfg2 cfg3_62 cfg3_75 cfg4_65b; do
  NM_SIMT_MODE=$mode timeout 300 python bench.py --quick --steps 10 --warmup 3 --config $cfg > gpurun_out/simt_${mode}_${cfg}.json 2>&1
done; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_simt_pipe -s 3 -c 1 -o gpurun_out/prof_simt3 -f python bench.py --profile --steps 2 --warmup 3 --config cfg4_65b > gpurun_out/ncu_simt3.out 2>&1
