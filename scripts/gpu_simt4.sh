#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "f32" > gpurun_out/pytest_simt.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_simt.log
for sp in 1 0; do for cfg in cfg2 cfg3_62 cfg3_75 cfg4_65b; do
  if [ $sp = 1 ]; then export NM_SIMT_SPLIT=1; else unset NM_SIMT_SPLIT; fi
  timeout 300 python bench.py --quick --steps 10 --warmup 3 --config $cfg > gpurun_out/split_${sp}_${cfg}.json 2>&1
done; done
