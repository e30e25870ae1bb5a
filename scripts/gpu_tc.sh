#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in "128 128 128 16 32 32" "300 384 512 16 32 32" "130 256 256 8 32 16" "64 256 256 8 32 128"; do
  echo "== $c" >> gpurun_out/tc_quick.log
  timeout 60 python scripts/tc_quick.py $c >> gpurun_out/tc_quick.log 2>&1
  echo "rc=$?" >> gpurun_out/tc_quick.log
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "tc" -x > gpurun_out/pytest_tc.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_tc.log
