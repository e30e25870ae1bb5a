#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "tc or bf16 or prepack" > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
timeout 200 python scripts/tc_trace.py > gpurun_out/trace.log 2>&1
timeout 300 python scripts/tc_ablate.py > gpurun_out/ablate_cfg2.log 2>&1
timeout 300 python scripts/tc_ablate.py 2048 22016 8192 4 32 32 > gpurun_out/ablate_cfg4.log 2>&1
