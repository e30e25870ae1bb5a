#!/bin/bash
# One gpurun call: tests, smoke, bench, ncu launch list + full capture of the top kernel.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --quick --steps 10 --warmup 3 > gpurun_out/launches.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_simt -s 3 -c 1 -o gpurun_out/prof_simt -f python bench.py --profile --steps 2 --warmup 3 > gpurun_out/ncu_full.out 2>&1
ls -la gpurun_out
