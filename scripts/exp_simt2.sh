#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "f32 or simt or fp32 or scaled or peers or host or packed or split" > gpurun_out/pytest_simt.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_simt.log
AB_TAG=new python scripts/simt_ab.py > gpurun_out/simt_ab3.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --variants cfg1:f32,cfg3_62:f32,cfg3_75:f32,cfg4_13b:f32,cfg4_13b_sq:f32,cfg4_65b_sq:f32,cfg4_65b:f32,cfg4_65b_m256:f32 > gpurun_out/bench_simt.json 2> gpurun_out/bench_simt.err
