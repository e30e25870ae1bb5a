#!/bin/bash
# fp32 SIMT: build, SIMT parity tests, fp32 bench variants, small shapes
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "f32 or simt or fp32 or scaled or peers or host or packed" > gpurun_out/pytest_simt.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_simt.log
timeout 600 python bench.py --steps 10 --warmup 3 --variants cfg1:f32,cfg3_62:f32,cfg3_75:f32,cfg4_13b:f32,cfg4_13b_sq:f32,cfg4_65b_sq:f32,cfg4_65b:f32,cfg4_65b_m256:f32 > gpurun_out/bench_simt.json 2> gpurun_out/bench_simt.err
SPLITS="auto 1 2" timeout 300 python scripts/small_shapes.py f32 1024 2048 > gpurun_out/small_f32.log 2>&1
