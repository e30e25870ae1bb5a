#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pair.py -q -x -k "tc or sp or bf16 or prepacked or peers or scaled or host or pair" > gpurun_out/pytest_sel.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sel.log
timeout 900 python scripts/paper_protocol.py af > gpurun_out/proto_af2.csv 2> gpurun_out/proto_af2.err
timeout 900 python bench.py --steps 10 --warmup 3 --dtype bf16 --variants cfg3_62:bf16,cfg3_75:bf16,cfg4_13b:bf16,cfg4_13b_sq:bf16,cfg4_65b_sq:bf16,cfg4_65b:bf16,cfg4_65b_m256:bf16,cfg4_13b_m256:bf16,cfg2_shard8:bf16,cfg3_75_shard8:bf16,cfg4_65b_shard8:bf16 > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err
