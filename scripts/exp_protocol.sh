#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python scripts/paper_protocol.py v123 > gpurun_out/proto_v123.csv 2> gpurun_out/proto_v123.err
timeout 1500 python scripts/paper_protocol.py af > gpurun_out/proto_af.csv 2> gpurun_out/proto_af.err
timeout 2400 python scripts/llama_dataset.py > gpurun_out/llama_dataset.csv 2> gpurun_out/llama_dataset.err
python scripts/llama_summary.py gpurun_out/llama_dataset.csv > gpurun_out/llama_summary.txt 2>&1
