#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "f32 or simt or fp32 or scaled or peers or host or packed or stream_k" > gpurun_out/pytest_simt.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_simt.log
AB_TAG=base NM_LIB_PATH=$PWD/build_ab/libnmspmm_base.so python scripts/simt_ab.py > gpurun_out/simt_ab.log 2>&1
AB_TAG=new python scripts/simt_ab.py >> gpurun_out/simt_ab.log 2>&1
AB_TAG=new NM_SIMT_SK=0 python scripts/simt_ab.py >> gpurun_out/simt_ab.log 2>&1
