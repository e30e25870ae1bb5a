#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
AB_TAG=base NM_LIB_PATH=$PWD/build_ab/libnmspmm_base.so python scripts/simt_ab.py
AB_TAG=new python scripts/simt_ab.py
AB_TAG=new NM_SIMT_SK=0 python scripts/simt_ab.py
done > gpurun_out/simt_ab.log 2>&1
