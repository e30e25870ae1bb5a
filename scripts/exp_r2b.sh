#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "index or prepacked_fp32 or packed_indices or tf32_prepacked" > gpurun_out/pytest_idx.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_idx.log
for shp in "4096 4096 4096 16 32 32" "256 22016 8192 4 32 32"; do
  tag=$(echo $shp | tr ' ' _)
  timeout 600 ncu --set full --clock-control none -k regex:spmm_tc_sp -s 2 -c 1 -o gpurun_out/prof_$tag -f python scripts/prof_sp.py $shp > gpurun_out/ncu_$tag.out 2>&1
  python scripts/ncu_l2.py gpurun_out/prof_$tag.ncu-rep > gpurun_out/ncu_l2_$tag.txt 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_$tag.ncu-rep > gpurun_out/ncu_sum_$tag.txt 2>&1
done
rm -f gpurun_out/*.ncu-rep
