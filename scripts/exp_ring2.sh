#!/bin/bash
mkdir -p gpurun_out
for cp in 1 0; do for lay in 0 1 4 5; do for st in 4 5 6; do
  timeout 10 ./scripts/ubench_ring2 $lay $st $cp || echo "cp=$cp layout $lay ST=$st: TIMEOUT/FAIL"
done; done; done > gpurun_out/ubench_ring2b.log 2>&1
