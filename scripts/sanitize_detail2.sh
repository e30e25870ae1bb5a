#!/bin/bash
mkdir -p gpurun_out
F="--kernel-name regex=nm|simt|tcs|spmm|compress|decompress|validate|unshard|peer|transpose|sp_|index|generic"
{
for c in format slot tf32 peers pair; do
  echo "=== initcheck (all kernels tracked) $c"; timeout 900 compute-sanitizer --tool initcheck --print-limit 5 python scripts/sanitize_run.py $c 2>&1 | grep -v "Host Frame" | head -30
done
for c in slot pair tf32; do
  echo "=== racecheck hazard kinds $c"
  timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard $F --print-limit 0 python scripts/sanitize_run.py $c 2>&1 | grep -E "Potential|at .* in .*:[0-9]+" | sed -E 's/0x[0-9a-f]+//g; s/block \([0-9,]+\)//; s/Thread \([0-9,]+\)//g' | sort | uniq -c | sort -rn | head -20
done
echo "=== memcheck slot host backtrace"; timeout 600 compute-sanitizer --tool memcheck $F --print-limit 5 python scripts/sanitize_run.py slot 2>&1 | head -30
} > gpurun_out/sanitize_detail2.log 2>&1
