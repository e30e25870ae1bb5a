#!/bin/bash
# compute-sanitizer over every product kernel (scripts/sanitize_run.py), one process per (tool, case);
# only our kernels are checked (torch's own fills / copies are excluded by the name filter)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
F="--kernel-name regex=nm|simt|tcs|spmm|compress|decompress|validate|unshard|peer|transpose|sp_|index|generic"
for tool in memcheck racecheck synccheck initcheck; do
  for c in format simt generic slot tf32 unshard peers at bf16simt; do
    extra=""; [ $tool = racecheck ] && extra="--racecheck-report all"
    echo "=== $tool $c"
    timeout 900 compute-sanitizer --tool $tool $extra $F --print-limit 20 python scripts/sanitize_run.py $c 2>&1 | grep -v "^$" | tail -12
  done
done > gpurun_out/sanitize.log 2>&1
