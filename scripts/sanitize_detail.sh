#!/bin/bash
mkdir -p gpurun_out
F="--kernel-name regex=nm|simt|tcs|spmm|compress|decompress|validate|unshard|peer|transpose|sp_|index|generic"
{
echo "=== memcheck slot (full)"; timeout 600 compute-sanitizer --tool memcheck $F --print-limit 5 python scripts/sanitize_run.py slot 2>&1 | head -60
echo "=== initcheck format"; timeout 600 compute-sanitizer --tool initcheck $F --print-limit 3 python scripts/sanitize_run.py format 2>&1 | head -40
echo "=== initcheck peers"; timeout 600 compute-sanitizer --tool initcheck $F --print-limit 3 python scripts/sanitize_run.py peers 2>&1 | head -40
echo "=== initcheck slot"; timeout 600 compute-sanitizer --tool initcheck $F --print-limit 3 python scripts/sanitize_run.py slot 2>&1 | head -50
echo "=== racecheck slot"; timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard $F --print-limit 6 python scripts/sanitize_run.py slot 2>&1 | head -80
echo "=== racecheck pair"; timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard $F --print-limit 6 python scripts/sanitize_run.py pair 2>&1 | head -60
} > gpurun_out/sanitize_detail.log 2>&1
