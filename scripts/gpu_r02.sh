#!/bin/bash
# Round-2 evidence: build, smoke, all GPU tests, default bench line (+ variants), bf16 headline line,
# reference arm, launch lists (fp32 / bf16), ncu --set full of the SIMT (cfg2), bf16 slot (cfg2 and
# cfg4-65B m=256) and tf32 slot (cfg2) kernels -> summaries in gpurun_out/
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --dtype bf16 --variants "" > gpurun_out/bench_bf16_headline.json 2> gpurun_out/bench_bf16_headline.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv python bench.py --quick --steps 10 --warmup 3 > gpurun_out/launches.out 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_bf16.csv python bench.py --quick --dtype bf16 --steps 10 --warmup 3 > gpurun_out/launches_bf16.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_simt -s 3 -c 1 -o gpurun_out/prof_simt -f python bench.py --profile --steps 2 --warmup 3 > gpurun_out/ncu_simt.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_tc_sp -s 2 -c 1 -o gpurun_out/prof_tc -f python scripts/prof_sp.py 4096 4096 4096 16 32 32 > gpurun_out/ncu_tc.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_tc_sp -s 2 -c 1 -o gpurun_out/prof_tc_m256 -f python scripts/prof_sp.py 256 22016 8192 4 32 32 > gpurun_out/ncu_tc_m256.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_tc_sp -s 3 -c 1 -o gpurun_out/prof_tf32 -f python scripts/tf32_profile.py > gpurun_out/ncu_tf32.out 2>&1
for r in simt tc tc_m256 tf32; do python scripts/ncu_summary.py gpurun_out/prof_$r.ncu-rep > gpurun_out/ncu_${r}_summary.txt 2>&1; done
python scripts/ncu_hot.py gpurun_out/prof_simt.ncu-rep > gpurun_out/ncu_simt_hot.txt 2>&1
rm -f gpurun_out/*.ncu-rep
