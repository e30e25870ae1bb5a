#!/bin/bash
# Full round check: build, smoke, all GPU tests, default bench, sharded path at world 1,
# launch list, ncu of the SIMT, bf16 and tf32 SpMM kernels.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --sharded --steps 10 --warmup 3 > gpurun_out/bench_sharded1.json 2> gpurun_out/bench_sharded1.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv python bench.py --quick --steps 10 --warmup 3 > gpurun_out/launches.out 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_bf16.csv python bench.py --quick --dtype bf16 --steps 10 --warmup 3 > gpurun_out/launches_bf16.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_simt -s 3 -c 1 -o gpurun_out/prof_simt -f python bench.py --profile --steps 2 --warmup 3 > gpurun_out/ncu_simt.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_tc -s 3 -c 1 -o gpurun_out/prof_tc -f python bench.py --dtype bf16 --profile --steps 2 --warmup 3 > gpurun_out/ncu_tc.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_tc_sp -s 3 -c 1 -o gpurun_out/prof_tf32 -f python scripts/tf32_profile.py > gpurun_out/ncu_tf32.out 2>&1
# summaries on the box; the .ncu-rep files are dropped so gpurun_out stays under the 64 MiB pull limit
for r in simt tc tf32; do python scripts/ncu_summary.py gpurun_out/prof_$r.ncu-rep > gpurun_out/ncu_${r}_summary.txt 2>&1; done
rm -f gpurun_out/*.ncu-rep
