#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu4.txt 2>&1
timeout 600 python bench.py --no-baselines --no-cpu --out gpurun_out/bench_r01d.json > gpurun_out/bench_r01d.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sconv -c 4 -f -o gpurun_out/prof_r01d python bench.py --steps 1 --warmup 1 --no-baselines --no-cpu > gpurun_out/ncu_r01d.log 2>&1
