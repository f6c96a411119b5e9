#!/bin/bash
cd $GRAFT_REPO_ROOT
TAG=${TAG:-x}
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_$TAG.txt 2>&1
timeout 600 python tools/variant_sweep.py ${SWEEP:-alexnet} > gpurun_out/sweep_$TAG.log 2>&1
timeout 600 python bench.py --no-baselines --no-cpu --out gpurun_out/bench_$TAG.json > gpurun_out/bench_$TAG.log 2>&1
