#!/bin/bash
# A/B of the bench's JIT tuning list on AlexNet (no baselines / CPU legs).
cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --no-baselines --no-cpu --jit-tunings "0;32,1,0,0,32,1;64,1,0,0,16,1;48,1,0,0,24,1;40,1,0,0,28,1" --out gpurun_out/bench_alexnet_t5.json > gpurun_out/bench_alexnet_t5.log 2>&1
timeout 900 python bench.py --no-baselines --no-cpu --out gpurun_out/bench_alexnet_t3.json > gpurun_out/bench_alexnet_t3.log 2>&1
