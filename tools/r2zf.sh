#!/bin/bash
# GoogLeNet 1x1 group with the interpreter variants in the autotune as well
cd "$(dirname "$0")/.."
TAG=r02zf
export ESCOIN_JIT_CACHE=/tmp/escoin_jit_cache; mkdir -p $ESCOIN_JIT_CACHE
timeout 1200 python bench.py --workload googlenet_1x1 --tune-variants --no-baselines --out gpurun_out/bench_googlenet_1x1_${TAG}.json > gpurun_out/${TAG}_bench.log 2>&1
timeout 1200 python bench.py --workload googlenet --tune-variants --no-baselines --out gpurun_out/bench_googlenet_${TAG}.json > gpurun_out/${TAG}_bench_g.log 2>&1
