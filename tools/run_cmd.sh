#!/bin/bash
cd $GRAFT_REPO_ROOT
TAG=${TAG:-x}
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_$TAG.txt 2>&1
if [ -n "$SWEEP" ]; then timeout 900 python tools/variant_sweep.py $SWEEP > gpurun_out/sweep_$TAG.log 2>&1; fi
for wl in ${WLS:-alexnet}; do
timeout 900 python bench.py --workload $wl --no-baselines --no-cpu --out gpurun_out/bench_${wl}_$TAG.json > gpurun_out/bench_${wl}_$TAG.log 2>&1
done
