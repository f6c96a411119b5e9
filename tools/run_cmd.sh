#!/bin/bash
# GPU round trip: gpu tests, optional variant sweeps, bench per workload.
# TAG names the outputs; SWEEP = workloads to sweep; SWEEP2 = workloads to
# sweep again with ESCOIN_STAGES=2; WLS = bench workloads.
cd $GRAFT_REPO_ROOT
TAG=${TAG:-x}
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_$TAG.txt 2>&1
if [ -n "$SWEEP" ]; then timeout 900 python tools/variant_sweep.py $SWEEP > gpurun_out/sweep_$TAG.log 2>&1; cp gpurun_out/variant_sweep.json gpurun_out/variant_sweep_$TAG.json; fi
if [ -n "$SWEEP2" ]; then ESCOIN_STAGES=2 timeout 900 python tools/variant_sweep.py $SWEEP2 > gpurun_out/sweep_${TAG}_ns2.log 2>&1; cp gpurun_out/variant_sweep.json gpurun_out/variant_sweep_${TAG}_ns2.json; fi
for wl in ${WLS:-alexnet}; do
timeout 900 python bench.py --workload $wl --no-baselines --no-cpu --out gpurun_out/bench_${wl}_$TAG.json > gpurun_out/bench_${wl}_$TAG.log 2>&1
done
