#!/bin/bash
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r01}
timeout 900 python -m pytest tests/test_jit_gpu.py -x -q > gpurun_out/pytest_jit_$TAG.txt 2>&1
timeout 900 python bench.py --workload alexnet --out gpurun_out/bench_alexnet_$TAG.json > gpurun_out/bench_alexnet_$TAG.log 2>&1
for wl in ${WLS:-}; do
timeout 1200 python bench.py --workload $wl --no-baselines --no-cpu --out gpurun_out/bench_${wl}_$TAG.json > gpurun_out/bench_${wl}_$TAG.log 2>&1
done
if [ "${SWEEP:-0}" = "1" ]; then
timeout 1500 python tools/density_sweep.py > gpurun_out/density_sweep_$TAG.log 2>&1
cp gpurun_out/density_sweep.json gpurun_out/density_sweep_$TAG.json; cp gpurun_out/density_sweep.md gpurun_out/density_sweep_$TAG.md
fi
du -sh gpurun_out
