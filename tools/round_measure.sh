#!/bin/bash
# Full measurement call: GPU tests, default bench (all legs), other workloads, ncu launch list + full capture.
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r01}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_$TAG.txt 2>&1
for wl in ${WLS:-}; do
timeout 900 python bench.py --workload $wl --out gpurun_out/bench_${wl}_$TAG.json > gpurun_out/bench_${wl}_$TAG.log 2>&1
done
WL=alexnet TAG=$TAG bash tools/gpu_bench.sh
