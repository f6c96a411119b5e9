#!/bin/bash
# One GPU session: bench JSON, ncu launch list, ncu --set full of the sconv kernels.
cd $GRAFT_REPO_ROOT
WL=${WL:-alexnet}
TAG=${TAG:-r01}
nproc > gpurun_out/host_${TAG}.txt; lscpu | grep -E 'Model name' >> gpurun_out/host_${TAG}.txt
timeout 600 python bench.py --workload $WL --out gpurun_out/bench_${WL}_${TAG}.json > gpurun_out/bench_${WL}_${TAG}.log 2>&1
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${WL}_${TAG}.csv \
  python bench.py --workload $WL --steps 3 --warmup 1 --no-baselines --no-cpu > gpurun_out/ncu_launch_${WL}_${TAG}.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:sconv -c ${NCU_COUNT:-4} -f \
  -o gpurun_out/prof_${WL}_${TAG} python bench.py --workload $WL --steps 1 --warmup 1 --no-baselines --no-cpu \
  > gpurun_out/ncu_full_${WL}_${TAG}.log 2>&1
fi
