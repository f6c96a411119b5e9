#!/bin/bash
# ncu evidence for the current build: launch list + one --set full capture of the AlexNet sconv
# launches, exported to CSV on the box (the .ncu-rep of specialised kernels is too large to bring back).
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r01}
timeout 600 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_alexnet_$TAG.csv \
  python bench.py --workload alexnet --steps 3 --warmup 1 --no-baselines --no-cpu > gpurun_out/ncu_launch_alexnet_$TAG.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none -k regex:sconv -c 4 -f \
  -o /tmp/prof_alexnet_$TAG python bench.py --workload alexnet --steps 1 --warmup 1 --no-baselines --no-cpu \
  > gpurun_out/ncu_full_alexnet_$TAG.log 2>&1
ncu -i /tmp/prof_alexnet_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_alexnet_${TAG}_raw.csv 2>&1
