#!/bin/bash
# strong-scaling shard sizes on one GPU: each rank of a G-GPU run owns 128/G images (G = 2, 4, 8)
cd $GRAFT_REPO_ROOT
TAG=r02m
for wl in resnet50 alexnet googlenet; do
  for b in 64 32 16; do
    timeout 1200 python bench.py --workload $wl --batch $b --no-baselines --no-cpu --out gpurun_out/shard_${wl}_b${b}_${TAG}.json \
      > gpurun_out/${TAG}_${wl}_b${b}.log 2>&1
  done
done
timeout 1500 python bench.py --workload resnet50 --skew --no-baselines --no-cpu --out gpurun_out/bench_resnet50_skew_${TAG}.json > gpurun_out/${TAG}_skew.log 2>&1
timeout 2400 python bench.py --workload resnet50_convs --no-cpu --out gpurun_out/bench_resnet50_convs_${TAG}.json > gpurun_out/${TAG}_convs.log 2>&1
