#!/bin/bash
cd $GRAFT_REPO_ROOT
TAG=r02g
timeout 600 python -m pytest tests/test_jit_gpu.py -x -q > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
for wl in resnet50 alexnet googlenet googlenet_1x1 resnet50_v15 alexnet_conv1; do
  timeout 1500 python bench.py --workload $wl --out gpurun_out/bench_${wl}_${TAG}.json > gpurun_out/${TAG}_bench_${wl}.log 2>&1
  echo "bench $wl rc=$?" >> gpurun_out/${TAG}_bench_${wl}.log
done
timeout 2400 python -m pytest tests/test_bench_parity_gpu.py -x -q > gpurun_out/${TAG}_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/${TAG}_parity.log
