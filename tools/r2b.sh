#!/bin/bash
# round 2, second GPU pass: linked multi-unit kernels; FFMA peak; ResNet bench + ncu evidence
cd $GRAFT_REPO_ROOT
TAG=r02b
./tools/ffma_peak > gpurun_out/ffma_peak.json 2> gpurun_out/ffma_peak.err
timeout 1200 python -m pytest tests/test_jit_gpu.py "tests/test_sconv_gpu.py::test_bench_two_ranks_same_device" "tests/test_sconv_gpu.py::test_two_ranks_shard_parity" -x -q > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 1500 python bench.py --steps 50 --warmup 5 --no-cpu --out gpurun_out/bench_resnet50_${TAG}.json > gpurun_out/${TAG}_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_resnet50_$TAG.csv \
  python bench.py --steps 2 --warmup 1 --no-baselines --no-cpu > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 1200 ncu --nvtx --nvtx-include "prof/" --set full --import-source on --clock-control none -f -o /tmp/prof_resnet50_$TAG \
  python tools/prof_jit.py resnet50 res2a_branch2b,res3a_branch2b,res4a_branch2b,res5a_branch2b 0 > gpurun_out/${TAG}_ncu_full.log 2>&1
ncu -i /tmp/prof_resnet50_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_resnet50_${TAG}_raw.csv 2>&1
ncu -i /tmp/prof_resnet50_$TAG.ncu-rep --page details --csv > gpurun_out/prof_resnet50_${TAG}_details.csv 2>&1
