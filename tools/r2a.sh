#!/bin/bash
# round 2, first GPU pass: new JIT units/cache/flushed autotune tests + ResNet-50 bench
cd $GRAFT_REPO_ROOT
nproc > gpurun_out/r2a_host.txt; lscpu | grep -E 'Model name|^CPU\(s\)' >> gpurun_out/r2a_host.txt
timeout 900 python -m pytest tests/test_jit_gpu.py -x -q > gpurun_out/r2a_jit_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2a_jit_tests.log
timeout 1500 python bench.py --steps 20 --warmup 3 --no-baselines --no-cpu --out gpurun_out/r2a_resnet.json > gpurun_out/r2a_resnet.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2a_resnet.log
