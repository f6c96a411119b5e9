#!/bin/bash
# round 2: the whole GPU suite (incl. 2-rank driver tests), sanitizers, skewed-sparsity load balance A/B
cd $GRAFT_REPO_ROOT
TAG=r02j
timeout 2400 python -m pytest tests -m gpu -q --deselect tests/test_bench_parity_gpu.py > gpurun_out/${TAG}_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_gpu_tests.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > gpurun_out/${TAG}_sanitizer_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_sanitizer_${tool}.log
done
L=res3a_branch2b,res4a_branch2b,res5a_branch2b
AB_SKEW=1 timeout 1200 python tools/ab.py resnet50 $L "32,1,0,0,24,1,0,0,0,0,-1;32,1,0,0,24,1,0,0,0,0,1;32,1,16,3,24,1,0,0,0,0,-1;32,1,16,3,24,1,0,0,0,0,1" 20 > gpurun_out/${TAG}_ab_skew.jsonl 2> gpurun_out/${TAG}_ab_skew.err
