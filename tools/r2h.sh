#!/bin/bash
cd $GRAFT_REPO_ROOT
TAG=r02h
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > gpurun_out/${TAG}_sanitizer_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_sanitizer_${tool}.log
done
L=res2a_branch2b,res3a_branch2b,res4a_branch2b,res5a_branch2b
timeout 1500 python tools/ab.py resnet50 $L "32,1,0,0,24,1;48,1,0,0,24,1;40,1,0,0,24,1;48,1,0,0,20,1;64,1,0,0,20,1;48,1,16,3,24,1;48,1,0,0,16,2" 20 > gpurun_out/${TAG}_ab.jsonl 2> gpurun_out/${TAG}_ab.err
timeout 900 python tools/ab.py alexnet all "32,1,0,0,32,1;48,1,0,0,24,1;40,1,0,0,24,1;64,1,0,0,20,1;48,1,0,0,20,1" 20 > gpurun_out/${TAG}_ab_alexnet.jsonl 2>> gpurun_out/${TAG}_ab.err
