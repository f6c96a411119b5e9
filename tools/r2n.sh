#!/bin/bash
cd $GRAFT_REPO_ROOT
TAG=r02n
timeout 900 python -m pytest tests/test_jit_gpu.py -x -q > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
L=res2a_branch2b,res3a_branch2b,res4a_branch2b,res5a_branch2b
timeout 1500 python tools/ab.py resnet50 $L "32,1,0,0,16,2;32,1,0,0,32,1;48,1,0,0,16,2;32,1,0,0,24,1;32,1,16,3,24,1" 20 > gpurun_out/${TAG}_ab.jsonl 2> gpurun_out/${TAG}_ab.err
timeout 900 python tools/ab.py alexnet all "32,1,0,0,32,1;0" 20 > gpurun_out/${TAG}_ab_alexnet.jsonl 2>> gpurun_out/${TAG}_ab.err
