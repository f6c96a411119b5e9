#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_jit_gpu.py tests/test_dense_tc_gpu.py -x -q > gpurun_out/r2f_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2f_tests.log
L=res2a_branch2b,res3a_branch2b,res4a_branch2b,res5a_branch2b
timeout 1500 python tools/ab.py resnet50 $L "32,1,0,0,24,1;32,1,0,0,24,1,0,0,0,0,0,1;32,1,0,0,16,2;32,1,0,0,16,2,0,0,0,0,0,1;32,1,0,0,32,1;32,1,16,3,24,1;32,1,16,3,24,1,0,0,0,0,0,1" 20 > gpurun_out/r2f_ab.jsonl 2> gpurun_out/r2f_ab.err
timeout 900 python tools/ab.py alexnet all "0;32,1,0,0,32,1;32,1,0,0,24,1;32,1,4,3,24,1;32,1,0,0,16,2" 20 > gpurun_out/r2f_ab_alexnet.jsonl 2>> gpurun_out/r2f_ab.err
