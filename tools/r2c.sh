#!/bin/bash
cd $GRAFT_REPO_ROOT
L=res2a_branch2b,res3a_branch2b,res4a_branch2b,res5a_branch2b
timeout 1500 python tools/ab.py resnet50 $L "32,1,0,0,32,1,0,0,1;32,1,0,0,32,1,0,0,2;32,1,0,0,24,1,0,0,1;32,1,0,0,24,1,0,0,4;64,1,0,0,16,1,0,0,1;64,1,0,0,16,1,0,0,3;16,1,0,0,16,2,0,0,1;16,1,0,0,12,2,0,0,1;16,1,0,0,8,3,0,0,1" 20 > gpurun_out/r2c_ab.jsonl 2> gpurun_out/r2c_ab.err
