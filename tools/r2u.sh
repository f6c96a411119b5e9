#!/bin/bash
# balanced groups + auto warps + FFMA2 at 2 CTAs/SM, one layer per ResNet-50 stage
cd "$(dirname "$0")/.."
TAG=r02u
T="32,1,8,3,16,2;48,1,8,3,16,2;32,1,8,3,24,1;32,1,8,3,0,1;48,1,8,3,0,2;20,2,8,3,16,2,-1;24,2,8,3,12,2,-1;32,2,8,3,12,2,-1;24,2,8,3,0,2,-1;32,1,8,3,0,2"
timeout 2400 python tools/ab.py resnet50 res2a_branch2b,res3a_branch2b,res4a_branch2b,res5a_branch2b "$T" 20 > gpurun_out/${TAG}_ab.jsonl 2> gpurun_out/${TAG}_ab.err
