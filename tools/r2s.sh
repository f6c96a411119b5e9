#!/bin/bash
# FFMA2 slot-pair A/B on one layer per ResNet-50 stage (flushed L2, bitwise vs the first tuning)
cd "$(dirname "$0")/.."
T="32,1,8,3,16,2;48,1,8,3,16,2;32,1,8,3,24,1;32,2,8,3,16,1;32,2,8,3,8,2;48,2,8,3,12,1;64,2,8,3,8,1;16,2,8,3,16,2;24,2,8,3,16,1;32,2,8,3,16,1,-1"
python tools/ab.py resnet50 res2a_branch2b,res3a_branch2b,res4a_branch2b,res5a_branch2b "$T" 20 > gpurun_out/r02s_ab.jsonl 2> gpurun_out/r02s_ab.err
