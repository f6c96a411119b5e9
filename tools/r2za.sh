#!/bin/bash
# FFMA2 with wave-exact shapes on res4/res5 (64 pixels per warp: res5 98 warp-tiles = 7 tiles of 14 warps)
cd "$(dirname "$0")/.."
TAG=r02za
export ESCOIN_JIT_CACHE=/tmp/escoin_jit_cache; mkdir -p $ESCOIN_JIT_CACHE
timeout 1500 python tools/ab.py resnet50 res5a_branch2b "32,1,0,0,24,1;25,2,8,3,14,1,-1;25,2,8,3,7,2,-1;20,2,8,3,0,1,-1" 20 > gpurun_out/${TAG}_ab.jsonl 2> gpurun_out/${TAG}_ab.err
timeout 900 python tools/ab.py resnet50 res4a_branch2b "48,1,0,0,16,2;52,2,8,3,14,1,-1;22,2,8,3,0,1,-1" 20 >> gpurun_out/${TAG}_ab.jsonl 2>> gpurun_out/${TAG}_ab.err
timeout 600 python tools/ab.py googlenet_1x1 inception_3a/1x1,inception_4a/1x1,inception_4e/1x1,inception_5b/1x1,conv2/3x3_reduce "0;32,1,16,4,0,1;32,1,32,4,0,1;32,1,16,3,0,2;32,1,32,4,16,1,0,0,0,0,0,0,0,0,0,0,0,-1" 20 >> gpurun_out/${TAG}_ab.jsonl 2>> gpurun_out/${TAG}_ab.err
