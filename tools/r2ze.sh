#!/bin/bash
# res5: 32-warp CTAs (more warps share each fetched instruction), Q 26 -> 20 groups x 7 tiles = 140 CTAs
cd "$(dirname "$0")/.."
TAG=r02ze
export ESCOIN_JIT_CACHE=/tmp/escoin_jit_cache; mkdir -p $ESCOIN_JIT_CACHE
timeout 1200 python tools/ab.py resnet50 res5a_branch2b "32,1,0,0,24,1;26,1,8,3,32,1;26,1,16,3,32,1" 20 > gpurun_out/${TAG}_ab.jsonl 2> gpurun_out/${TAG}_ab.err
