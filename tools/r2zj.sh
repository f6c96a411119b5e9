#!/bin/bash
# res2 FFMA2: warps for the wave fill (w11: 1142 CTAs = 3.86 waves of 296 vs w12: 3.53)
cd "$(dirname "$0")/.."
TAG=r02zj
export ESCOIN_JIT_CACHE=/tmp/escoin_jit_cache; mkdir -p $ESCOIN_JIT_CACHE
timeout 600 python tools/ab.py resnet50 res2a_branch2b,res2b_branch2b "32,2,8,3,12,2,-1;32,2,8,3,11,2,-1;32,2,8,3,0,2,-1;32,2,8,3,11,2" 30 > gpurun_out/${TAG}_ab.jsonl 2> gpurun_out/${TAG}_ab.err
