#!/bin/bash
# res5: two CTAs per SM (different groups) instead of one 24-warp CTA
cd "$(dirname "$0")/.."
TAG=r02zd
export ESCOIN_JIT_CACHE=/tmp/escoin_jit_cache; mkdir -p $ESCOIN_JIT_CACHE
timeout 1500 python tools/ab.py resnet50 res5a_branch2b "32,1,0,0,24,1;32,1,8,3,12,2;32,1,8,3,11,2;24,1,8,3,16,2;28,1,8,3,14,2" 20 > gpurun_out/${TAG}_ab.jsonl 2> gpurun_out/${TAG}_ab.err
