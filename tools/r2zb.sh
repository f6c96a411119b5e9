#!/bin/bash
# FFMA2 wave-exact shapes WITH the instruction-prefetch pass on res5/res4 (r02za ran them without)
cd "$(dirname "$0")/.."
TAG=r02zb
export ESCOIN_JIT_CACHE=/tmp/escoin_jit_cache; mkdir -p $ESCOIN_JIT_CACHE
timeout 1200 python tools/ab.py resnet50 res5a_branch2b "32,1,0,0,24,1;25,2,8,3,14,1;20,2,8,3,20,1;32,2,8,3,12,1" 20 > gpurun_out/${TAG}_ab.jsonl 2> gpurun_out/${TAG}_ab.err
timeout 600 python tools/ab.py resnet50 res4a_branch2b "48,1,0,0,16,2;52,2,8,3,14,1;22,2,8,3,17,1" 20 >> gpurun_out/${TAG}_ab.jsonl 2>> gpurun_out/${TAG}_ab.err
