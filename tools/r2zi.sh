#!/bin/bash
# res3/res4 (q43 w16 b2): bank-conflict deal, stride model, chunk sizes
cd "$(dirname "$0")/.."
TAG=r02zi
export ESCOIN_JIT_CACHE=/tmp/escoin_jit_cache; mkdir -p $ESCOIN_JIT_CACHE
timeout 900 python tools/ab.py resnet50 res3a_branch2b,res4a_branch2b "48,1,0,0,16,2;48,1,0,0,16,2,0,0,0,0,0,0,1;48,1,0,0,16,2,0,0,0,0,0,-1;48,1,16,2,16,2;48,1,12,3,16,2;48,1,4,4,16,2" 20 > gpurun_out/${TAG}_ab.jsonl 2> gpurun_out/${TAG}_ab.err
