#!/bin/bash
# prefetch-warp parity + A/B on one layer per ResNet-50 stage
cd "$(dirname "$0")/.."
TAG=r02w
timeout 900 python -m pytest tests/test_jit_gpu.py -x -q -k "parity_grid" > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
export ESCOIN_JIT_CACHE=/tmp/jit_cache; mkdir -p $ESCOIN_JIT_CACHE
W=0,0,0,0,0,0,0,0,0,0,1
timeout 900 python tools/ab.py resnet50 res2a_branch2b "32,1,8,3,16,2;32,1,8,3,16,2,$W;32,1,8,3,24,1,$W;32,2,8,3,12,2,-1;32,2,8,3,12,1,$W" 20 > gpurun_out/${TAG}_ab.jsonl 2> gpurun_out/${TAG}_ab.err
timeout 900 python tools/ab.py resnet50 res4a_branch2b "48,1,8,3,16,2;48,1,8,3,15,2,$W;32,1,8,3,22,1,$W;32,2,8,3,11,1,$W" 20 >> gpurun_out/${TAG}_ab.jsonl 2>> gpurun_out/${TAG}_ab.err
timeout 1500 python tools/ab.py resnet50 res5a_branch2b "32,1,8,3,24,1;32,1,8,3,24,1,$W;32,2,8,3,12,1,$W" 20 >> gpurun_out/${TAG}_ab.jsonl 2>> gpurun_out/${TAG}_ab.err
