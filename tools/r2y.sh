#!/bin/bash
# prefetch warp (paired barrier protocol) + split channels: parity, then a short A/B with tight timeouts
cd "$(dirname "$0")/.."
TAG=r02y
timeout 300 python -m pytest tests/test_jit_gpu.py -x -q -k "parity_grid or split_channels or horizontal" > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
export ESCOIN_JIT_CACHE=/tmp/jit_cache; mkdir -p $ESCOIN_JIT_CACHE
W=0,0,0,0,0,0,0,0,0,0,1
timeout 300 python tools/ab.py resnet50 res2a_branch2b "32,1,8,3,16,2;32,1,8,3,15,2,$W;32,1,8,3,24,1,$W;32,2,8,3,11,2,$W" 20 > gpurun_out/${TAG}_ab.jsonl 2> gpurun_out/${TAG}_ab.err
timeout 400 python tools/ab.py resnet50 res4a_branch2b "48,1,8,3,16,2;48,1,8,3,15,2,$W;32,1,8,3,22,1,$W;32,2,8,3,11,1,$W" 20 >> gpurun_out/${TAG}_ab.jsonl 2>> gpurun_out/${TAG}_ab.err
K=0,0,0,0,0,0,0,0,0,0,0,-1
timeout 400 python tools/ab.py googlenet inception_5a/5x5,inception_5b/5x5,inception_4a/5x5,inception_4d/5x5 "32,1,0,0,0,1;32,1,4,2,16,1,$K;32,1,2,2,16,1,$K;16,1,2,2,16,1,$K" 20 >> gpurun_out/${TAG}_ab.jsonl 2>> gpurun_out/${TAG}_ab.err
timeout 400 python tools/ab.py googlenet_1x1 inception_5a/5x5_reduce,inception_5a/pool_proj,inception_4a/5x5_reduce,inception_5b/3x3_reduce "32,1,0,0,0,1;32,1,8,2,8,1,$K;32,1,4,2,16,1,$K;16,1,4,2,16,1,$K" 20 >> gpurun_out/${TAG}_ab.jsonl 2>> gpurun_out/${TAG}_ab.err
