#!/bin/bash
# AlexNet conv2-5 with FFMA2 shapes (conv2 is AlexNet's dominant kernel)
cd "$(dirname "$0")/.."
TAG=r02zl
export ESCOIN_JIT_CACHE=/tmp/escoin_jit_cache; mkdir -p $ESCOIN_JIT_CACHE
timeout 900 python tools/ab.py alexnet conv2,conv3,conv5 "32,1,0,0,32,1;32,2,4,4,12,1,-1;24,2,4,4,16,1,-1;32,2,0,0,12,2,-1;16,2,0,0,16,2,-1" 20 > gpurun_out/${TAG}_ab.jsonl 2> gpurun_out/${TAG}_ab.err
