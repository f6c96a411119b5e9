#!/bin/bash
# GoogLeNet 5x5 layers (16-48 input channels): whole-channel chunks (one load, one barrier) vs the default
cd "$(dirname "$0")/.."
TAG=r02zg
export ESCOIN_JIT_CACHE=/tmp/escoin_jit_cache; mkdir -p $ESCOIN_JIT_CACHE
L=inception_3a/5x5,inception_4a/5x5,inception_4b/5x5,inception_4c/5x5,inception_4d/5x5,inception_5a/5x5,inception_5b/5x5
timeout 900 python tools/ab.py googlenet $L "0;32,1,16,2,0,1;16,1,16,2,0,1;32,1,8,2,0,2;16,1,16,2,8,2;32,1,48,2,0,1;16,1,8,3,0,2" 20 > gpurun_out/${TAG}_ab.jsonl 2> gpurun_out/${TAG}_ab.err
