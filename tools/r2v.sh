#!/bin/bash
# i-cache microbench + res5 A/B (bank deal, stride model, chunking, Q, mbarrier, split)
cd "$(dirname "$0")/.."
TAG=r02v
nproc > gpurun_out/${TAG}_nproc.txt; free -g >> gpurun_out/${TAG}_nproc.txt
timeout 600 python tools/icache_bench.py > gpurun_out/${TAG}_icache.jsonl 2> gpurun_out/${TAG}_icache.err
export ESCOIN_JIT_CACHE=/tmp/jit_cache; mkdir -p $ESCOIN_JIT_CACHE
T="32,1,8,3,24,1;32,1,8,3,24,1,0,0,0,0,0,0,1;32,1,8,3,24,1,0,0,0,0,0,-1;32,1,16,3,24,1;32,1,8,4,24,1;48,1,8,3,16,1;64,1,8,3,11,1;32,1,8,4,24,1,0,1;32,1,8,3,24,1,0,0,0,0,0,0,0,2;32,1,4,4,24,1"
timeout 2400 python tools/ab.py resnet50 res5a_branch2b "$T" 20 > gpurun_out/${TAG}_ab.jsonl 2> gpurun_out/${TAG}_ab.err
