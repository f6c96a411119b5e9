#!/bin/bash
# final check of the committed tree: the default bench from an empty cubin cache (as the driver runs it), then
# the whole GPU suite (every output of every bench layer vs the oracle included) and smoke
cd "$(dirname "$0")/.."
TAG=r02zh
export ESCOIN_JIT_CACHE=/tmp/escoin_jit_cache_final; rm -rf $ESCOIN_JIT_CACHE; mkdir -p $ESCOIN_JIT_CACHE
s=$(date +%s)
timeout 2400 python bench.py --out gpurun_out/bench_resnet50_${TAG}.json > gpurun_out/${TAG}_bench_resnet50.log 2>&1
echo "bench resnet50 rc=$? wall_s=$(( $(date +%s) - s ))" >> gpurun_out/${TAG}_bench_resnet50.log
timeout 3600 python -m pytest tests/ -q -m gpu > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
