#!/bin/bash
# final pass B (this session): every other workload's bench line, full-size parity of every bench layer, smoke
cd "$(dirname "$0")/.."
TAG=r02zc
export ESCOIN_JIT_CACHE=/tmp/escoin_jit_cache; mkdir -p $ESCOIN_JIT_CACHE
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
for wl in alexnet googlenet googlenet_1x1 resnet50_v15 alexnet_conv1 alexnet_convs; do
  s=$(date +%s)
  timeout 1500 python bench.py --workload $wl --out gpurun_out/bench_${wl}_${TAG}.json > gpurun_out/${TAG}_bench_${wl}.log 2>&1
  echo "bench $wl rc=$? wall_s=$(( $(date +%s) - s ))" >> gpurun_out/${TAG}_bench_${wl}.log
done
timeout 3000 python -m pytest tests/test_bench_parity_gpu.py -q > gpurun_out/${TAG}_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/${TAG}_parity.log
