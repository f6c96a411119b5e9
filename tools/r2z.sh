#!/bin/bash
# final pass A (this session): the default bench fresh (its compile time included), GPU unit tests, ncu of ResNet-50
cd "$(dirname "$0")/.."
TAG=r02z
export ESCOIN_JIT_CACHE=/tmp/escoin_jit_cache; mkdir -p $ESCOIN_JIT_CACHE
s=$(date +%s)
timeout 2400 python bench.py --out gpurun_out/bench_resnet50_${TAG}.json > gpurun_out/${TAG}_bench_resnet50.log 2>&1
echo "bench resnet50 rc=$? wall_s=$(( $(date +%s) - s ))" >> gpurun_out/${TAG}_bench_resnet50.log
timeout 600 python -m pytest tests/ -x -q -m gpu --deselect tests/test_bench_parity_gpu.py > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
wl=resnet50
timeout 600 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${wl}_${TAG}.csv python bench.py --workload $wl --steps 2 --warmup 1 --no-baselines --no-cpu \
  > gpurun_out/${TAG}_ncu_launch_${wl}.log 2>&1
timeout 1200 ncu --nvtx --nvtx-include "layers/" --set full --import-source on \
  --metrics sm__sass_thread_inst_executed_op_ffma_pred_on.sum,lts__t_bytes.sum --clock-control none -f -o /tmp/prof_${wl} \
  python bench.py --workload $wl --steps 2 --warmup 1 --no-baselines --no-cpu > gpurun_out/${TAG}_ncu_full_${wl}.log 2>&1
ncu -i /tmp/prof_${wl}.ncu-rep --page raw --csv > gpurun_out/prof_${wl}_${TAG}_raw.csv 2>&1
ncu -i /tmp/prof_${wl}.ncu-rep --page source --csv --print-source sass > /tmp/sass_${wl}.csv 2>&1
python tools/sass_summary.py /tmp/sass_${wl}.csv > gpurun_out/prof_${wl}_${TAG}_sass_summary.txt 2>&1
rm -f /tmp/sass_${wl}.csv
