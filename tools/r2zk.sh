#!/bin/bash
# ncu evidence of the final build for AlexNet and GoogLeNet (launch list + one --set full capture of bench.py's eager pass)
cd "$(dirname "$0")/.."
TAG=r02zk
export ESCOIN_JIT_CACHE=/tmp/escoin_jit_cache; mkdir -p $ESCOIN_JIT_CACHE
for wl in alexnet googlenet; do
  timeout 1200 python bench.py --workload $wl --no-baselines --no-cpu --out gpurun_out/bench_${wl}_${TAG}.json > gpurun_out/${TAG}_bench_${wl}.log 2>&1
  timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${wl}_${TAG}.csv python bench.py --workload $wl --steps 2 --warmup 1 --no-baselines --no-cpu \
    > gpurun_out/${TAG}_ncu_launch_${wl}.log 2>&1
  timeout 1500 ncu --nvtx --nvtx-include "layers/" --set full --import-source on \
    --metrics sm__sass_thread_inst_executed_op_ffma_pred_on.sum,lts__t_bytes.sum --clock-control none -f -o /tmp/prof_${wl} \
    python bench.py --workload $wl --steps 2 --warmup 1 --no-baselines --no-cpu > gpurun_out/${TAG}_ncu_full_${wl}.log 2>&1
  ncu -i /tmp/prof_${wl}.ncu-rep --page raw --csv > gpurun_out/prof_${wl}_${TAG}_raw.csv 2>&1
  ncu -i /tmp/prof_${wl}.ncu-rep --page source --csv --print-source sass > /tmp/sass_${wl}.csv 2>&1
  python tools/sass_summary.py /tmp/sass_${wl}.csv > gpurun_out/prof_${wl}_${TAG}_sass_summary.txt 2>&1
  rm -f /tmp/sass_${wl}.csv
done
