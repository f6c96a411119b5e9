#!/bin/bash
# round 2 final-build pass: GPU tests, full-size parity of every workload, every bench line, ncu evidence
cd $GRAFT_REPO_ROOT
TAG=r02l
timeout 900 python -m pytest tests/test_jit_gpu.py -x -q > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 3000 python -m pytest tests/test_bench_parity_gpu.py -q > gpurun_out/${TAG}_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/${TAG}_parity.log
for wl in resnet50 alexnet googlenet googlenet_1x1 resnet50_v15 alexnet_conv1 alexnet_convs; do
  timeout 1500 python bench.py --workload $wl --out gpurun_out/bench_${wl}_${TAG}.json > gpurun_out/${TAG}_bench_${wl}.log 2>&1
  echo "bench $wl rc=$?" >> gpurun_out/${TAG}_bench_${wl}.log
done
for wl in resnet50 googlenet alexnet; do
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
du -sh gpurun_out > gpurun_out/${TAG}_du.txt
