#!/bin/bash
# Final measurement of a round: smoke, all GPU tests, the default bench (all legs), the other
# workloads, ncu launch list + full capture of the AlexNet sconv launches (exported to CSV).
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r01}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_$TAG.txt 2>&1
timeout 900 python bench.py --out gpurun_out/bench_alexnet_$TAG.json > gpurun_out/bench_alexnet_$TAG.log 2>&1
for wl in ${WLS:-}; do
timeout 1500 python bench.py --workload $wl --no-baselines --no-cpu --out gpurun_out/bench_${wl}_$TAG.json > gpurun_out/bench_${wl}_$TAG.log 2>&1
done
timeout 600 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_alexnet_$TAG.csv \
  python bench.py --workload alexnet --steps 3 --warmup 1 --no-baselines --no-cpu > gpurun_out/ncu_launch_alexnet_$TAG.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none -k regex:sconv -c 4 -f \
  -o /tmp/prof_alexnet_$TAG python bench.py --workload alexnet --steps 1 --warmup 1 --no-baselines --no-cpu \
  > gpurun_out/ncu_full_alexnet_$TAG.log 2>&1
ncu -i /tmp/prof_alexnet_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_alexnet_${TAG}_raw.csv 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference_$TAG.log 2>&1
du -sh gpurun_out
