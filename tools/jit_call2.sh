cd $GRAFT_REPO_ROOT
TAG=${TAG:-r01m}
timeout 900 python -m pytest tests/test_jit_gpu.py -x -q > gpurun_out/pytest_jit_$TAG.txt 2>&1
LAYERS=conv3 NO_AUTOTUNE=1 timeout 600 python tools/jit_probe.py alexnet 0,0,0,0,0,0 128,1,8,3,8,1 96,1,8,3,8,1 64,1,8,4,16,1 64,1,4,3,16,1 64,1,16,3,16,1 > gpurun_out/jit_probe2_$TAG.txt 2>&1
timeout 900 python bench.py --workload alexnet --out gpurun_out/bench_alexnet_$TAG.json > gpurun_out/bench_alexnet_$TAG.log 2>&1
timeout 600 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_alexnet_$TAG.csv \
  python bench.py --workload alexnet --steps 3 --warmup 1 --no-baselines --no-cpu > gpurun_out/ncu_launch_alexnet_$TAG.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none -k regex:sconv -c 4 -f \
  -o /tmp/prof_alexnet_$TAG python bench.py --workload alexnet --steps 1 --warmup 1 --no-baselines --no-cpu \
  > gpurun_out/ncu_full_alexnet_$TAG.log 2>&1
ncu -i /tmp/prof_alexnet_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_alexnet_${TAG}_raw.csv 2>&1
for wl in resnet50 googlenet; do
timeout 900 python bench.py --workload $wl --no-baselines --no-cpu --out gpurun_out/bench_${wl}_$TAG.json > gpurun_out/bench_${wl}_$TAG.log 2>&1
done
du -sh gpurun_out
