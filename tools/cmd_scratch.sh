cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_g60.txt 2>&1
for wl in alexnet resnet50 googlenet googlenet_1x1 resnet50_v15; do
t0=$(date +%s); timeout 900 python bench.py --workload $wl --no-baselines --no-cpu --out gpurun_out/bench_${wl}_g60.json > gpurun_out/bench_${wl}_g60.log 2>&1; echo "$wl $(( $(date +%s) - t0 )) s" >> gpurun_out/times_g60.txt
done
