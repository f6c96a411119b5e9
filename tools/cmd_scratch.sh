cd $GRAFT_REPO_ROOT
for wl in alexnet resnet50 googlenet; do
t0=$(date +%s); timeout 900 python bench.py --workload $wl --no-baselines --no-cpu --out gpurun_out/bench_${wl}_g39.json > gpurun_out/bench_${wl}_g39.log 2>&1; echo "$wl $(( $(date +%s) - t0 )) s" >> gpurun_out/times_g39.txt
done
