cd $GRAFT_REPO_ROOT
WL=alexnet TAG=r01i bash tools/gpu_bench.sh
for wl in resnet50 googlenet googlenet_1x1 resnet50_v15; do
timeout 900 python bench.py --workload $wl --no-cpu --out gpurun_out/bench_${wl}_r01i.json > gpurun_out/bench_${wl}_r01i.log 2>&1
done
