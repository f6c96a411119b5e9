cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01k.txt 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_r01k.txt 2>&1
WL=alexnet TAG=r01k bash tools/gpu_bench.sh
for wl in resnet50 googlenet googlenet_1x1 resnet50_v15; do
timeout 900 python bench.py --workload $wl --no-cpu --out gpurun_out/bench_${wl}_r01k.json > gpurun_out/bench_${wl}_r01k.log 2>&1
done
