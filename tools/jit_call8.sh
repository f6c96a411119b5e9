cd $GRAFT_REPO_ROOT
TAG=r01v
timeout 900 python -m pytest tests/test_jit_gpu.py -x -q > gpurun_out/pytest_jit_$TAG.txt 2>&1
timeout 1500 python bench.py --workload resnet50_v15 --no-baselines --no-cpu --out gpurun_out/bench_resnet50_v15_$TAG.json > gpurun_out/bench_resnet50_v15_$TAG.log 2>&1
