cd $GRAFT_REPO_ROOT
TAG=r01x
timeout 900 python -m pytest tests/test_jit_gpu.py -x -q > gpurun_out/pytest_jit_$TAG.txt 2>&1
timeout 900 python bench.py --out gpurun_out/bench_alexnet_$TAG.json > gpurun_out/bench_alexnet_$TAG.log 2>&1
timeout 900 python bench.py --workload googlenet --no-baselines --no-cpu --out gpurun_out/bench_googlenet_$TAG.json > gpurun_out/bench_googlenet_$TAG.log 2>&1
