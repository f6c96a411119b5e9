cd $GRAFT_REPO_ROOT
TAG=${TAG:-r01p}
timeout 900 python -m pytest tests/test_jit_gpu.py -x -q > gpurun_out/pytest_jit_$TAG.txt 2>&1
NO_AUTOTUNE=1 FLUSH=1 timeout 900 python tools/jit_probe.py alexnet 0 64,1,8,3,16,1 32,1,8,3,32,1 32,1,8,3,16,1 > gpurun_out/jit_probe5_$TAG.txt 2>&1
LAYERS=res2a_branch2b,res3a_branch2b,res4a_branch2b,res5a_branch2b NO_AUTOTUNE=1 FLUSH=1 timeout 900 python tools/jit_probe.py resnet50 0 64,1,8,3,16,1 > gpurun_out/jit_probe5r_$TAG.txt 2>&1
timeout 900 python bench.py --workload alexnet --out gpurun_out/bench_alexnet_$TAG.json > gpurun_out/bench_alexnet_$TAG.log 2>&1
