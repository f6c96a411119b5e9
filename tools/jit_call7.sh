cd $GRAFT_REPO_ROOT
TAG=${TAG:-r01t}
timeout 900 python -m pytest tests/test_jit_gpu.py -x -q > gpurun_out/pytest_jit_$TAG.txt 2>&1
NO_AUTOTUNE=1 FLUSH=1 timeout 1200 python tools/jit_probe.py alexnet 32,1,8,3,32,1,0,0 32,1,8,4,32,1,0,1 32,1,8,5,32,1,0,1 32,1,4,6,32,1,0,1 64,1,8,4,16,1,0,1 > gpurun_out/jit_probe7_$TAG.txt 2>&1
LAYERS=res2a_branch2b,res4a_branch2b NO_AUTOTUNE=1 FLUSH=1 timeout 900 python tools/jit_probe.py resnet50 64,1,8,3,16,1,0,0 64,1,8,4,16,1,0,1 32,1,8,4,32,1,0,1 > gpurun_out/jit_probe7r_$TAG.txt 2>&1
