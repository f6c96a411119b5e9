cd $GRAFT_REPO_ROOT
TAG=${TAG:-r01n}
timeout 900 python -m pytest tests/test_jit_gpu.py -x -q > gpurun_out/pytest_jit_$TAG.txt 2>&1
LAYERS=conv2,conv3,conv5 NO_AUTOTUNE=1 FLUSH=1 timeout 900 python tools/jit_probe.py alexnet 0,0,0,0,0,0,0 0,0,0,0,0,0,-1 64,1,8,3,8,2,0 32,1,8,3,16,1,0 > gpurun_out/jit_probe3_$TAG.txt 2>&1
LAYERS=conv3 NO_AUTOTUNE=1 timeout 900 python tools/jit_probe.py alexnet 0,0,0,0,0,0,0 0,0,0,0,0,0,-1 > gpurun_out/jit_probe3hot_$TAG.txt 2>&1
LAYERS=res5a_branch2b,res4a_branch2b NO_AUTOTUNE=1 FLUSH=1 timeout 900 python tools/jit_probe.py resnet50 0,0,0,0,0,0,0 0,0,0,0,0,0,-1 32,1,8,3,16,1,0 > gpurun_out/jit_probe3r_$TAG.txt 2>&1
