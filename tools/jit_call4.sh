cd $GRAFT_REPO_ROOT
TAG=${TAG:-r01o}
timeout 900 python -m pytest tests/test_jit_gpu.py -x -q > gpurun_out/pytest_jit_$TAG.txt 2>&1
LAYERS=conv2,conv3,conv5 NO_AUTOTUNE=1 FLUSH=1 timeout 900 python tools/jit_probe.py alexnet 0,0,0,0,0,0,0 32,1,8,3,32,1,0 16,1,8,3,32,1,0 64,1,8,3,16,1,0 32,1,8,3,32,1,-1 > gpurun_out/jit_probe4_$TAG.txt 2>&1
LAYERS=conv3 NO_AUTOTUNE=1 timeout 900 python tools/jit_probe.py alexnet 32,1,8,3,32,1,0 32,1,8,3,32,1,-1 16,1,8,3,32,1,0 > gpurun_out/jit_probe4hot_$TAG.txt 2>&1
LAYERS=res2a_branch2b,res4a_branch2b,res5a_branch2b NO_AUTOTUNE=1 FLUSH=1 timeout 900 python tools/jit_probe.py resnet50 0,0,0,0,0,0,0 32,1,8,3,32,1,0 16,1,8,3,32,1,0 > gpurun_out/jit_probe4r_$TAG.txt 2>&1
