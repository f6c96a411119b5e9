cd $GRAFT_REPO_ROOT
TAG=${TAG:-r01r}
NO_AUTOTUNE=1 FLUSH=1 timeout 1200 python tools/jit_probe.py alexnet 32,1,8,3,32,1 32,1,16,2,32,1 32,1,12,3,32,1 32,1,4,4,32,1 32,1,8,2,32,1 > gpurun_out/jit_probe6_$TAG.txt 2>&1
LAYERS=res2a_branch2b,res4a_branch2b,res5a_branch2b NO_AUTOTUNE=1 FLUSH=1 timeout 900 python tools/jit_probe.py resnet50 64,1,8,3,16,1 64,1,16,2,16,1 32,1,8,3,16,1 32,1,16,3,16,1 16,1,8,3,32,1 > gpurun_out/jit_probe6r_$TAG.txt 2>&1
