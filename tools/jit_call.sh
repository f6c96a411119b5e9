cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_jit_gpu.py -x -q > gpurun_out/pytest_jit.txt 2>&1
LAYERS=conv3,conv2 timeout 600 python tools/jit_probe.py alexnet 0,0,0,0,0,0 32,2,8,3,8,2 64,1,8,3,16,1 64,1,16,2,8,2 > gpurun_out/jit_probe_alexnet.txt 2>&1
LAYERS=res2a_branch2b,res3a_branch2b,res4a_branch2b,res5a_branch2b timeout 600 python tools/jit_probe.py resnet50 0,0,0,0,0,0 32,2,8,3,8,2 > gpurun_out/jit_probe_resnet.txt 2>&1
