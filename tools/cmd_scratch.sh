cd $GRAFT_REPO_ROOT
cat > /tmp/tcprof.py <<'PY'
import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_1802_10280_b200 import escoin, inputs, workloads
W = workloads.workload("alexnet"); L = [l for l in W.layers if l.name == "conv3"][0]
w = torch.from_numpy(inputs.layer_weights(W.net, L, 800)).cuda()
x = torch.from_numpy(inputs.activations(W.net, L.name, 0, 128, L.C, L.H, L.W)).cuda()
for _ in range(2): escoin.bench_dense_tc_forward(w, x, None, 1, 1, True, 1)
torch.cuda.synchronize()
PY
timeout 300 ncu --set full --import-source on --clock-control none -k regex:dense_tc -s 1 -c 1 -f -o gpurun_out/prof_tc python /tmp/tcprof.py > gpurun_out/prof_tc.log 2>&1
