cd $GRAFT_REPO_ROOT
WL=alexnet TAG=r01j bash tools/gpu_bench.sh
for wl in resnet50 googlenet googlenet_1x1 resnet50_v15; do
timeout 900 python bench.py --workload $wl --no-cpu --out gpurun_out/bench_${wl}_r01j.json > gpurun_out/bench_${wl}_r01j.log 2>&1
done
cat > /tmp/tcprof.py <<'PY'
import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_1802_10280_b200 import escoin, inputs, workloads
W = workloads.workload("alexnet"); L = [l for l in W.layers if l.name == "conv3"][0]
w = torch.from_numpy(inputs.layer_weights(W.net, L, 800)).cuda()
x = torch.from_numpy(inputs.activations(W.net, L.name, 0, 128, L.C, L.H, L.W)).cuda()
for ns in (1, 3):
    for _ in range(2): escoin.bench_dense_tc_forward(w, x, None, 1, 1, True, ns)
torch.cuda.synchronize()
PY
timeout 300 ncu --set full --clock-control none -k regex:dense_tc -f -o gpurun_out/prof_tc_r01j python /tmp/tcprof.py > gpurun_out/prof_tc_r01j.log 2>&1
