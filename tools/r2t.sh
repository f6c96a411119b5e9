#!/bin/bash
# HP parity + FFMA2/HP A/B on res2a/res4a + ncu of res2a (scalar best, FFMA2, HP)
cd "$(dirname "$0")/.."
TAG=r02t
timeout 1200 python -m pytest tests/test_jit_gpu.py -x -q -k "horizontal or parity_grid" > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
H=0,0,0,0,0,0,0,0,1
T="32,1,8,3,16,2;48,1,8,3,16,2;32,2,8,3,16,1,-1;32,2,8,3,16,1,-1,$H;32,2,8,3,16,1,0,$H;32,2,8,3,32,1,-1;32,2,8,3,32,1,-1,$H;16,2,8,3,32,1,-1,$H;48,2,8,3,16,1,-1,$H"
timeout 1200 python tools/ab.py resnet50 res2a_branch2b,res4a_branch2b "$T" 20 > gpurun_out/${TAG}_ab.jsonl 2> gpurun_out/${TAG}_ab.err
for t in "32,1,8,3,16,2" "32,2,8,3,16,1,-1" "32,2,8,3,16,1,-1,$H"; do
  n=$(echo $t | tr ',' '_')
  timeout 600 ncu --nvtx --nvtx-include "prof/" --set full --import-source on --clock-control none -k regex:escoin_jit -c 1 -f \
    -o /tmp/p_$n python tools/prof_jit.py resnet50 res2a_branch2b $t > gpurun_out/${TAG}_ncu_$n.log 2>&1
  ncu -i /tmp/p_$n.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw_$n.csv 2>&1
  ncu -i /tmp/p_$n.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_src_$n.csv 2>&1
done
ls -la gpurun_out/ >> gpurun_out/${TAG}_tests.log
