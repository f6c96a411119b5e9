#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python tools/variant_sweep.py alexnet > gpurun_out/sweep_g14.log 2>&1
for k in ${KS:-t3s1_q1_4x4 t3s1_q2_4x4}; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:sconv -s 1 -c 1 -f -o gpurun_out/prof_conv3_$k python tools/prof_layer.py alexnet conv3 $k > gpurun_out/prof_conv3_$k.log 2>&1
done
