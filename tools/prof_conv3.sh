#!/bin/bash
# ncu --set full captures of chosen variants on one layer (WL, LAYER, KS env).
cd $GRAFT_REPO_ROOT
WL=${WL:-alexnet}
LAYER=${LAYER:-conv3}
for k in ${KS:-t3s1_q4_4x4_x}; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:sconv -s 1 -c 1 -f -o gpurun_out/prof_${LAYER}_$k python tools/prof_layer.py $WL $LAYER $k > gpurun_out/prof_${LAYER}_$k.log 2>&1
done
