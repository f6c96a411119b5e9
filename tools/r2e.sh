#!/bin/bash
cd $GRAFT_REPO_ROOT
TAG=r02e
timeout 1500 python bench.py --out gpurun_out/bench_resnet50_${TAG}.json > gpurun_out/${TAG}_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
for spec in "res2a_branch2b 32,1,0,0,16,2" "res3a_branch2b,res5a_branch2b 32,1,0,0,24,1"; do
  set -- $spec
  n=$(echo $1 | cut -c1-5)
  timeout 900 ncu --nvtx --nvtx-include "prof/" --set full --import-source on --clock-control none -f -o /tmp/p_$n \
    python tools/prof_jit.py resnet50 $1 $2 > gpurun_out/${TAG}_ncu_$n.log 2>&1
  ncu -i /tmp/p_$n.ncu-rep --page raw --csv > gpurun_out/prof_${n}_${TAG}_raw.csv 2>&1
  ncu -i /tmp/p_$n.ncu-rep --page source --csv --print-source sass > /tmp/sass_$n.csv 2>&1
  python tools/sass_summary.py /tmp/sass_$n.csv > gpurun_out/prof_${n}_${TAG}_sass_summary.txt 2>&1
  head -c 2000000 /tmp/sass_$n.csv > gpurun_out/prof_${n}_${TAG}_sass_head.csv
done
du -sh gpurun_out/* > gpurun_out/${TAG}_du.txt
