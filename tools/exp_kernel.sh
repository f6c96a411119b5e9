#!/bin/bash
cd $GRAFT_REPO_ROOT
for m in 0 1 2 4 7; do
ESCOIN_DEBUG_KERNEL=$m timeout 300 python tools/variant_sweep.py alexnet > gpurun_out/exp_kernel_$m.log 2>&1
done
