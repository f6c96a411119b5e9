#!/bin/bash
cd $GRAFT_REPO_ROOT
for m in 0 1 2; do
ESCOIN_DEBUG_CODES=$m timeout 300 python tools/variant_sweep.py alexnet > gpurun_out/exp_codes_$m.log 2>&1
done
