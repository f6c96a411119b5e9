#!/bin/bash
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/mb_smi.txt 2>&1
nproc > gpurun_out/mb_host.txt; lscpu | grep -E 'Model name|^CPU\(s\)' >> gpurun_out/mb_host.txt
timeout 300 ./tools/microbench > gpurun_out/mb1.txt 2>&1

