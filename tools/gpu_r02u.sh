#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
for i in 1 2; do for m in 2 4 8 1000; do for k in 1 2; do
DDPPO_GEMM_MINCH=$m DDPPO_GEMM_SMMUL=$k timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('minch $m smmul $k', round(d['value']), d['ms_per_step'])"
done; done; done
