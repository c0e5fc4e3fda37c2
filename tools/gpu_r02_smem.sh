#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
for c in depth rgbd; do S=50; [ $c = rgbd ] && S=6; timeout 600 python bench.py --config $c --steps $S --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/smem_$c.json 2>gpurun_out/smem_$c.err; echo "$c rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/smem_$c.json')); r=d['roofline']; print('$c', round(d['value']), r['frac'], r.get('smem'))"; done
