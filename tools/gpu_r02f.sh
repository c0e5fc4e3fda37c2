#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^E  " gpurun_out/pytest_gpu.log | cut -c1-300 | head -30
for cfg in depth rgbd; do
timeout 900 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; echo "bench $cfg rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_$cfg.json')); print(d['value'], d['ms_per_step'], d['e2e'])"
done
