#!/bin/bash
# LSTM-1024: act parity, kernel timing on the Depth config, the paper's best agent (SE-ResNeXt101 + LSTM-1024) bench
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_collect.py -x -q > gpurun_out/pytest_z.log 2>&1; echo "pytest collect rc=$?"; tail -3 gpurun_out/pytest_z.log
timeout 600 python tools/kprof.py depth 5 1024 > gpurun_out/kprof_depth1024.txt 2>&1; grep -E "lstm|ms/step" gpurun_out/kprof_depth1024.txt | head -6
for c in serx101 serx101_1024; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; echo "bench $c rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['value']), d['ms_per_step'], d.get('e2e',{}).get('value'))"
done
