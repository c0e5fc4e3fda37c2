#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_depth_layers.py -q -x -k conv2d > gpurun_out/pytest_conv.log 2>&1; echo "conv rc=$?"; grep -E "passed|failed|^FAILED|^E  " gpurun_out/pytest_conv.log | cut -c1-300 | head -20
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "gpu rc=$?"; grep -E "passed|failed|^FAILED|^E  " gpurun_out/pytest_gpu.log | cut -c1-300 | head -20
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_depth.json 2> gpurun_out/bench_depth.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_depth.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'])"
timeout 900 python tools/kprof.py depth 5 > gpurun_out/kprof_depth.txt 2>&1; head -30 gpurun_out/kprof_depth.txt | cut -c1-160
