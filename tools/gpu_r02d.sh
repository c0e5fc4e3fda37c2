#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_depth_layers.py -q -x -k conv2d > gpurun_out/pytest_conv.log 2>&1; echo "conv rc=$?"; tail -5 gpurun_out/pytest_conv.log | cut -c1-300
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log | cut -c1-300
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_depth_tma.json 2> gpurun_out/bench_depth_tma.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/bench_depth_tma.json
timeout 600 python tools/kprof.py depth > gpurun_out/kprof_depth.txt 2>&1; echo "kprof rc=$?"; head -45 gpurun_out/kprof_depth.txt | cut -c1-200
