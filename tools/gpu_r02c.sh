#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log | cut -c1-300
for eng in tma cpasync; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --conv-engine $eng > gpurun_out/bench_depth_$eng.json 2> gpurun_out/bench_depth_$eng.err; echo "bench $eng rc=$?"; cut -c1-700 gpurun_out/bench_depth_$eng.json
done
timeout 600 python tools/kprof.py depth > gpurun_out/kprof_depth.txt 2>&1; echo "kprof rc=$?"; head -45 gpurun_out/kprof_depth.txt | cut -c1-200
