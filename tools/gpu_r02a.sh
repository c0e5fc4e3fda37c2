#!/bin/bash
# round-2 check: build, full GPU test suite, default bench (depth) + GPS line
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_depth.json 2> gpurun_out/bench_depth.err; echo "bench rc=$?"; cat gpurun_out/bench_depth.json
timeout 600 python bench.py --config gps --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_gps.json 2> gpurun_out/bench_gps.err; echo "gps rc=$?"; cat gpurun_out/bench_gps.json
