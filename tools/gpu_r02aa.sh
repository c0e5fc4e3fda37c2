#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail -20 gpurun_out/build.log; exit 1; }
timeout 120 ./tools/rnn_floor > gpurun_out/rnn_floor2.txt 2>&1; echo "floor rc=$?"; cat gpurun_out/rnn_floor2.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "lstm1024" > gpurun_out/pytest_aa.log 2>&1; echo "pytest lstm1024 rc=$?"; tail -2 gpurun_out/pytest_aa.log
timeout 600 python tools/kprof.py depth 5 1024 > gpurun_out/kprof_depth1024b.txt 2>&1; grep -E "lstm|ms/step" gpurun_out/kprof_depth1024b.txt | head -4
