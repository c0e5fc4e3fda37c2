#!/bin/bash
# phase trace of the GRU recurrence (debug build with DDPPO_TRACE)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
bash tools/build_trace.sh > gpurun_out/build_trace.log 2>&1 || { echo TRACE BUILD FAIL; tail gpurun_out/build_trace.log; exit 1; }
timeout 300 python tools/trace_gru.py 2>&1 | tail -8
