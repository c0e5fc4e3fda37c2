#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
timeout 300 python tools/trace_tconv.py depth > gpurun_out/tctrace_depth.txt 2>&1; echo "rc=$?"; cat gpurun_out/tctrace_depth.txt | grep -v Warn | tail -80
