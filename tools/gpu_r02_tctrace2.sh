#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
for m in 1 0; do echo "=== DDPPO_TCONV_HALO=$m"; DDPPO_TCONV_HALO=$m timeout 300 python tools/trace_tconv.py depth 2>&1 | grep -v Warn | grep -v warn_once | head -40; done
