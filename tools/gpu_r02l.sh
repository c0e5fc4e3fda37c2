#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/pytest_multi.log 2>&1; echo "multi rc=$?"; grep -E "passed|failed|^E  |Error" gpurun_out/pytest_multi.log | head -20 | cut -c1-300
