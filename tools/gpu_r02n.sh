#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "rgbd_network or serx" > gpurun_out/pytest_serx.log 2>&1; echo "rc=$?"; grep -E "passed|failed|^FAILED|^E  " gpurun_out/pytest_serx.log | cut -c1-300 | head -30
