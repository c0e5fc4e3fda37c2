#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests/test_gpu_parity.py -q -k "network_parity or learner" --durations=15 > gpurun_out/pytest_parity.log 2>&1; echo "parity rc=$?"; grep -E "passed|failed|Error|assert|^FAILED|s call" gpurun_out/pytest_parity.log | cut -c1-400 | head -60
