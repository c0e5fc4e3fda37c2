#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_transfer.py tests/test_gpu_parity.py -q -k "transfer or chain or reinit or freeze or goal" > gpurun_out/pytest_tr.log 2>&1; echo "rc=$?"; grep -E "passed|failed|^FAILED|^E  " gpurun_out/pytest_tr.log | cut -c1-300 | head -30
