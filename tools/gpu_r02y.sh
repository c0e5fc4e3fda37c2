#!/bin/bash
# LSTM-1024 (lstm_wide.cu) parity + regression of the 512 path
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "lstm1024" > gpurun_out/pytest_y1.log 2>&1; echo "pytest lstm1024 rc=$?"; tail -30 gpurun_out/pytest_y1.log | cut -c1-400
timeout 900 python -m pytest tests -m gpu -x -q -k "gps or depth or rgbd or learner or act" > gpurun_out/pytest_y2.log 2>&1; echo "pytest rest rc=$?"; tail -3 gpurun_out/pytest_y2.log
