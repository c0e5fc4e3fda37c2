#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_depth_layers.py -q -k conv2d > gpurun_out/pytest_conv.log 2>&1; echo "conv rc=$?"; tail -40 gpurun_out/pytest_conv.log | cut -c1-300
