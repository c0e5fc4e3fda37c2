#!/bin/bash
# compute-sanitizer, one tool per call (B200_PROFILING.md), on toy-sized calls of the cluster / mbarrier /
# TMA / peer-flag kernels: tconv (FPROP / DGRAD / WGRAD / stride-2 phases), GroupNorm incl. the cluster
# backward, LSTM + GRU recurrences, the peer a8 / a10 emulation, the act path
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
TOOL=$1
K="test_conv2d and tma and (2-16-32-32-3-1-1 or 2-16-32-64-3-2-1 or 5-2-256-128) or test_groupnorm and (2-16-1024 or 3-1024-32) or test_gps_network_parity and 3-37 or test_depth_network_parity and 2-6-2 or test_peer_a8_emulated and 4-4099 or test_peer_counts_emulated and 2 or test_policy_act_matches_oracle_step and gps-4"
timeout 2400 compute-sanitizer --tool $TOOL --print-limit 50 --log-file gpurun_out/sanitizer_$TOOL.log python -m pytest tests/test_gpu_depth_layers.py tests/test_gpu_parity.py tests/test_gpu_peer_emu.py tests/test_gpu_collect.py -q -k "$K" -p no:cacheprovider > gpurun_out/sanitizer_${TOOL}_pytest.log 2>&1
echo "$TOOL rc=$?"; tail -3 gpurun_out/sanitizer_${TOOL}_pytest.log; tail -5 gpurun_out/sanitizer_$TOOL.log
