#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 120 ./tools/rnn_floor > gpurun_out/rnn_floor3.txt 2>&1; echo "floor rc=$?"; head -8 gpurun_out/rnn_floor3.txt
