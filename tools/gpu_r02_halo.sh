#!/bin/bash
# TC_HALO conv path: layer + network parity first (bounded), then A/B against the im2col path
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_depth_layers.py -x -q > gpurun_out/pytest_halo1.log 2>&1; echo "layers rc=$?"; tail -15 gpurun_out/pytest_halo1.log | cut -c1-300
timeout 900 python -m pytest tests -m gpu -x -q -k "depth_network or rgbd_network or chain" > gpurun_out/pytest_halo2.log 2>&1; echo "nets rc=$?"; tail -5 gpurun_out/pytest_halo2.log | cut -c1-300
for i in 1 2; do for m in 0 1; do
DDPPO_TCONV_HALO=$m timeout 300 python bench.py --config depth --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('halo $m', round(d['value']), d['ms_per_step'])"
done; done
for m in 0 1; do DDPPO_TCONV_HALO=$m timeout 300 python bench.py --config rgbd --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('rgbd halo $m', round(d['value']), d['ms_per_step'])"; done
