#!/bin/bash
# round-2 final weak-scaling set on one box: N = 1 and N (= number of visible GPUs) for Depth (the
# metric's config) and GPS; the stress config (configs[4]) at N = 4; the 2-rank GPU tests at N = 2
cd $GRAFT_REPO_ROOT
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
mkdir -p gpurun_out/scale
if [ "$N" = "2" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "depth_network or depth_layers or chain" > gpurun_out/scale/pytest_depth.log 2>&1; echo "depth tests rc=$?"; tail -2 gpurun_out/scale/pytest_depth.log; timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/scale/pytest_multi.log 2>&1; echo "multi rc=$?"; tail -2 gpurun_out/scale/pytest_multi.log; fi
for c in depth gps; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/scale/${c}_n1.json 2> gpurun_out/scale/${c}_n1.err; echo "$c n1 rc=$?"
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N bench.py \
    --gpus $N --config $c --no-cpu-baseline > gpurun_out/scale/${c}_n$N.json 2> gpurun_out/scale/${c}_n$N.err; echo "$c n$N rc=$?"
done
if [ "$N" = "4" ]; then
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29641 bench.py \
    --gpus 4 --config stress --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/scale/stress_n4.json 2> gpurun_out/scale/stress_n4.err; echo "stress rc=$?"
fi
for f in gpurun_out/scale/*.json; do python -c "
import json; d=json.load(open('$f')); print('$f', round(d['value']), d['ms_per_step'], (d.get('e2e') or {}).get('value'), d.get('clocks'))"; done
