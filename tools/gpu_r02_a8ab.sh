#!/bin/bash
# a8 form at N = 4 for GPS (P = 0.9 M): all-read (AUTO's choice) vs sharded
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
port=29900
for r in 1 2; do for m in allread sharded; do
port=$((port+1))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py \
  --gpus 4 --config gps --no-cpu-baseline --no-e2e --steps 100 --warmup 5 --a8 $m > gpurun_out/a8.json 2>gpurun_out/a8_$m.err; echo "rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/a8.json')); print('gps a8 $m', round(d['value']), d['ms_per_step'])" || tail -3 gpurun_out/a8_$m.err
done; done
