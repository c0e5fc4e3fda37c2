#!/bin/bash
# e2e at N = 4: one vs two device rollout arenas (GPS, Depth)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
port=29800
for r in 1 2; do for c in gps depth; do for a in 1 2; do
port=$((port+1))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py \
  --gpus 4 --config $c --no-cpu-baseline --steps 100 --warmup 5 --e2e-arenas $a > gpurun_out/e2e4.json 2>gpurun_out/e2e4_$c$a.err; echo "rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/e2e4.json')); print('$c arenas $a', round(d['value']), round(d['e2e']['value']))" || tail -5 gpurun_out/e2e4_$c$a.err
done; done; done
