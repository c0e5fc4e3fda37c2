#!/bin/bash
# 4-GPU lease: scaling lines at N=4 (depth both a8 forms, gps, stress)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail gpurun_out/build.log; exit 1; }
run() { # cfg a8 n
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $3 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $3 --steps 30 --warmup 5 --config $1 --a8 $2 > gpurun_out/bench_$1_n$3_$2.json 2> gpurun_out/bench_$1_n$3_$2.err; echo "bench $1 n$3 $2 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_$1_n$3_$2.json')); print(d['value'], d['ms_per_step'], d['kernel_ms'].get('allreduce'), d['e2e']['value'])"
}
run depth sharded 4; run depth allread 4; run gps auto 4; run stress auto 4
