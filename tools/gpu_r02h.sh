#!/bin/bash
# 2-GPU lease: multi-rank parity test + a8 forms at N=2
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/pytest_multi.log 2>&1; echo "multi rc=$?"; grep -E "passed|failed|^E  |Error" gpurun_out/pytest_multi.log | head -20 | cut -c1-300
for cfg in depth gps; do for a8 in sharded allread; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 30 --warmup 5 --config $cfg --a8 $a8 --no-e2e > gpurun_out/bench_${cfg}_n2_$a8.json 2> gpurun_out/bench_${cfg}_n2_$a8.err; echo "bench $cfg n2 $a8 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_${cfg}_n2_$a8.json')); print(d['value'], d['ms_per_step'], d['kernel_ms'].get('allreduce'))"
done; done
