#!/bin/bash
# 2-GPU lease: multi-rank parity test + depth / gps benches at N=2
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail gpurun_out/build.log; exit 1; }
nvidia-smi -L
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/pytest_multi.log 2>&1; echo "multi rc=$?"; grep -E "passed|failed|^E  |Error" gpurun_out/pytest_multi.log | head -20 | cut -c1-300
for cfg in depth gps; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 5 --config $cfg > gpurun_out/bench_${cfg}_n2.json 2> gpurun_out/bench_${cfg}_n2.err; echo "bench $cfg n2 rc=$?"; cut -c1-250 gpurun_out/bench_${cfg}_n2.json
done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_depth_n1.json 2>/dev/null; cut -c1-200 gpurun_out/bench_depth_n1.json
