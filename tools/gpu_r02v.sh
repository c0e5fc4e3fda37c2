#!/bin/bash
# recurrence floor microbench + ncu --set full over one whole Depth learner step (per-kernel table)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
timeout 120 ./tools/rnn_floor > gpurun_out/rnn_floor.txt 2>&1; echo "floor rc=$?"; cat gpurun_out/rnn_floor.txt
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain2.log 2>&1 && timeout 2700 ncu --set full --clock-control none -s 800 -c 760 -o /tmp/r02_depth_step $B > gpurun_out/ncu_f.log 2>&1; echo "ncu full rc=$?"
ls -la /tmp/r02_depth_step.ncu-rep
python tools/make_kernel_table.py /tmp/r02_depth_step.ncu-rep depth > gpurun_out/kt.log 2>&1; echo "table rc=$?"; cat gpurun_out/kt.log | head -20
mkdir -p gpurun_out/profiles && cp profiles/r02_kernels_depth.md profiles/r02_traffic.json gpurun_out/profiles/
du -sh gpurun_out
