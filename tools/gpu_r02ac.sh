#!/bin/bash
# kernel gaps on the critical stream + the per-kernel ncu table (reduced sections)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python tools/gaps.py depth 3 2>&1 | grep -v Warn | tail -6
timeout 300 python tools/gaps.py gps 3 2>&1 | grep -v Warn | tail -4
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain3.log 2>&1 && timeout 1800 ncu --section SpeedOfLight --section ComputeWorkloadAnalysis --section MemoryWorkloadAnalysis --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -s 800 -c 700 -o /tmp/r02_depth_k $B > gpurun_out/ncu_k.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_k.log
python tools/make_kernel_table.py /tmp/r02_depth_k.ncu-rep depth > gpurun_out/kt2.log 2>&1; echo "table rc=$?"; head -16 gpurun_out/kt2.log
mkdir -p gpurun_out/profiles && cp profiles/r02_kernels_depth.md profiles/r02_traffic.json gpurun_out/profiles/
