#!/bin/bash
# round-2 profile set (part 2): ncu --set full of one Depth learner step's top kernels, summarised on the box
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain2.log 2>&1 && timeout 2400 ncu --set full --clock-control none -k "regex:tconv|gn_|lstm|stem|maxpool|adam|grad_norm|gemm_bf16|relu_mask|weights_prep" -s 400 -c 40 -o /tmp/r02_depth_full $B > gpurun_out/ncu_f.log 2>&1; echo "ncu full rc=$?"
python tools/make_kernel_table.py /tmp/r02_depth_full.ncu-rep depth > gpurun_out/kt.log 2>&1; echo "table rc=$?"; tail -5 gpurun_out/kt.log
mkdir -p gpurun_out/profiles && cp profiles/r02_kernels_depth.md profiles/r02_traffic.json gpurun_out/profiles/
ncu -i /tmp/r02_depth_full.ncu-rep --page details --csv > /tmp/details.csv 2>/dev/null; gzip -c /tmp/details.csv > gpurun_out/r02_depth_full_details.csv.gz
ls -la /tmp/r02_depth_full.ncu-rep; S=$(stat -c %s /tmp/r02_depth_full.ncu-rep); if [ $S -lt 40000000 ]; then cp /tmp/r02_depth_full.ncu-rep gpurun_out/; fi
du -sh gpurun_out
