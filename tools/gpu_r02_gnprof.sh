#!/bin/bash
# one ncu --set full capture of the GroupNorm backward kernels of a Depth step, summarised on the box
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none -k "regex:gn_bwd_kernel|gn_fwd_kernel" -s 20 -c 4 -o /tmp/gn $B > gpurun_out/ncu_gn.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/gn.ncu-rep --page details --csv > /tmp/gn_details.csv 2>/dev/null
python - <<'PY'
import csv
rows = list(csv.reader(open('/tmp/gn_details.csv')))
h = rows[0]
ki, si, mi, vi, ui = h.index('Kernel Name'), h.index('Section Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
want = ('Duration', 'Achieved Occupancy', 'Theoretical Occupancy', 'Registers Per Thread', 'Block Size', 'Grid Size',
        'Memory Throughput', 'DRAM Throughput', 'Compute (SM) Throughput', 'Dynamic Shared Memory Per Block',
        'Waves Per SM', 'Block Limit Shared Mem', 'Block Limit Registers', 'L2 Hit Rate', 'Executed Ipc Active',
        'Stall Long Scoreboard', 'Stall Barrier', 'Stall Short Scoreboard', 'Warp Cycles Per Issued Instruction',
        'Stall Wait', 'Stall Math Pipe Throttle', 'Stall MIO Throttle', 'Stall LG Throttle')
seen = set()
for r in rows[1:]:
    if len(r) > vi and r[mi] in want:
        key = (r[0], r[mi])
        if key in seen: continue
        seen.add(key)
        print(r[0], r[ki].split('(')[0][:40], '|', r[mi], r[vi], r[ui])
PY
