# Round profile set (one GPU): bench lines, launch lists, ncu --set full of the top kernels,
# CUPTI per-kernel splits for depth / rgbd, HBM microbenchmarks.  Output: gpurun_out/prof/
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"gps_gru|head_loss|gemm_bf16|adam_kernel|gae1_kernel" \
    -s 20 -c 8 -o gpurun_out/prof/gps_full -f python tools/prof_step.py 3 gps > gpurun_out/prof/ncu_gps.log 2>&1
python tools/kprof.py gps 20 > gpurun_out/prof/kprof_gps.txt 2>&1
python bench.py --config depth --steps 20 --warmup 3 > gpurun_out/prof/depth_bench.json 2>/dev/null
python tools/kprof.py depth 5 > gpurun_out/prof/kprof_depth.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:"igemm_kernel|gn_bwd|gn_fwd|lstm_fwd|stem_wgrad" \
    -s 40 -c 8 -o gpurun_out/prof/depth_full -f python tools/prof_step.py 2 depth > gpurun_out/prof/ncu_depth.log 2>&1
python bench.py --config rgbd --steps 5 --warmup 3 > gpurun_out/prof/rgbd_bench.json 2>/dev/null
python tools/kprof.py rgbd 2 > gpurun_out/prof/kprof_rgbd.txt 2>&1
python tools/microbench.py > gpurun_out/prof/microbench.jsonl 2> gpurun_out/prof/microbench.err
# then, here: cp the captures into profiles/ and run tools/make_traffic.py + tools/make_summary.py
echo done
