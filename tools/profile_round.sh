# Round profile set (one GPU): bench line, launch lists, ncu --set full of the bench's kernels,
# HBM microbenchmarks.  Output: gpurun_out/prof/
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"gps_gru|head_loss|gemm_bf16|adam_kernel|peer_|gae_kernel" \
    -s 20 -c 8 -o gpurun_out/prof/gps_full -f python tools/prof_step.py 3 gps > gpurun_out/prof/ncu_gps.log 2>&1
python bench.py --config depth --steps 20 --warmup 3 > gpurun_out/prof/depth_bench.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/depth_launches.csv \
    python bench.py --config depth --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"igemm_kernel|gn_bwd_kernel|gn_fwd_kernel|lstm_fwd" \
    -s 40 -c 6 -o gpurun_out/prof/depth_full -f python tools/prof_step.py 2 depth > gpurun_out/prof/ncu_depth.log 2>&1
python bench.py --config rgbd --steps 5 --warmup 3 > gpurun_out/prof/rgbd_bench.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/rgbd_launches.csv \
    python bench.py --config rgbd --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/microbench.py > gpurun_out/prof/microbench.jsonl 2> gpurun_out/prof/microbench.err
echo done
