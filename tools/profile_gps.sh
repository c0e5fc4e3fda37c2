# GPS-only profile refresh (one GPU): bench line, launch list, ncu --set full, CUPTI split.  Output: gpurun_out/prof/
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"gps_gru|gemm_bf16|adam_kernel|grad_norm|gae1_kernel" \
    -s 20 -c 9 -o gpurun_out/prof/gps_full -f python tools/prof_step.py 3 gps > gpurun_out/prof/ncu_gps.log 2>&1
python tools/kprof.py gps 20 > gpurun_out/prof/kprof_gps.txt 2>&1
echo done
