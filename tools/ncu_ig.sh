ncu --set full --import-source on --clock-control none -k regex:igemm_kernel -s 1 -c 1 -o gpurun_out/ig_fwd -f python bench.py --config depth --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_ig.log 2>&1
echo rc=$?
tail -3 gpurun_out/ncu_ig.log
