timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -3 > gpurun_out/gpu_tests.txt
python bench.py --steps 50 --warmup 5 > gpurun_out/gps_bench.json 2> gpurun_out/gps_bench.err || tail -5 gpurun_out/gps_bench.err
python bench.py --config depth --steps 20 --warmup 3 > gpurun_out/depth_bench.json 2> gpurun_out/depth_bench.err || tail -5 gpurun_out/depth_bench.err
echo done
