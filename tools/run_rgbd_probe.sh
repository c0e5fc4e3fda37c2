timeout 900 python -m pytest tests/test_gpu_depth_layers.py tests/test_gpu_parity.py -q -x -k "depth or rgbd or conv2d or groupnorm or maxpool" 2>&1 | tail -3 > gpurun_out/rgbd_tests.txt
python bench.py --config rgbd --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/rgbd_bench.json 2> gpurun_out/rgbd_bench.err || tail -5 gpurun_out/rgbd_bench.err
python bench.py --config depth --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/depth_bench.json 2> gpurun_out/depth_bench.err || tail -5 gpurun_out/depth_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rgbd_launches.csv python bench.py --config rgbd --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done
