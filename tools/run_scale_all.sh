# GPS weak scaling on one box (N = 1, 2, 4) + the stress config at N = 4.  Output: gpurun_out/scale/
mkdir -p gpurun_out/scale
python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/scale/gps_1.json 2> gpurun_out/scale/gps_1.err
for N in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py \
    --gpus $N --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/scale/gps_$N.json 2> gpurun_out/scale/gps_$N.err
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py \
  --gpus 4 --config stress --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/scale/stress_4.json 2> gpurun_out/scale/stress_4.err
echo done
