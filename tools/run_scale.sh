N=$1
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/scale_gps_$N.json 2> gpurun_out/scale_gps_$N.err
