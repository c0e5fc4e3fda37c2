mkdir -p gpurun_out/prof
ncu --set full --import-source on --clock-control none -k regex:"gps_gru|head_loss|gemm_bf16|adam_kernel|gae_kernel" \
    -s 20 -c 8 -o gpurun_out/prof/gps_full -f python tools/prof_step.py 3 gps > gpurun_out/prof/ncu_gps.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"igemm_kernel|gn_bwd_kernel|gn_fwd_kernel|lstm_fwd" \
    -s 40 -c 6 -o gpurun_out/prof/depth_full -f python tools/prof_step.py 2 depth > gpurun_out/prof/ncu_depth.log 2>&1
echo done
