# Launch list of one host-loop epoch + full captures of the narrow-layer and
# non-conv kernels (run on the GPU box after the plain command exited 0).
mkdir -p gpurun_out
python tools/ncu_target.py 1 > gpurun_out/nt.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
  --log-file gpurun_out/launches_epoch.csv python tools/ncu_target.py 1 > /dev/null 2>&1
cap() {  # name regex skip
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$2" --launch-skip $3 \
    --launch-count 1 -o gpurun_out/$1 -f python tools/ncu_target.py 1 > gpurun_out/ncu_$1.log 2>&1
}
cap fwdL2 "k_conv3x3_dy" 0
cap wgL2 "k_wgrad3x3_tc" 6
cap wgL3 "k_wgrad3x3_tc" 5
cap dgL3 "k_conv3x3_dy" 12
cap first_fwd "k_conv_first" 0
cap first_wg "k_wgrad_first" 0
cap adam "k_adam" 0
echo done
