# Round profiling bundle (run on the GPU box): bench line, launch list of the
# same bench command, full ncu captures of the dominant kernels, graph-epoch
# timings.  Each ncu pass runs only after the plain command exited 0.
set -x
mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --host-loop --no-cpu-baseline \
  > gpurun_out/ncu_bench.log 2>&1
python tools/ncu_target.py 1 > gpurun_out/nt.log 2>&1 || exit 1
# one host-loop epoch: k_conv3x3_dy launches 0..6 = fwd L2..L8 (6 = L8 + head), 7 = dgrad L8
cap() {  # name regex skip
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$2" --launch-skip $3 \
    --launch-count 1 -o gpurun_out/$1 -f python tools/ncu_target.py 1 > gpurun_out/ncu_$1.log 2>&1
}
cap fwdL8 k_conv3x3_dy 6
cap dgL8 k_conv3x3_dy 7
cap wgL8 k_wgrad3x3_tc 0
cap fwdL2 k_conv3x3_dy 0
cap adam k_adam 0
for e in 5 60 200; do python tools/graph_epoch.py --epochs $e >> gpurun_out/graph_epochs.txt 2>&1; done
N2F_PDL=0 python tools/graph_epoch.py --epochs 60 > gpurun_out/graph_nopdl.txt 2>&1
python tools/profile_epoch.py --size 512 --json gpurun_out/profile_epoch_512.json > gpurun_out/profile_epoch_512.txt 2>&1
echo done
