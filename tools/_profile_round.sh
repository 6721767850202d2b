# Round profiling bundle (run on the GPU box): bench line, launch list of the
# same bench command, one full ncu capture of the dominant conv kernel.
set -x
mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_bench.log 2>&1
python tools/ncu_target.py 1 3 > gpurun_out/nt.log 2>&1 || exit 1
# dominant kernel: dgrad L8 = 8th k_conv3x3_tc launch of an epoch (fwd L2..L8, then dgrad L8)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_conv3x3_tc" \
  --launch-skip 7 --launch-count 1 -o gpurun_out/dominant python tools/ncu_target.py 1 3 \
  > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_wgrad3x3_tc" \
  --launch-count 1 -o gpurun_out/wgrad8 python tools/ncu_target.py 1 3 > gpurun_out/ncu_wg.log 2>&1
echo done
