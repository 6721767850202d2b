# profiling experiment helper: per-kernel durations of the tcgen05 conv under N2F_TC_DEBUG modes
mkdir -p gpurun_out
python tools/ncu_target.py 1 ${IMPL:-3} > gpurun_out/nt.log 2>&1 || exit 1
for d in ${MODES:-0 31}; do
  N2F_TC_DEBUG=$d timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_conv3x3_tc" -c 16 --csv python tools/ncu_target.py 1 ${IMPL:-3} > gpurun_out/ncu_dbg$d.csv 2>/dev/null
done
