# Round-end profiling bundle (run on the GPU box): bench line, launch list of
# the same bench command (host loop), one ncu --set full capture of a whole
# host-loop epoch -> per-kernel-class table, graph-epoch timings.  Each ncu
# pass runs only after the plain command exited 0.
set -x
O=gpurun_out/${1:-final}
mkdir -p $O
timeout 900 python bench.py --steps 3 --warmup 3 > $O/bench.json 2> $O/bench.err || exit 1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_bench.csv python bench.py --steps 1 --warmup 0 --host-loop --no-cpu-baseline --no-config4 \
  > $O/ncu_bench.log 2>&1
python tools/ncu_target.py 1 > $O/nt.log 2>&1 || exit 1
timeout 1500 ncu --set full --import-source on --clock-control none -o $O/epoch512 -f \
  python tools/ncu_target.py 1 > $O/ncu_epoch.log 2>&1
ncu -i $O/epoch512.ncu-rep --page raw --csv 2> /dev/null | gzip > $O/epoch512_raw.csv.gz
python tools/ncu_epoch_table.py $O/epoch512_raw.csv.gz --out $O/ncu_epoch512.json > $O/ncu_epoch512.txt 2>&1
for e in 5 200; do python tools/graph_epoch.py --epochs $e >> $O/graph_epochs.txt 2>&1; done
python tools/profile_epoch.py --size 512 --json $O/profile_epoch_512.json > $O/profile_epoch_512.txt 2>&1
python tools/profile_epoch.py --size 1024 > $O/profile_epoch_1024.txt 2>&1
python tools/profile_epoch.py --size 4096 > $O/profile_epoch_4096.txt 2>&1
rm -f $O/epoch512.ncu-rep
ls -la $O; cut -c1-300 $O/bench.json; tail -5 $O/ncu_epoch512.txt
