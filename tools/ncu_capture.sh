# One ncu --set full capture of a workload's sweep kernel + the raw DRAM bytes:
#   WL=cfg3 KERN=k_dense_tma OUT=gpurun_out/ncu_cfg3 bash tools/ncu_capture.sh
WL=${WL:-cfg3}; KERN=${KERN:-k_dense_tma}; OUT=${OUT:-gpurun_out/ncu_$WL}
ncu --set full --clock-control none --import-source on -k regex:$KERN -s 3 -c 1 -o $OUT \
  python bench.py --workload $WL --steps 4 --warmup 3 --no-cpu --no-e2e --no-per-config > $OUT.log 2>&1
ncu -i $OUT.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv, sys
r = list(csv.reader(sys.stdin)); h, u, v = r[0], r[1], r[2]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size']
for k in want:
    if k in h: i = h.index(k); print(k, v[i], u[i])
" > $OUT.raw.txt
cat $OUT.raw.txt
