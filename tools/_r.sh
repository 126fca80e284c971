WL=cfg4 KERN=k_sparse_count8 OUT=gpurun_out/ncu_c8f bash tools/ncu_capture.sh
ncu -i gpurun_out/ncu_c8f.ncu-rep --page details > gpurun_out/ncu_c8f_details.txt 2>&1
ncu -i gpurun_out/ncu_c8f.ncu-rep --page raw --csv > gpurun_out/ncu_c8f_raw.csv 2>&1
rm -f gpurun_out/ncu_c8f.ncu-rep
WL=cfg3 KERN=k_neuron_split OUT=gpurun_out/ncu_kns bash tools/ncu_capture.sh
rm -f gpurun_out/ncu_kns.ncu-rep
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/cfg4_launches.csv python bench.py --workload cfg4 --steps 4 --warmup 3 --no-cpu --no-per-config > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/cfg3_launches.csv python bench.py --workload cfg3 --steps 4 --warmup 3 --no-cpu --no-per-config > /dev/null 2>&1
ls gpurun_out
