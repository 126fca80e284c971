python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_full.txt 2>&1; tail -3 gpurun_out/pytest_gpu_full.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 100 gpurun_out/bench_final.json
ncu --set full --clock-control none -k regex:k_cluster_count -s 1 -c 1 -o gpurun_out/ncu_cl python bench.py --workload cfg2 --steps 200 --warmup 3 --no-cpu --no-e2e --no-per-config > /dev/null 2>&1
ncu -i gpurun_out/ncu_cl.ncu-rep --page details > gpurun_out/ncu_cl_details.txt 2>&1; rm -f gpurun_out/ncu_cl.ncu-rep
