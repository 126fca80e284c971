# A/B of k_neuron min-blocks-per-SM builds (libsnmat_nb<N>.so, -DSNB_NEURON_MINB=<N>) on cfg4:
# ncu launch durations of k_neuron (serialised) + the bench step time without ncu
for lib in "" ${LIBS}; do
  env ${lib:+SNB_LIB=$PWD/$lib} timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_neuron --launch-skip 20 -c 40 --csv \
    python bench.py --workload ${WL:-cfg4} --steps 30 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python3 -c "
import csv,sys
r=[x for x in csv.reader(l for l in sys.stdin if l.startswith('\"'))]
h=r[0]; i=h.index('Metric Value'); v=[float(x[i].replace(',','')) for x in r[1:] if x[h.index('Metric Name')]=='gpu__time_duration.sum']
print('$lib', 'k_neuron mean', sum(v)/len(v), 'n', len(v))"
  for rep in 1 2; do env ${lib:+SNB_LIB=$PWD/$lib} python bench.py --workload ${WL:-cfg4} --steps 30 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', round(d['ms_per_step'],4))"; done
done
