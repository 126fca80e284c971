# compute-sanitizer over the hot kernels (tools/sanitize_cases.py); one log per
# tool x case under ${OUT:-gpurun_out/sanitize}.
out=${OUT:-gpurun_out/sanitize}
mkdir -p "$out"
for tool in memcheck racecheck synccheck initcheck; do
  for c in dense_tma dense_tma_delay cluster tiny count16 sparse_pull p2p; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py $c > "$out/${tool}_${c}.txt" 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' "$out/${tool}_${c}.txt" | tail -1)"
  done
done
