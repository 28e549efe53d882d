mkdir -p gpurun_out
out=gpurun_out/${OUT:-sanitizer_r01.txt}
: > $out
for tool in memcheck racecheck synccheck; do
  for k in ${CASES:-0 1 2 3 4 5 6 7 8 9 10 11 12 13}; do
    echo "=== $tool case $k" >> $out
    timeout 600 compute-sanitizer --tool $tool --print-limit 5 python tools/sanitize_cases.py $k >> $out 2>&1
    echo "exit=$?" >> $out
  done
done
grep -E "^===|ERROR SUMMARY|exit=|^[0-9]+ " $out | paste - - - - | head -40
