#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_cases.py);
# logs under gpurun_out/sanitize/, summary on stdout.
mkdir -p gpurun_out/sanitize
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  for fam in ${FAMS:-bulk short long tma packed crs build coo host}; do
    timeout ${TMO:-900} compute-sanitizer --tool $tool --target-processes all \
      --error-exitcode 99 --print-limit 20 \
      python tools/sanitize_cases.py $fam > gpurun_out/sanitize/${tool}_${fam}.log 2>&1
    rc=$?
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/sanitize/${tool}_${fam}.log | sort | uniq -c | tr '\n' ';')
    echo "$tool $fam rc=$rc $summ"
  done
done
