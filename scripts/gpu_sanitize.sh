mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
for T in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $T --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitize_$T.log 2>&1
  echo "$T rc $? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$T.log | tail -1)"
done
