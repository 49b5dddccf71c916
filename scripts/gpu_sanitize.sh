# compute-sanitizer over one toy detection (race detection / sanitizers)
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_toy.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool: exit $?"; tail -3 gpurun_out/sanitize_$tool.log
done
