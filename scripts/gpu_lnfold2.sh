# LN fold masks (DART_LN_FOLD bit 0 LN1 -> QKV, bit 1 LN2 -> fc1): parity, launch lists, bench A/B
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "full_width" -s 2>&1 | grep -E "fold|passed|failed|Error" | head -20
for f in 1 0; do
  DART_LN_FOLD=$f timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none \
    --csv --log-file gpurun_out/launches_fold$f.csv python scripts/profile_step.py --classes 4 > /dev/null 2>&1
  python scripts/summarize_launches.py gpurun_out/launches_fold$f.csv > gpurun_out/launches_fold$f.txt 2>&1
  echo "== fold $f"; head -9 gpurun_out/launches_fold$f.txt
done
for i in 1 2; do for f in 1 0; do
  DART_LN_FOLD=$f timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-n80 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('fold $f', round(d['value'],2), round(d['e2e']['value'],2), round(d['value_serial'],2), 'launches', d['gpu_launches'])"
done; done
