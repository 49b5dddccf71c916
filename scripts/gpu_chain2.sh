# chain A/B: serial stage times and warm launch lists (ncu serialises: per-kernel durations)
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "full_width and B-0" 2>&1 | tail -1
for i in 1 2; do for c in 1 0; do
  DART_CHAIN=$c timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-n80 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('chain $c', round(d['value'],2), round(d['value_serial'],2), d['stage_ms_serial'])"
done; done
for c in 1 0; do
  DART_CHAIN=$c timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none \
    --csv --log-file gpurun_out/launches_chain$c.csv python scripts/profile_step.py --classes 4 > /dev/null 2>&1
  python scripts/summarize_launches.py gpurun_out/launches_chain$c.csv > gpurun_out/launches_chain$c.txt 2>&1
  echo "== chain $c"; head -10 gpurun_out/launches_chain$c.txt
done
