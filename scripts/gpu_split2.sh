for k in 2 1; do
  DART_ATTN_SPLIT=$k timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none \
    --csv --log-file gpurun_out/launches_split$k.csv python scripts/profile_step.py --classes 4 > /dev/null 2>&1
  python scripts/summarize_launches.py gpurun_out/launches_split$k.csv > gpurun_out/launches_split$k.txt 2>&1
  echo "== split $k"; head -1 gpurun_out/launches_split$k.txt; grep -E "fa_tc_kernel<16|split_combine" gpurun_out/launches_split$k.txt
done
