# query-tile chains per CTA (hd 16 variants 6-10) vs production: correctness (bench_attn checks), interleaved A/B
for v in 7; do DART_FA_VARIANT=$v timeout 300 python scripts/bench_attn.py 2>&1 | grep -E "hd=16|enc self"; done
timeout 600 python scripts/ab_attn.py 0 6 7 8 9 10 2>&1 | grep -v "bb "
