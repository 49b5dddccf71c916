for m in 0 2; do echo "=== DART_FA_SOFTMAX_ONLY=$m"; DART_FA_SOFTMAX_ONLY=$m python scripts/trace_attn.py 16 2>&1 | sed -n '22,45p;46,70p' | grep -v "^$" | tail -32; done
