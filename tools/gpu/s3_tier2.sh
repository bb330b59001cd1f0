QLM_LIB_PATH=build/variants/libqlm_trem.so timeout 900 python -m pytest tests -q -m gpu -x -k "tier or tiers" 2>&1 | tail -2
for r in 1 2 3; do for v in tcur trem; do QLM_LIB_PATH=build/variants/libqlm_$v.so python tools/tier_time.py; done; done
