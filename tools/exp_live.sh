# live-frame bench (stage split) for the shipped lib and every exp/*/ variant
line() { python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 2 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['full_traversal_mrays_s'], {k:v['ms_per_frame'] for k,v in d['stages'].items()})"; }
echo "shipped $(line "$@")"
for d in exp/*/; do [ -f "$d/libhrpp_b200.so" ] && echo "$d $(HRPP_LIB=$d/libhrpp_b200.so line "$@")"; done
true
