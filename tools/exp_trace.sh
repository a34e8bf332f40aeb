# compare traversal kernel variants built under exp/*/ (tools/trace_bench.py);
# the shipped lib first.  Usage: bash tools/exp_trace.sh [trace_bench args]
echo "shipped $(python tools/trace_bench.py "$@" 2>&1 | tail -1)"
for d in exp/*/; do [ -f "$d/libhrpp_b200.so" ] && echo "$d $(HRPP_LIB=$d/libhrpp_b200.so python tools/trace_bench.py "$@" 2>&1 | tail -1)"; done
true
