# compare traversal kernel variants built under exp/*/ (tools/trace_bench.py)
for d in exp/*/; do echo "$d $(HRPP_LIB=$d/libhrpp_b200.so python tools/trace_bench.py --persistent 1 2>&1 | tail -1)"; done
echo "one-ray-per-thread $(python tools/trace_bench.py --persistent 0 2>&1 | tail -1)"
