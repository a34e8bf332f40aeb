# coherence-sort key width sweep: begin bit of the 30-bit key (fewer bits = fewer radix passes)
for bb in 22 14 6; do echo "begin_bit $bb $(HRPP_COH_BEGIN_BIT=$bb python tools/trace_bench.py --coherent 1 | tail -1)"; done
echo "no-sort $(python tools/trace_bench.py --coherent 0 | tail -1)"
