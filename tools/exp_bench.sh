# compare library variants built under exp/*/ on the bench (c2 live frame):
# value, full traversal, ms/frame and stage times.  Usage: bash tools/exp_bench.sh [bench args]
shopt -s nullglob
for L in "" exp/*/libhrpp_b200.so; do
  HRPP_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/eb.log 2>&1
  python - "$L" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/eb.log").read().strip().splitlines()[-1])
    print(sys.argv[1] or "shipped", d["value"], d["full_traversal_mrays_s"], d["ms_per_step"],
          {k: v["ms_per_frame"] for k, v in d["stages"].items()})
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
