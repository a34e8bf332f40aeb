# BASELINE configs beyond the headline c5: one bench line each (JSON lines
# to gpurun_out/configs.jsonl; stderr tails to configs.err)
mkdir -p gpurun_out
: > gpurun_out/configs.jsonl
run() { python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 2 "$@" 2>>gpurun_out/configs.err | tail -1 >> gpurun_out/configs.jsonl; }
run --config c1
for p in 3 4 5 6 7; do run --config c3 --precision $p; done
for p in 5 6; do for g in 0 1 2; do run --config c4 --precision $p --go-up $g; done; done
run --config c2
python - <<'PY'
import json
for ln in open("gpurun_out/configs.jsonl"):
    d = json.loads(ln)
    c = d["config"]
    print(c["workload"].split(":")[0], "p%s g%s" % (c["precision"], c["go_up"]), d["value"],
          d["full_traversal_mrays_s"], d["nodes_skipped_percent"])
PY
