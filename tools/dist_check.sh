# N=1 bench three ways: plain, distributed key sharding (NCCL, 1 rank) and
# distributed ray blocks; the stats and table stats must agree exactly.
set -e
mkdir -p gpurun_out
python bench.py --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/d_plain.json
python bench.py --no-cpu-baseline --steps 2 --warmup 3 --force-dist --shard keys > gpurun_out/d_keys.json
python bench.py --no-cpu-baseline --steps 2 --warmup 3 --force-dist --shard blocks > gpurun_out/d_blocks.json
python - <<'PY'
import json
r = {k: json.loads(open(f"gpurun_out/d_{k}.json").read().splitlines()[-1]) for k in ("plain", "keys", "blocks")}
for k in ("keys", "blocks"):
    for f in ("limit_stats", "live_stats", "table_stats", "nodes_skipped_percent"):
        print(k, f, "OK" if r[k][f] == r["plain"][f] else f"MISMATCH {r[k][f]} vs {r['plain'][f]}")
for k, v in r.items():
    print(k, v["value"], v["e2e"]["value"] if v.get("e2e") else None, v["config"]["parallelism"])
PY
