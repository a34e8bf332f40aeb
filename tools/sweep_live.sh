# live-mode consult tuning sweep (prints one line per setting)
mkdir -p gpurun_out
for r in ${ROUNDS:-0}; do for s in ${SHORTS:-1 8 32 128}; do
  python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 2 --live-rounds $r --consult-short $s 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rounds $r short $s', d['value'], d['full_traversal_mrays_s'], {k:v['ms_per_frame'] for k,v in d['stages'].items()})"
done; done
