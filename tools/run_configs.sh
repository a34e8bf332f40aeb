# BASELINE configs beyond the headline c2 (one bench line each)
mkdir -p gpurun_out
run() { echo "== $*"; python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 2 "$@" 2>gpurun_out/cfg.err | tail -1; tail -2 gpurun_out/cfg.err; }
run --config c1
run --config c3
for p in 5 6; do for g in 0 1 2; do run --config c4 --precision $p --go-up $g; done; done
for p in 3 4 5 7; do run --config c3 --precision $p; done
